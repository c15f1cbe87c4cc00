#!/bin/bash
# A/B of the launch-order ramp: same library, PQKV_RAMP=ctas,slope at run time
# (and the previous library as the schedule baseline).  usage: bash scripts/ab_ramp.sh <tag> "<lib>:<ramp>" ...
T=$1; shift; mkdir -p gpurun_out/$T
for spec in "$@"; do
  lib=${spec%%:*}; ramp=${spec#*:}
  for mode in exact f16; do
    extra=""; [ $mode = f16 ] && extra="--f16-value-codebook"
    name=$(basename $lib .so)_${ramp/,/_}_$mode
    PQKV_SM100_LIB=paper_2504_03661_b200/_lib/$lib PQKV_RAMP=$ramp timeout 300 python bench.py --no-cpu-baseline --no-encode --no-f16-mode --no-extra-configs --steps 50 $extra \
      > gpurun_out/$T/$name.json 2> gpurun_out/$T/$name.err
    python - "$name" gpurun_out/$T/$name.json <<'PY' | tee -a gpurun_out/$T/summary.txt
import json,sys
try:
    j=json.loads(open(sys.argv[2]).read().strip().splitlines()[-1])
    print(f'{sys.argv[1]:34s} {j["value"]:8.1f} tok/s  frac {j["roofline"]["frac"]:.3f}  sm {j["clocks"]["sm_mhz"]}')
except Exception as e:
    print(sys.argv[1], "FAILED", e)
PY
  done
done
