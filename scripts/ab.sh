#!/bin/bash
# A/B the decode library variants built into paper_2504_03661_b200/_lib/ab_*.so
# (scripts/build_variants.py)
# usage (under gpurun): bash scripts/ab.sh <tag> [bench args...]
T=${1:-ab}; shift; mkdir -p gpurun_out/$T
for lib in paper_2504_03661_b200/_lib/ab_*.so; do
  name=$(basename $lib .so)
  PQKV_SM100_LIB=$lib timeout 300 python bench.py --no-cpu-baseline --no-encode --steps 50 "$@" \
     > gpurun_out/$T/$name.json 2> gpurun_out/$T/$name.err
  python - "$name" gpurun_out/$T/$name.json <<'PY' | tee -a gpurun_out/$T/summary.txt
import json,sys
try:
    j=json.loads(open(sys.argv[2]).read().strip().splitlines()[-1])
    r=j["roofline"]
    print(f'{sys.argv[1]:28s} {j["value"]:9.1f} tok/s  step {j["code_stream_gbs_step"]:7.0f} GB/s  kernel {r["kernel_ms_per_launch"]*1e3:6.1f} us {r["frac"]:.3f}  sm {j["clocks"]["sm_mhz"]}')
except Exception as e:
    print(sys.argv[1], "FAILED", e)
PY
done
