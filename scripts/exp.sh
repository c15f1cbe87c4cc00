#!/bin/bash
# quick experiment loop: trace + bench (no CPU baseline) + ncu of one fused launch
T=${1:-exp}; mkdir -p gpurun_out/$T
python scripts/trace_decode.py > gpurun_out/$T/trace.txt 2>&1
timeout 300 python bench.py --no-cpu-baseline --no-encode --steps 100 > gpurun_out/$T/bench.json 2> gpurun_out/$T/bench.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:decode_partials_m64b8 -s 40 -c 1 \
  -o gpurun_out/$T/full python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-encode > gpurun_out/$T/ncu.log 2>&1
python scripts/ncu_summary.py gpurun_out/$T/full.ncu-rep > gpurun_out/$T/ncu_summary.txt 2>&1
