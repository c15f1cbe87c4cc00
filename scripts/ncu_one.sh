#!/bin/bash
# ncu --set full of one fused decode launch in the bench step; summary into gpurun_out/<tag>/
T=${1:-exp}; shift; mkdir -p gpurun_out/$T
timeout 600 ncu --set full --clock-control none --import-source on -k regex:decode_partials_m64b8 -s 40 -c 1 \
  -o gpurun_out/$T/full python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-encode "$@" > gpurun_out/$T/ncu.log 2>&1
python scripts/ncu_summary.py gpurun_out/$T/full.ncu-rep > gpurun_out/$T/ncu_summary.txt 2>&1
cat gpurun_out/$T/ncu_summary.txt | head -30
