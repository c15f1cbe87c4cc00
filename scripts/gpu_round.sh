#!/bin/bash
# One GPU session: parity tests, smoke, bench (+GQA config, reference arm),
# launch list + one full ncu capture of the decode kernel, step timeline.
# Usage (from the repo root, under gpurun): bash scripts/gpu_round.sh <tag> [stages]
set -u
TAG=${1:-r01}
STAGES=${2:-"test smoke bench ncu"}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > $OUT/gpu.txt 2>&1
for s in $STAGES; do
  case $s in
    test)
      timeout 1500 python -m pytest tests -m gpu -q -rf > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/status.txt ;;
    smoke)
      timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/status.txt ;;
    bench)
      timeout 600 python bench.py --steps 20 --warmup 3 > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?" >> $OUT/status.txt ;;
    bench3)
      timeout 600 python bench.py --steps 10 --warmup 3 --config llama3-gqa-32k --no-cpu-baseline > $OUT/bench_gqa.json 2> $OUT/bench_gqa.err; echo "bench3 rc=$?" >> $OUT/status.txt ;;
    ref)
      timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $OUT/bench_ref.json 2> $OUT/bench_ref.err; echo "ref rc=$?" >> $OUT/status.txt ;;
    trace)
      GRAPH=1 timeout 300 python scripts/trace_graph.py > $OUT/trace_graph.txt 2>&1; echo "trace rc=$?" >> $OUT/status.txt ;;
    ncu)
      timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
        --log-file $OUT/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-encode --no-f16-mode > $OUT/ncu_bench.log 2>&1
      echo "ncu-launches rc=$?" >> $OUT/status.txt
      python scripts/launch_summary.py $OUT/launches.csv > $OUT/launches_summary.txt 2>&1
      timeout 900 ncu --set full --clock-control none --import-source on -k regex:decode_partials_m64b8 -s 40 -c 1 \
        -o $OUT/decode_full python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-encode --no-f16-mode > $OUT/ncu_full.log 2>&1
      echo "ncu-full rc=$?" >> $OUT/status.txt
      python scripts/ncu_summary.py $OUT/decode_full.ncu-rep > $OUT/ncu_summary.txt 2>&1 ;;
  esac
done
cat $OUT/status.txt
