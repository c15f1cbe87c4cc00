# bench config 2 at several grid sizes (PQKV_BENCH_CTAS), exact and fp16 modes
T=${1:-ctas}; shift; mkdir -p gpurun_out/$T
for n in "$@"; do
  for mode in "" "--f16-value-codebook"; do
    PQKV_BENCH_CTAS=$n timeout 300 python bench.py --no-cpu-baseline --no-encode --no-f16-mode --steps 50 $mode > gpurun_out/$T/c$n$mode.json 2>/dev/null
    python -c "import json,sys;j=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]);print(sys.argv[2], sys.argv[3], round(j['value'],1), round(j['roofline']['frac'],3))" gpurun_out/$T/c$n$mode.json $n "x$mode" | tee -a gpurun_out/$T/summary.txt
  done
done
