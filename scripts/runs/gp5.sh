T=gpurun_out/gp5; mkdir -p $T
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "gqa" > $T/pytest.log 2>&1; echo "pytest rc=$?" >> $T/status.txt
timeout 600 python bench.py --steps 10 --warmup 3 --config llama3-gqa-32k --no-cpu-baseline --no-encode --no-f16-mode > $T/bench_gqa.json 2> $T/bench_gqa.err; echo "bench3 rc=$?" >> $T/status.txt
cat $T/status.txt
