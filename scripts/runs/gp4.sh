T=gpurun_out/gp4; mkdir -p $T
timeout 1500 python -m pytest tests -m gpu -q -rf > $T/pytest.log 2>&1; echo "pytest rc=$?" >> $T/status.txt
timeout 600 python bench.py --steps 10 --warmup 3 --config llama3-gqa-32k --no-cpu-baseline --no-encode > $T/bench_gqa.json 2> $T/bench_gqa.err; echo "bench3 rc=$?" >> $T/status.txt
timeout 600 python bench.py --steps 5 --warmup 3 --config llama3-gqa-128k --no-cpu-baseline --no-encode > $T/bench_128k.json 2> $T/bench_128k.err; echo "bench4 rc=$?" >> $T/status.txt
cat $T/status.txt
