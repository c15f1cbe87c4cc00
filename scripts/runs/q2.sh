T=gpurun_out/q2; mkdir -p $T
timeout 600 python -m pytest tests/test_gpu_gqa_tables.py tests/test_gpu_full_shapes.py -q -x > $T/pytest.log 2>&1; echo "pytest rc=$?" >> $T/status.txt
timeout 600 python bench.py --steps 10 --warmup 3 --config llama3-gqa-32k --no-cpu-baseline --no-encode > $T/bench_gqa.json 2> $T/bench_gqa.err; echo "bench3 rc=$?" >> $T/status.txt
cat $T/status.txt
