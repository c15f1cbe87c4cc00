mkdir -p gpurun_out/g4a
timeout 900 python -m pytest tests/test_gpu_gqa_tables.py tests/test_gpu_full_shapes.py -q -x -rf > gpurun_out/g4a/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/g4a/status.txt
timeout 600 python bench.py --steps 10 --warmup 3 --config llama3-gqa-32k --no-cpu-baseline --no-encode > gpurun_out/g4a/bench_gqa.json 2> gpurun_out/g4a/bench_gqa.err; echo "bench rc=$?" >> gpurun_out/g4a/status.txt
cat gpurun_out/g4a/status.txt
