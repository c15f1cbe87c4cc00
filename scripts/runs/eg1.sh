T=gpurun_out/eg1; mkdir -p $T
timeout 600 python -m pytest tests/test_gpu_encode_grid.py -q -x -rf > $T/pytest_grid.log 2>&1; echo "grid rc=$?" >> $T/status.txt
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-f16-mode --no-extra-configs > $T/bench.json 2> $T/bench.err; echo "bench rc=$?" >> $T/status.txt
cat $T/status.txt
