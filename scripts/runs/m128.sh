T=gpurun_out/m128; mkdir -p $T
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "lazy or batched or step_plan" > $T/pytest.log 2>&1; echo "pytest rc=$?" >> $T/status.txt
timeout 600 python bench.py --steps 5 --warmup 3 --config llama2-mha-128k --no-cpu-baseline --no-encode > $T/bench_mha128k.json 2> $T/bench_mha128k.err; echo "bench rc=$?" >> $T/status.txt
timeout 600 python bench.py --steps 3 --warmup 3 --config llama2-mha-128k --no-cpu-baseline --no-encode --seq-split-one --no-f16-mode > $T/bench_mha128k_split.json 2> $T/bench_mha128k_split.err; echo "split rc=$?" >> $T/status.txt
tail -3 $T/pytest.log; cat $T/status.txt
