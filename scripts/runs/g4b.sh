T=gpurun_out/g4b; mkdir -p $T
timeout 900 python -m pytest tests/test_gpu_gqa_tables.py -q -rf > $T/pytest.log 2>&1; echo "pytest rc=$?" >> $T/status.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:decode_gqa4 -s 2 -c 1 -o $T/quad python scripts/gqa_layer.py --mode quad > $T/ncu_quad.log 2>&1; echo "ncu rc=$?" >> $T/status.txt
python scripts/ncu_summary.py $T/quad.ncu-rep > $T/ncu_quad.txt 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 --config llama3-gqa-32k --no-cpu-baseline --no-encode > $T/bench_gqa.json 2> $T/bench_gqa.err; echo "bench rc=$?" >> $T/status.txt
cat $T/status.txt
