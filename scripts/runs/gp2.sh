T=gpurun_out/gp2; mkdir -p $T
timeout 1500 python -m pytest tests -m gpu -q -rf > $T/pytest.log 2>&1; echo "pytest rc=$?" >> $T/status.txt
timeout 600 python bench.py --steps 10 --warmup 3 --config llama3-gqa-32k --no-cpu-baseline --no-encode > $T/bench_gqa.json 2> $T/bench_gqa.err; echo "bench3 rc=$?" >> $T/status.txt
timeout 600 python bench.py --steps 5 --warmup 3 --config llama3-gqa-128k --no-cpu-baseline --no-encode > $T/bench_128k.json 2> $T/bench_128k.err; echo "bench4 rc=$?" >> $T/status.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:decode_gqa_pair -s 2 -c 1 -o $T/pair python scripts/gqa_layer.py --mode exact > $T/ncu_pair.log 2>&1; echo "ncu rc=$?" >> $T/status.txt
python scripts/ncu_summary.py $T/pair.ncu-rep > $T/ncu_pair.txt 2>&1
cat $T/status.txt
