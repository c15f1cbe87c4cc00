# refreshed evidence after the GQA select-free reductions + lazy rescale
T=gpurun_out/r02k; mkdir -p $T
timeout 600 python bench.py --steps 20 --warmup 3 > $T/bench.json 2> $T/bench.err; echo "bench rc=$?" >> $T/status.txt
timeout 600 python bench.py --steps 10 --warmup 3 --config llama3-gqa-32k --no-cpu-baseline > $T/bench_gqa.json 2> $T/bench_gqa.err; echo "bench3 rc=$?" >> $T/status.txt
timeout 600 python bench.py --steps 5 --warmup 3 --config llama3-gqa-128k --no-cpu-baseline --no-encode > $T/bench_128k.json 2> $T/bench_128k.err; echo "bench4 rc=$?" >> $T/status.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:decode_gqa_pair -s 2 -c 1 -o $T/pair python scripts/gqa_layer.py --mode exact > $T/ncu_pair.log 2>&1; echo "ncu pair rc=$?" >> $T/status.txt
python scripts/ncu_summary.py $T/pair.ncu-rep > $T/pair.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:decode_gqa4 -s 2 -c 1 -o $T/quad python scripts/gqa_layer.py --mode quad > $T/ncu_quad.log 2>&1; echo "ncu quad rc=$?" >> $T/status.txt
python scripts/ncu_summary.py $T/quad.ncu-rep > $T/quad.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:decode_partials_m64b8 -s 40 -c 1 -o $T/decode_full python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-encode --no-f16-mode > $T/ncu_full.log 2>&1; echo "ncu mha rc=$?" >> $T/status.txt
python scripts/ncu_summary.py $T/decode_full.ncu-rep > $T/mha.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $T/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-encode --no-f16-mode > $T/ncu_bench.log 2>&1; echo "launches rc=$?" >> $T/status.txt
python scripts/launch_summary.py $T/launches.csv > $T/launches_summary.txt 2>&1
cat $T/status.txt
