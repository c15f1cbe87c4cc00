T=gpurun_out/pr; mkdir -p $T
timeout 600 ncu --set full --clock-control none --import-source on -k regex:decode_gqa_pair -s 2 -c 1 -o $T/pair python scripts/gqa_layer.py --mode exact > $T/ncu_pair.log 2>&1
python scripts/ncu_summary.py $T/pair.ncu-rep > $T/pair.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:decode_gqa4 -s 2 -c 1 -o $T/quad python scripts/gqa_layer.py --mode quad > $T/ncu_quad.log 2>&1
python scripts/ncu_summary.py $T/quad.ncu-rep > $T/quad.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:encode_dsub2_grid -s 1 -c 1 -o $T/grid python scripts/enc_grid_run.py > $T/ncu_grid.log 2>&1
python scripts/ncu_summary.py $T/grid.ncu-rep > $T/grid.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $T/launches_gqa.csv python bench.py --steps 2 --warmup 3 --config llama3-gqa-32k --no-cpu-baseline --no-encode --no-f16-mode > $T/ncu_bench3.log 2>&1
python scripts/launch_summary.py $T/launches_gqa.csv > $T/launches_gqa.txt 2>&1
ls $T
