T=gpurun_out/p3; mkdir -p $T
timeout 600 ncu --set full --clock-control none --import-source on -k regex:decode_gqa_pair -s 2 -c 1 -o $T/pair python scripts/gqa_layer.py --mode exact > $T/ncu_pair.log 2>&1; echo "ncu rc=$?" >> $T/status.txt
python scripts/ncu_summary.py $T/pair.ncu-rep > $T/ncu_pair.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:decode_gqa4 -s 2 -c 1 -o $T/quad python scripts/gqa_layer.py --mode quad > $T/ncu_quad.log 2>&1; echo "ncu rc=$?" >> $T/status.txt
python scripts/ncu_summary.py $T/quad.ncu-rep > $T/ncu_quad.txt 2>&1
cat $T/status.txt
