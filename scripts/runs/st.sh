T=gpurun_out/st; mkdir -p $T
for n in st1 st0; do
PQKV_SM100_LIB=paper_2504_03661_b200/_lib/ab_$n.so timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-f16-mode --no-extra-configs > $T/$n.json 2> $T/$n.err
python -c "
import json; j=json.loads(open('$T/$n.json').read().strip().splitlines()[-1]); e=j['encode']; print('$n', round(e['vectors_per_s']/1e6,1))" >> $T/summary.txt 2>&1
done
cat $T/summary.txt
