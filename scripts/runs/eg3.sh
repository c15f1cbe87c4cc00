T=gpurun_out/eg3; mkdir -p $T
for lib in paper_2504_03661_b200/_lib/ab_*.so; do
  n=$(basename $lib .so)
  PQKV_SM100_LIB=$lib timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-f16-mode --no-extra-configs > $T/$n.json 2> $T/$n.err
  python -c "
import json; j=json.loads(open('$T/$n.json').read().strip().splitlines()[-1]); e=j['encode']; print('$n', round(e['vectors_per_s']/1e6,1), round(e['full_scan']['vectors_per_s']/1e6,1), e['bit_exact'])" >> $T/summary.txt 2>&1
done
cat $T/summary.txt
