T=gpurun_out/${TAG:-pf}; mkdir -p $T
for lib in paper_2504_03661_b200/_lib/ab_*.so; do
  n=$(basename $lib .so)
  PQKV_SM100_LIB=$lib timeout 600 python bench.py --steps 10 --warmup 3 --config llama3-gqa-32k --no-cpu-baseline --no-encode > $T/$n.json 2> $T/$n.err
  python -c "
import json; j=json.loads(open('$T/$n.json').read().strip().splitlines()[-1]); f=j['f16_value_codebook_mode']; print('$n', round(j['value'],1), round(f['value'],1), round(f['f16_key_table']['value'],1))" >> $T/summary.txt 2>&1
done
cat $T/summary.txt
