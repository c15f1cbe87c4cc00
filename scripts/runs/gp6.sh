T=gpurun_out/gp6; mkdir -p $T
PQKV_SM100_LIB=paper_2504_03661_b200/_lib/ab_f16pair.so timeout 600 python -m pytest tests/test_gpu_gqa_tables.py tests/test_gpu_full_shapes.py -q -x > $T/pytest.log 2>&1; echo "pytest rc=$?" >> $T/status.txt
for n in f16pair f16quad; do
PQKV_SM100_LIB=paper_2504_03661_b200/_lib/ab_$n.so timeout 600 python bench.py --steps 10 --warmup 3 --config llama3-gqa-32k --no-cpu-baseline --no-encode > $T/$n.json 2> $T/$n.err
python -c "
import json; j=json.loads(open('$T/$n.json').read().strip().splitlines()[-1]); f=j['f16_value_codebook_mode']; print('$n', round(j['value'],1), round(f['value'],1), round(f['f16_key_table']['value'],1), round(f['f16_key_table']['roofline_frac'],3))" >> $T/summary.txt 2>&1
done
cat $T/status.txt $T/summary.txt
