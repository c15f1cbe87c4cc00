# A/B of library variants (_lib/ab_*.so) on config 2 (exact + fp16 value codebook) and config 3
T=gpurun_out/${1:-lzab}; mkdir -p $T
for rep in 1 2; do
for lib in paper_2504_03661_b200/_lib/ab_*.so; do
  name=$(basename $lib .so)
  PQKV_SM100_LIB=$lib timeout 400 python bench.py --no-cpu-baseline --no-encode --no-extra-configs --steps 30 > $T/${name}_c2_$rep.json 2> $T/${name}_c2_$rep.err
  PQKV_SM100_LIB=$lib timeout 400 python bench.py --config llama3-gqa-32k --no-cpu-baseline --no-encode --steps 20 > $T/${name}_c3_$rep.json 2> $T/${name}_c3_$rep.err
  python - $name $T/${name}_c2_$rep.json $T/${name}_c3_$rep.json <<'PY' | tee -a $T/summary.txt
import json,sys
try:
    a=json.loads(open(sys.argv[2]).read().strip().splitlines()[-1])
    b=json.loads(open(sys.argv[3]).read().strip().splitlines()[-1])
    f=b["f16_value_codebook_mode"]["f16_key_table"]
    print(f'{sys.argv[1]:10s} c2 exact {a["value"]:7.1f} ({a["roofline"]["frac"]:.3f}) f16 {a["f16_value_codebook_mode"]["value"]:7.1f} | c3 exact {b["value"]:7.1f} f16 {b["f16_value_codebook_mode"]["value"]:7.1f} quad {f["value"]:7.1f} ({f["roofline_frac"]:.3f}) | sm {a["clocks"]["sm_mhz"]} {b["clocks"]["sm_mhz"]}')
except Exception as e: print(sys.argv[1], "FAILED", e)
PY
done
done
