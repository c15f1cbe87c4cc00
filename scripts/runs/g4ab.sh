# A/B of the four-head kernel variants (_lib/ab_*.so) on config 3
T=gpurun_out/${1:-g4ab}; mkdir -p $T
for lib in paper_2504_03661_b200/_lib/ab_*.so; do
  name=$(basename $lib .so)
  PQKV_SM100_LIB=$lib timeout 400 python bench.py --config llama3-gqa-32k --no-cpu-baseline --no-encode --steps 20 > $T/$name.json 2> $T/$name.err
  python - $name $T/$name.json <<'PY' | tee -a $T/summary.txt
import json,sys
try:
    j=json.loads(open(sys.argv[2]).read().strip().splitlines()[-1])
    f=j["f16"]["f16_key_table"]
    print(f'{sys.argv[1]:12s} exact {j["value"]:8.1f} f16 {j["f16"]["value"]:8.1f} quad {f["value"]:8.1f} ({f["roofline_frac"]:.3f}) pair16 {f.get("two_heads_per_cta",{}).get("value",0):8.1f} sm {j["clocks"]["sm_mhz"]}')
except Exception as e: print(sys.argv[1], "FAILED", e)
PY
done
