#!/bin/bash
# A/B the encoder of library variants: encode tests (bit-exactness) + bench encode rate
T=${1:-abe}; mkdir -p gpurun_out/$T
for lib in paper_2504_03661_b200/_lib/ab_*.so; do
  name=$(basename $lib .so)
  r=$(PQKV_SM100_LIB=$lib timeout 300 python -m pytest tests -m gpu -q -k "encode or smoke or cache or golden" 2>&1 | tail -1)
  PQKV_SM100_LIB=$lib timeout 300 python bench.py --steps 3 --no-cpu-baseline --no-f16-mode > gpurun_out/$T/$name.json 2>gpurun_out/$T/$name.err
  python -c "import json,sys; j=json.load(open('gpurun_out/$T/$name.json')); e=j['encode']; print('$name', round(e['value']), 'tok/s', round(e['vectors_per_s']/1e6,1), 'Mvec/s', 'bit_exact', e.get('bit_exact'), '|', '$r')"
done
