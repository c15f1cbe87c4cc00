T=gpurun_out/lz; mkdir -p $T
PQKV_SM100_LIB=paper_2504_03661_b200/_lib/ab_lazy0.so timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "lazy" > $T/lazy0.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "lazy" > $T/lazy8.log 2>&1
grep -E "passed|failed|Max abs|Max rel" $T/lazy0.log $T/lazy8.log
