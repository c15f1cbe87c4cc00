T=gpurun_out/${1:-pwab}; mkdir -p $T
PQKV_SM100_LIB=paper_2504_03661_b200/_lib/ab_pw1.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_full_shapes.py tests/test_gqa4_layout.py -q -x -k "gqa or pair or full or config" > $T/pytest.log 2>&1; echo "pytest rc=$?" >> $T/status.txt
bash scripts/runs/lzab.sh ${1:-pwab}
tail -3 $T/pytest.log
