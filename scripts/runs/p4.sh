T=gpurun_out/p4; mkdir -p $T
PQKV_SM100_LIB=paper_2504_03661_b200/_lib/ab_p4w16.so timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_full_shapes.py -q -x -k "gqa or full or randomized" > $T/pytest.log 2>&1; echo "pytest rc=$?" >> $T/status.txt
cat $T/status.txt
