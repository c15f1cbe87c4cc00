set -u
OUT=gpurun_out/r02e; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_full_shapes.py -m gpu -q -rf -x > $OUT/pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/status.txt
bash scripts/ab.sh r02e_ab > /dev/null 2>&1; echo "ab rc=$?" >> $OUT/status.txt
bash scripts/ab.sh r02e_ab2 > /dev/null 2>&1
GRAPH=1 TRACE_LIB=paper_2504_03661_b200/_lib/libpqkv_sm100_trace.so timeout 300 python scripts/trace_graph.py > $OUT/trace.txt 2>&1; echo "trace rc=$?" >> $OUT/status.txt
cat $OUT/status.txt
