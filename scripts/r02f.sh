set -u
OUT=gpurun_out/r02f; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_seam.py tests/test_gpu_parity.py -m gpu -q -rf > $OUT/pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/status.txt
timeout 1200 python tests/ref_suite/run_ref_suite.py run $OUT/ref_suite.json > $OUT/ref_suite.log 2>&1; echo "refsuite rc=$?" >> $OUT/status.txt
GRAPH=1 TRACE_LIB=paper_2504_03661_b200/_lib/libpqkv_sm100_trace.so timeout 300 python scripts/trace_graph.py > $OUT/trace.txt 2>&1; echo "trace rc=$?" >> $OUT/status.txt
bash scripts/ab.sh r02f_ab > /dev/null 2>&1; echo "ab rc=$?" >> $OUT/status.txt
bash scripts/ab.sh r02f_ab16 --f16-value-codebook --no-f16-mode > /dev/null 2>&1
cat $OUT/status.txt
