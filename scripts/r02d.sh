set -u
OUT=gpurun_out/r02d; mkdir -p $OUT
timeout 900 python -m pytest tests/test_fileio_c.py tests/test_gpu_seam.py tests/test_harness.py -m gpu -q -rf > $OUT/pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/status.txt
timeout 1200 python tests/ref_suite/run_ref_suite.py run $OUT/ref_suite.json > $OUT/ref_suite.log 2>&1; echo "refsuite rc=$?" >> $OUT/status.txt
cat $OUT/status.txt
