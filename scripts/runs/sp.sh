T=gpurun_out/sp; mkdir -p $T
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_serving_cache.py tests/test_gpu_paged_store.py tests/test_gpu_seam.py -q -x > $T/pytest.log 2>&1; echo "pytest rc=$?" >> $T/status.txt
timeout 300 python scripts/ds_time.py > $T/ds.txt 2>&1; echo "ds rc=$?" >> $T/status.txt
timeout 300 python scripts/prof_decode_step.py > $T/prof.txt 2>&1; echo "prof rc=$?" >> $T/status.txt
timeout 1200 python tests/ref_suite/run_ref_suite.py run $T/ref_suite.json > $T/ref_suite.log 2>&1; echo "ref rc=$?" >> $T/status.txt
cat $T/status.txt
