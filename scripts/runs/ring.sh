T=gpurun_out/ring; mkdir -p $T
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_serving_cache.py tests/test_gpu_paged_store.py tests/test_gpu_seam.py tests/test_gpu_full_shapes.py -q -x > $T/pytest.log 2>&1; echo "pytest rc=$?" >> $T/status.txt
timeout 600 python scripts/runs/bd.py > $T/bd.txt 2>&1; echo "bd rc=$?" >> $T/status.txt
timeout 1200 python tests/ref_suite/run_ref_suite.py run $T/ref_suite.json > $T/ref_suite.log 2>&1; echo "ref rc=$?" >> $T/status.txt
tail -2 $T/pytest.log; cat $T/bd.txt | grep context; tail -2 $T/ref_suite.log; cat $T/status.txt
