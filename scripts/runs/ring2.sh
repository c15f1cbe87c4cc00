T=gpurun_out/ring2; mkdir -p $T
timeout 1800 python -m pytest tests -m gpu -q -x > $T/pytest.log 2>&1; echo "pytest rc=$?" >> $T/status.txt
timeout 600 python scripts/runs/bd.py > $T/bd.txt 2>&1; echo "bd rc=$?" >> $T/status.txt
timeout 1200 python tests/ref_suite/run_ref_suite.py run $T/ref_suite.json > $T/ref_suite.log 2>&1; echo "ref rc=$?" >> $T/status.txt
tail -2 $T/pytest.log; cat $T/bd.txt | grep context; tail -2 $T/ref_suite.log; cat $T/status.txt
