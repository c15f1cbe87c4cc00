# final evidence on the committed tree
T=gpurun_out/final; mkdir -p $T
timeout 1500 python -m pytest tests -m gpu -q > $T/pytest.log 2>&1; echo "pytest rc=$?" >> $T/status.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $T/smoke.log 2>&1; echo "smoke rc=$?" >> $T/status.txt
timeout 600 python bench.py > $T/bench.json 2> $T/bench.err; echo "bench rc=$?" >> $T/status.txt
timeout 600 python scripts/runs/bd.py > $T/bd.txt 2>&1; echo "bd rc=$?" >> $T/status.txt
timeout 1200 python tests/ref_suite/run_ref_suite.py run $T/ref_suite.json > $T/ref_suite.log 2>&1; echo "ref rc=$?" >> $T/status.txt
tail -1 $T/pytest.log; grep context $T/bd.txt; tail -1 $T/ref_suite.log; cat $T/status.txt
