T=gpurun_out/${1:-tg}; mkdir -p $T
timeout 1800 python -m pytest tests -m gpu -q -x -rf > $T/pytest.log 2>&1; echo "pytest rc=$?" >> $T/status.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $T/smoke.log 2>&1; echo "smoke rc=$?" >> $T/status.txt
tail -3 $T/pytest.log; cat $T/status.txt
