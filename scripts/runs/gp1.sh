T=gpurun_out/gp1; mkdir -p $T
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "gqa_exact" > $T/pytest_pair.log 2>&1; echo "pair rc=$?" >> $T/status.txt
cat $T/status.txt
