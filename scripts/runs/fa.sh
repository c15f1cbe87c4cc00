T=gpurun_out/fa; mkdir -p $T
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_paged_store.py tests/test_serving_cache.py -q -x > $T/pytest.log 2>&1; echo "pytest rc=$?" >> $T/status.txt
for v in fa1 fa0; do
  echo "== $v" >> $T/out.txt
  PQKV_SM100_LIB=paper_2504_03661_b200/_lib/ab_$v.so DS_BRIEF=1 timeout 300 python scripts/ds_time.py 2>&1 | grep -v -i warn >> $T/out.txt
  PQKV_SM100_LIB=paper_2504_03661_b200/_lib/ab_$v.so timeout 300 python scripts/step_hist.py 2>&1 | grep "rep 2" >> $T/out.txt
done
tail -1 $T/pytest.log; cat $T/out.txt
