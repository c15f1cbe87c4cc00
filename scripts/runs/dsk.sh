T=gpurun_out/dsk; mkdir -p $T
for tpc in 1 256 512 1024 2048; do
  echo "== tokens/CTA $tpc" >> $T/out.txt
  DS_BRIEF=1 PQKV_STEP_TOKENS_PER_CTA=$tpc timeout 300 python scripts/ds_time.py 2>&1 | grep -v Warn | grep -v _warn >> $T/out.txt
done
cat $T/out.txt
