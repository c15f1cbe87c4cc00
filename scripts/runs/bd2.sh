T=gpurun_out/bd2; mkdir -p $T
for tpc in 1 1024 4096; do
  echo "== tokens/CTA $tpc" >> $T/out.txt
  PQKV_STEP_TOKENS_PER_CTA=$tpc timeout 600 python scripts/runs/bd.py >> $T/out.txt 2>&1
done
cat $T/out.txt
