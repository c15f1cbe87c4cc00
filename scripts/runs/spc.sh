# decode_step (one head) vs the step plan's grid size and the finish batch
T=gpurun_out/spc; mkdir -p $T
for lib in paper_2504_03661_b200/_lib/ab_*.so; do
  for tpc in 1 256 512 1024 2048 4096; do
    echo "== $(basename $lib) tokens/CTA $tpc" >> $T/ds.txt
    PQKV_SM100_LIB=$lib PQKV_STEP_TOKENS_PER_CTA=$tpc timeout 300 python scripts/ds_time.py 2>&1 | grep "ctx" >> $T/ds.txt
  done
done
cat $T/ds.txt
bash scripts/runs/lzab.sh spc_ab
