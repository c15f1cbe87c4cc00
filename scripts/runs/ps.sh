T=gpurun_out/ps; mkdir -p $T
for n in ps0 ps1; do
  PQKV_SM100_LIB=paper_2504_03661_b200/_lib/ab_$n.so timeout 600 python scripts/quad_err.py > $T/err_$n.txt 2>&1
done
TAG=ps bash scripts/runs/pf.sh > /dev/null 2>&1
cat $T/err_*.txt $T/summary.txt
