for v in lazy0 lazy8; do echo "== $v"; PQKV_SM100_LIB=paper_2504_03661_b200/_lib/ab_$v.so timeout 300 python scripts/lazy_err.py; done
