#!/bin/bash
# A/B the library variants (paper_2504_03661_b200/_lib/ab_*.so) in both value-codebook modes
T=${1:-abm}; shift
bash scripts/ab.sh $T "$@"
bash scripts/ab.sh ${T}_f16 --f16-value-codebook "$@"
