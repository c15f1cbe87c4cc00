"""Build library variants for A/B runs (scripts/ab.sh, ab_modes.sh, ab_encode.sh).

usage: python scripts/build_variants.py name:DEF1=V,DEF2 name2: ...
       -> paper_2504_03661_b200/_lib/ab_<name>.so compiled with -D<DEF>...
Existing ab_*.so are removed first."""
import glob
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2504_03661_b200 import build as B  # noqa: E402

for f in glob.glob(os.path.join(B.OUT_DIR, "ab_*.so")):
    os.remove(f)
for spec in sys.argv[1:]:
    name, _, defs = spec.partition(":")
    d = tuple(x for x in defs.split(",") if x)
    B.build(force=True, lib=os.path.join(B.OUT_DIR, f"ab_{name}.so"), defines=d)
    print("built", name, d)
