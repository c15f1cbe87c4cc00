"""One config-3 (or config-4) GQA layer decoded a few times through PQDecoder --
the target of ncu captures of the GQA kernels.
usage: python scripts/gqa_layer.py [--n 32768] [--B 16] [--mode quad|pair|f16|exact] [--reps 5]"""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2504_03661_b200 import kernels as K
from paper_2504_03661_b200.engine import PQDecoder, random_codes
from paper_2504_03661_b200.pq_core import PQConfig

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=32768)
ap.add_argument("--B", type=int, default=16)
ap.add_argument("--mode", default="quad", choices=["quad", "pair", "f16", "exact"])
ap.add_argument("--reps", type=int, default=5)
a = ap.parse_args()
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev); g.manual_seed(0)
Hq, Hkv, R = 32, 8, 31
ck = random_codes((a.B, Hkv, a.n, 64), 8, g, dev)
cv = random_codes((a.B, Hkv, a.n, 64), 8, g, dev)
half = a.mode != "exact"
cbk = K.key_codebook_layout(torch.randn((64, 256, 2), generator=g, device=dev), 8)
cbv = K.value_codebook_layout(torch.randn((64, 256, 2), generator=g, device=dev), 8, half=half)
q = torch.randn((a.B, Hq, 128), generator=g, device=dev)
rk = torch.randn((a.B, Hkv, R, 128), generator=g, device=dev); rv = torch.randn_like(rk)
kc = torch.randn((a.B, Hkv, 128), generator=g, device=dev); vc = torch.randn_like(kc)
nq = torch.full((a.B,), a.n, dtype=torch.int32, device=dev)
nr = torch.full((a.B,), R, dtype=torch.int32, device=dev)
dec = PQDecoder(a.B, Hq, Hkv, PQConfig(128, 64, 8), device=dev,
                f16_key_table=a.mode in ("quad", "pair"), key_table_pairs=a.mode == "pair")
for _ in range(a.reps):
    out = dec(q, ck, cv, nq, cbk, cbv, rk, rv, nr, kc, vc)
torch.cuda.synchronize()
print("ok", a.mode, float(out.abs().mean()))
