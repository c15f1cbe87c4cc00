"""Diagnostic: the candidate-grid encoder on one config-5 layer (32K tokens x 8
KV heads, K), a few launches -- the target of ncu captures."""
import sys
sys.path.insert(0, '.')
import torch
from paper_2504_03661_b200 import kernels as K
g = torch.Generator(device="cuda"); g.manual_seed(7)
x = torch.randn((8 * 32768, 128), generator=g, device="cuda")
c = torch.randn((64, 256, 2), generator=g, device="cuda")
grid = K.encode_grid(c, 8)
out = torch.empty((x.shape[0], 64), dtype=torch.uint8, device="cuda")
for _ in range(4):
    K.encode(x, c, 8, out=out, layout="decode", grid=grid)
torch.cuda.synchronize()
print("ok")
