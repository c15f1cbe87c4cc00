"""Diagnostic: per-CTA timeline of the decode kernel (built with -DPQKV_TRACE).
usage: python scripts/trace_decode.py   (on a GPU box; prints a summary)"""
import ctypes, os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2504_03661_b200 import build as B
lib = os.environ.get("TRACE_LIB") or os.path.join(B.OUT_DIR, "libpqkv_sm100_trace.so")
if not os.path.exists(lib):
    B.build(force=True, lib=lib, defines=("PQKV_TRACE",))
os.environ["PQKV_SM100_LIB"] = lib
import torch
from paper_2504_03661_b200 import kernels as K, _native as N
if os.environ.get("TRACE_LIB"):  # an older library for A/B: bind what it has
    import ctypes as _c
    _l = _c.CDLL(lib)
    for _name in list(N.SIGNATURES):
        if not hasattr(_l, _name):
            del N.SIGNATURES[_name]
from paper_2504_03661_b200.engine import random_codes
dev = torch.device("cuda", 0)
B_, Hq, Hkv, n = [int(x) for x in (sys.argv[1:5] if len(sys.argv) > 4 else (1, 32, 32, 32768))]
g = torch.Generator(device=dev); g.manual_seed(0)
ck = random_codes((B_, Hkv, n, 64), 8, g, dev); cv = random_codes((B_, Hkv, n, 64), 8, g, dev)
cbk = K.key_codebook_layout(torch.randn((64, 256, 2), generator=g, device=dev), 8)
cbv = K.value_codebook_layout(torch.randn((64, 256, 2), generator=g, device=dev), 8)
q = torch.randn((B_ * Hq, 128), generator=g, device=dev)
nq = torch.full((B_,), n, dtype=torch.int32, device=dev)
ws = K.DecodeWorkspace(B_, Hq, 128, 64, 8, device=dev, num_ctas=int(os.environ.get("TRACE_CTAS", "0")) or None)
rk = torch.randn((B_, Hkv, 31, 128), generator=g, device=dev)
rv = torch.randn((B_, Hkv, 31, 128), generator=g, device=dev)
nr = torch.full((B_,), 31, dtype=torch.int32, device=dev)
out = torch.empty((B_ * Hq, 128), device=dev)
mode = os.environ.get("TRACE_MODE", "fused")
for _ in range(5):
    if mode == "fused":
        K.decode_attention(ws, Hkv, q, 0.088, cbk, ck, cv, nq, cbv, rk, rv, nr, out=out,
                           static_codebooks=os.environ.get("TRACE_STATIC") == "1")
    else:
        K.decode_partials(ws, Hkv, q, 0.088, cbk, ck, cv, nq, cbv)
torch.cuda.synchronize()
T = np.zeros(1024 * 16, dtype=np.uint64)
N.load().pqkv_debug_trace.argtypes = [ctypes.c_void_p, ctypes.c_int]
assert N.load().pqkv_debug_trace(T.ctypes.data, T.size) == 0
T = T.reshape(1024, 16)[: ws.num_ctas].astype(np.int64)
ntok = np.zeros(ws.num_ctas)
t0 = T[:, 1].min()
rel = (T[:, 1:5] - t0) / 1e3
seg_end = (T[:, 6] - t0) / 1e3
print(f"mode={mode} ctas={ws.num_ctas} span_us={(T[:,4].max()-t0)/1e3:.2f}")
for name, col in (("entry", 0), ("ready", 1), ("loop0_end", 2), ("exit", 3)):
    c = rel[:, col]
    print(f"{name:10s} min {c.min():7.2f} med {np.median(c):7.2f} max {c.max():7.2f} us")
print("nseg hist", np.bincount(T[:, 5]))
for name, col in (("post_wait", 7), ("lut_pre", 8), ("dense", 10), ("cv_ready", 9)):
    c = (T[:, col] - t0) / 1e3
    c = c[T[:, col] > 0]
    if len(c):
        print(f"{name:10s} min {c.min():7.2f} med {np.median(c):7.2f} max {c.max():7.2f} us")
print(f"segs_done  min {seg_end.min():7.2f} med {np.median(seg_end):7.2f} max {seg_end.max():7.2f} us")
for k in (1, 2):
    sel = T[:, 5] == k
    if sel.any():
        print(f"  nseg={k}: segs_done med {np.median(seg_end[sel]):7.2f} max {seg_end[sel].max():7.2f}"
              f"  exit med {np.median(rel[sel, 3]):7.2f} max {rel[sel, 3].max():7.2f}")
order = np.argsort(rel[:, 3])
print("slowest exits (cta, sm, nseg, entry, ready, loop0, segs_done, exit):")
for i in order[-8:]:
    print(i, T[i, 0], T[i, 5], *np.round(rel[i, :3], 2), round(seg_end[i], 2), round(rel[i, 3], 2))
print("fastest exits:")
for i in order[:8]:
    print(i, T[i, 0], T[i, 5], *np.round(rel[i], 2))
np.save(os.path.join(ROOT, "gpurun_out", "trace.npy"), T)
