"""Diagnostic: per-layer / per-CTA timeline of the decode kernel inside the
bench's graph-replayed 32-layer step (library built with -DPQKV_TRACE).
usage (GPU box): python scripts/trace_graph.py [bench flags...]"""
import ctypes, os, subprocess, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2504_03661_b200 import build as B
lib = os.environ.get("TRACE_LIB") or os.path.join(B.OUT_DIR, "libpqkv_sm100_trace.so")
if not os.environ.get("TRACE_LIB"):
    B.build(lib=lib, defines=("PQKV_TRACE",))  # rebuilt when older than the sources
os.environ["PQKV_SM100_LIB"] = lib
import torch
from paper_2504_03661_b200 import kernels as K, _native as N
from paper_2504_03661_b200.engine import PQDecoder, random_codes
from paper_2504_03661_b200.pq_core import PQConfig
dev = torch.device("cuda", 0)
L, Bb, Hq, Hkv, n, R = 32, 1, 32, 32, 32768, 31
g = torch.Generator(device=dev); g.manual_seed(0)
ck = [random_codes((Bb, Hkv, n, 64), 8, g, dev) for _ in range(L)]
cv = [random_codes((Bb, Hkv, n, 64), 8, g, dev) for _ in range(L)]
cb_all = torch.empty((L, 2, 64 * 256 * 2), device=dev)
cbk = [K.key_codebook_layout(torch.randn((64, 256, 2), generator=g, device=dev), 8, out=cb_all[l, 0]) for l in range(L)]
F16 = os.environ.get("F16") == "1"  # the fp16 value-codebook mode
cbv = [K.value_codebook_layout(torch.randn((64, 256, 2), generator=g, device=dev), 8, half=F16, out=None if F16 else cb_all[l, 1]) for l in range(L)]
q = torch.randn((L, Bb, Hq, 128), generator=g, device=dev)
rk = torch.randn((L, Bb, Hkv, R, 128), generator=g, device=dev); rv = torch.randn_like(rk)
kc = torch.randn((L, Bb, Hkv, 128), generator=g, device=dev); vc = torch.randn_like(kc)
nq = torch.full((Bb,), n, dtype=torch.int32, device=dev); nr = torch.full((Bb,), R, dtype=torch.int32, device=dev)
out = torch.empty((L, Bb, Hq, 128), device=dev)
torch.cuda.synchronize()
dec = PQDecoder(Bb, Hq, Hkv, PQConfig(128, 64, 8), device=dev, pdl=True, static_codebooks=os.environ.get("STATIC", "1") == "1", early_codes=os.environ.get("EARLY", "1") == "1")
st = torch.cuda.Stream()
if os.environ.get("L2_PERSIST") == "1":
    N.call("pqkv_l2_persist", N.ptr(cb_all), cb_all.numel() * 4, 1.0, N.stream_ptr(st))
    print("codebooks pinned in L2")
def step():
    for l in range(L):
        dec(q[l], ck[l], cv[l], nq, cbk[l], cbv[l], rk[l], rv[l], nr, kc[l], vc[l], out=out[l])
with torch.cuda.stream(st):
    step(); step()  # launches 0..63: the second step fills trace slots 32..63
if os.environ.get("GRAPH") == "1":  # replay a captured step (trace ids are baked in: 64..95 -> slots 0..31)
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr, stream=st):
        step()
    gr.replay(); gr.replay()
torch.cuda.synchronize()
T = np.zeros(64 * 256 * 32, dtype=np.uint64)
N.load().pqkv_debug_trace.argtypes = [ctypes.c_void_p, ctypes.c_int]
assert N.load().pqkv_debug_trace(T.ctypes.data, T.size) == 0
sl = slice(0, 32) if os.environ.get("GRAPH") == "1" else slice(32, 64)
T = T.reshape(64, 256, 32)[sl, :dec.ws.num_ctas].astype(np.int64)
t0 = T[0, :, 1].min()
rel = lambda c: (c - t0) / 1e3
print(f"{'layer':>5} {'first_in':>8} {'last_in':>8} {'post_wait':>9} {'ready_med':>9} {'ready_max':>9} "
      f"{'segs_med':>8} {'segs_max':>8} {'exit_min':>8} {'exit_max':>8}")
prev_exit = None
for l in range(32):
    x = T[l]
    print(f"{l:5d} {rel(x[:,1].min()):8.2f} {rel(x[:,1].max()):8.2f} {rel(np.median(x[:,7])):9.2f} "
          f"{rel(np.median(x[:,2])):9.2f} {rel(x[:,2].max()):9.2f} {rel(np.median(x[:,6])):8.2f} "
          f"{rel(x[:,6].max()):8.2f} {rel(x[:,4].min()):8.2f} {rel(x[:,4].max()):8.2f}")
span = (T[31, :, 4].max() - T[0, :, 1].min()) / 1e3
print(f"32 layers: {span:.1f} us -> {span/32:.2f} us/layer")
# average phase durations per CTA
ready = (T[:, :, 2] - T[:, :, 1]) / 1e3
loop = (T[:, :, 6] - T[:, :, 2]) / 1e3
fin = (T[:, :, 4] - T[:, :, 6]) / 1e3
for name, c in (("post_wait", 7),):
    v = np.median((T[4:, :, c] - T[4:, :, 7].min(axis=1, keepdims=True)) / 1e3)
    print(f"  {name:10s} median {v:6.2f} us after the layer's first post-wait (globaltimer)")
for name, c in (("ring_issued", 10), ("seg_ring", 11), ("sync1", 12), ("lut_built", 8),
                ("dense", 13), ("cv_ready", 9), ("loop_start", 16)):
    v = T[4:, :, c] / 1965.0
    print(f"  {name:10s} median {np.median(v):6.2f} us, p90 {np.percentile(v, 90):6.2f} us after the CTA's post-wait (clock64)")
print(f"per CTA (median over layers/CTAs): entry->ready {np.median(ready):.2f} us, ready->segs_done {np.median(loop):.2f} us, segs_done->exit {np.median(fin):.2f} us")
np.save(os.path.join(ROOT, "gpurun_out", "trace_graph.npy"), T)
# arrival / merge (clock64 cycles after segs_done, 1965 MHz), group 0's first segment
arr, fin = T[4:, :, 14] / 1965.0, T[4:, :, 15] / 1965.0
last = fin > 0
print(f"arrival after segs_done: median {np.median(arr):.2f} us, p90 {np.percentile(arr, 90):.2f}")
if last.any():
    print(f"last-arriver merge end after segs_done: median {np.median(fin[last]):.2f} us, "
          f"p90 {np.percentile(fin[last], 90):.2f}")
ex = T[4:, :, 4]
lc = ex.argmax(axis=1)
print("layer-last CTA: arrival %.2f us, merge end %.2f us (medians over layers)" % (
    np.median(arr[np.arange(len(lc)), lc]), np.median(fin[np.arange(len(lc)), lc])))
# per-warp main-loop end (first segment): spread within each CTA
Wt = np.zeros(64 * 256 * 32, dtype=np.uint64)
N.load().pqkv_debug_wtrace.argtypes = [ctypes.c_void_p, ctypes.c_int]
if N.load().pqkv_debug_wtrace(Wt.ctypes.data, Wt.size) == 0:
    Wt = Wt.reshape(64, 256, 32)[sl, :dec.ws.num_ctas, :16].astype(np.int64)
    nseg = T[:, :, 5]
    one = (nseg == 1)
    spread = (Wt.max(axis=2) - Wt.min(axis=2)) / 1e3
    order = np.argsort(np.median(((Wt - Wt.min(axis=2, keepdims=True)) / 1e3)[4:][one[4:]], axis=0))
    print(f"warp loop-end spread within a CTA (1-segment CTAs): median {np.median(spread[4:][one[4:]]):.2f} us, "
          f"p90 {np.percentile(spread[4:][one[4:]], 90):.2f} us")
    lag = np.median(((Wt - Wt.min(axis=2, keepdims=True)) / 1e3)[4:][one[4:]], axis=0)
    print("median lag per warp (us):", " ".join(f"{x:.2f}" for x in lag))
