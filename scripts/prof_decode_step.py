"""Diagnostic: host-side profile of decode_step (the reference-API per-token path) on a GPU box."""
import cProfile, pstats, sys, time
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2504_03661_b200 import harness as H
from paper_2504_03661_b200.attention import decode_step
from paper_2504_03661_b200.kv_cache import LayerKVCache
cfg = H.BenchConfig(context_lengths=[4096], gen_tokens=200)
cb_K, cb_V = H._codebooks(cfg, None)
K, V = H.synth_kv(H.SynthSpec(n_tokens=4096 + 400, d=128, seed=1))
cache = LayerKVCache(cb_K, cb_V, recent_capacity=32, flush_threshold=32, worker="thread")
cache.prefill_ingest(K[:4096], V[:4096]); cache.drain()
dev = torch.device("cuda")
q = torch.randn(400, 128, device=dev); kd = torch.from_numpy(K[4096:]).to(dev); vd = torch.from_numpy(V[4096:]).to(dev)
for i in range(100): decode_step(q[i], kd[i], vd[i], cache, cb_K, cb_V)
torch.cuda.synchronize()
pr = cProfile.Profile(); pr.enable()
t0 = time.perf_counter()
for i in range(100, 300): decode_step(q[i], kd[i], vd[i], cache, cb_K, cb_V)
torch.cuda.synchronize()
pr.disable()
print("per step ms", (time.perf_counter() - t0) / 200 * 1e3)
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
cache.close()
