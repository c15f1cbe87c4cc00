"""Diagnostic: per-step host time distribution of the reference-API decode loop
(harness.bench_decode's inner loop) at 1K and 32K contexts."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2504_03661_b200 import harness as H
from paper_2504_03661_b200.attention import Counters, decode_step
from paper_2504_03661_b200.kv_cache import LayerKVCache
NS = int(os.environ.get("STEPS", "100"))
cfg = H.BenchConfig(context_lengths=[1024, 32768], gen_tokens=NS)
cb_K, cb_V = H._codebooks(cfg, None)
dev = torch.device("cuda")
for ctx in (1024, 32768):
    K, V = H.synth_kv(H.SynthSpec(n_tokens=ctx + NS, d=128, seed=ctx))
    seed = LayerKVCache(cb_K, cb_V, worker="sync"); seed.prefill_ingest(K[:ctx], V[:ctx])
    snap = seed.snapshot()
    q = torch.randn(NS, 128, device=dev)
    kd = torch.from_numpy(np.ascontiguousarray(K[ctx:], np.float32)).to(dev)
    vd = torch.from_numpy(np.ascontiguousarray(V[ctx:], np.float32)).to(dev)
    for rep in range(3):
        cache = LayerKVCache(cb_K, cb_V, worker="thread"); cache.load_snapshot(snap)
        c = Counters(); torch.cuda.synchronize()
        ts = [time.perf_counter()]
        for i in range(NS):
            decode_step(q[i], kd[i], vd[i], cache, cb_K, cb_V, counters=c)
            ts.append(time.perf_counter())
        torch.cuda.synchronize(); tend = time.perf_counter()
        d = np.diff(ts) * 1e6
        print(f"ctx {ctx} rep {rep}: mean {d.mean():.1f} us, p50 {np.median(d):.1f}, p90 {np.percentile(d, 90):.1f}, "
              f"max {d.max():.1f} (step {d.argmax()}), first {d[0]:.1f}, drain {1e6 * (tend - ts[-1]):.1f} us")
        cache.close()
