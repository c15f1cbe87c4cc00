"""Diagnostic: decode_step per-token time (GPU-resident inputs) vs the fp16
SDPA loop at a few contexts, and the fused decode kernel's device time."""
import os, sys, time
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2504_03661_b200 import harness as H
from paper_2504_03661_b200.attention import decode_step
from paper_2504_03661_b200.kv_cache import LayerKVCache
cfg = H.BenchConfig(context_lengths=[1024, 32768], gen_tokens=100)
cb_K, cb_V = H._codebooks(cfg, None)
dev = torch.device("cuda")
for ctx in (1024, 32768):
    K, V = H.synth_kv(H.SynthSpec(n_tokens=ctx + 200, d=128, seed=1))
    cache = LayerKVCache(cb_K, cb_V, recent_capacity=32, flush_threshold=32, worker="thread")
    cache.prefill_ingest(K[:ctx], V[:ctx]); cache.drain()
    q = torch.randn(200, 128, device=dev); kd = torch.from_numpy(K[ctx:]).to(dev); vd = torch.from_numpy(V[ctx:]).to(dev)
    for i in range(50): decode_step(q[i], kd[i], vd[i], cache, cb_K, cb_V)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for i in range(50, 150): decode_step(q[i], kd[i], vd[i], cache, cb_K, cb_V)
    torch.cuda.synchronize()
    pq = (time.perf_counter() - t0) / 100 * 1e3
    with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
        for i in range(150, 170): decode_step(q[i], kd[i], vd[i], cache, cb_K, cb_V)
        torch.cuda.synchronize()
    cache.close()
    qf = np.random.default_rng(0).standard_normal((100, 128))
    H._fp_tpot_ms(K[:ctx + 100], V[:ctx + 100], qf, ctx, dev)  # warm-up (SDPA backend init)
    fp = H._fp_tpot_ms(K[:ctx + 100], V[:ctx + 100], qf, ctx, dev)
    print(f"ctx {ctx}: pq {pq:.3f} ms/step, fp {fp:.3f} ms/step")
    if os.environ.get("DS_BRIEF"):
        for e in prof.key_averages():
            if "decode_partials" in e.key:
                print(f"  decode kernel {e.device_time_total / max(1, e.count):.1f} us/launch ({e.count})")
    else:
        print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=8))
