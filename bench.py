"""Benchmark: PQ decode attention tokens/s at 32K context (BASELINE config 2).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config llama2-32k|llama3-gqa-32k|llama2-4k-1layer]

A step is one decode step of the whole model's attention over its PQ cache:
for each of the 32 layers, the fused quantized-span kernel over all heads
(key LUTs built in shared memory, code stream, online softmax, value
accumulation) and the dense recent-window merge + finalize -- 64 launches
captured in one CUDA graph.  Inputs are synthetic
(seeded uniform uint8 codes, N(0,1) codebooks / queries / recent rows) of the
named shape and are resident in HBM; the code stream (4.29 GB per step for
config 2) exceeds L2, so no flush is needed between steps.

Multi-GPU: one process per GPU (torchrun); each rank decodes its own
sequences (batch sharding, no data-path collective) -> weak scaling; the
reported value is the whole-job tokens/s, timed as the max over ranks.

``--impl reference`` times the reference algorithm's CPU implementation (the
C restatement in oracle/, all host cores) on the same config; rank 0 only.
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (layers, B per rank, Hq, Hkv, quantized ctx, recent rows)
    "llama2-32k": (32, 1, 32, 32, 32768, 31),
    "llama3-gqa-32k": (32, 16, 32, 8, 32768, 31),
    "llama2-4k-1layer": (1, 1, 32, 32, 4096, 31),
    # BASELINE config 4: 128K context, B=4, Llama-3-8B shape; under torchrun the
    # sequence is split across ranks (one all-gather of partial records per layer)
    "llama3-gqa-128k": (32, 4, 32, 8, 131072, 31),
}
SEQ_SPLIT = {"llama3-gqa-128k"}
# BASELINE config 3 is KV-head sharded under torchrun: rank r serves KV heads
# [r Hkv/N, (r+1) Hkv/N) (and their query heads) of every sequence -- no
# collective, total work fixed (strong scaling)
HEAD_SHARD = {"llama3-gqa-32k"}
D, M, NBITS = 128, 64, 8
METRIC = "decode attention tokens/s at 32K ctx (HBM GB/s of roofline); KV encode tok/s"
THROTTLE_BITS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
                 0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
                 0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
                 0x100: "display_clock_setting"}


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def ncu_traffic(cfg_name):
    """dram read+write bytes per launch of the decode kernel from a committed
    `ncu --set full` capture summary (profiles/*decode_ncu.json), else None."""
    pdir = os.path.join(ROOT, "profiles")
    best = None
    if os.path.isdir(pdir):
        for f in sorted(os.listdir(pdir)):
            if f.endswith("decode_ncu.json"):
                try:
                    with open(os.path.join(pdir, f)) as fh:
                        j = json.load(fh)
                    if j.get("config") == cfg_name:
                        best = j.get("dram_bytes_per_launch")
                except Exception:
                    pass
    return best


class ClockSampler:
    """SM clocks / throttle reasons sampled through NVML every few ms during the
    timed region (the recipe's clocks line); falls back to nvidia-smi."""

    def __init__(self, index: int, period_s: float = 0.005):
        self.index, self.period, self.samples = index, period_s, []
        self._stop = threading.Event()

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self._nv = (pynvml, h)
        except Exception:
            self._nv = None
        self.thread = threading.Thread(target=self._run, daemon=True)
        self.thread.start()
        return self

    def _run(self):
        while not self._stop.is_set():
            try:
                if self._nv is not None:
                    nv, h = self._nv
                    sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                    smx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
                    pw = nv.nvmlDeviceGetPowerUsage(h) / 1000.0
                    rs = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                else:
                    out = subprocess.run(
                        ["nvidia-smi", "-i", str(self.index), "--query-gpu=clocks.sm,clocks.max.sm,"
                         "power.draw,clocks_event_reasons.active", "--format=csv,noheader,nounits"],
                        capture_output=True, text=True, timeout=5).stdout.split(",")
                    sm, smx, pw, rs = float(out[0]), float(out[1]), float(out[2]), int(out[3], 16)
                self.samples.append((float(sm), float(smx), float(pw), int(rs)))
            except Exception:
                pass
            time.sleep(self.period)

    def __exit__(self, *a):
        self._stop.set()
        self.thread.join(timeout=5)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        busy = [s for s in self.samples if not (s[3] & 0x1)] or self.samples
        reasons = set()
        for s in busy:
            for bit, name in THROTTLE_BITS.items():
                if s[3] & bit and bit != 0x1:
                    reasons.add(name)
        return {"sm_mhz": statistics.median(s[0] for s in busy),
                "sm_max_mhz": max(s[1] for s in busy),
                "power_w_max": max(s[2] for s in busy),
                "samples": len(busy), "reasons": sorted(reasons)}


# ------------------------------------------------------------ CPU baseline --

def cpu_decode_rate(cfg_name, threads, budget_s, layers_per_rep=1, seed=0):
    """Time the C restatement of the reference decode (oracle/, fp64, numba-loop
    equivalent, block_size 8192 as harness.py:161) on `threads` host threads over
    a bounded sample of the workload; returns (tokens/s, sample description)."""
    from oracle import pqkv_oracle as O
    lib = O.c_library()
    if lib is None:
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle")], check=True)
        O._clib = None
        lib = O.c_library()
    L, B, Hq, Hkv, n, R = CONFIGS[cfg_name]
    G = Hq // Hkv
    heads = B * Hq
    rng = np.random.default_rng(seed)
    ck = rng.integers(0, 256, (B * Hkv, n, M), dtype=np.uint8)
    cv = rng.integers(0, 256, (B * Hkv, n, M), dtype=np.uint8)
    # GQA: q-head h reads KV head h // G; the C loop takes per-head strides, so
    # replicate pointers by laying q-heads out in KV-head-major order
    ck_h = ck if G == 1 else np.repeat(ck, G, axis=0)
    cv_h = cv if G == 1 else np.repeat(cv, G, axis=0)
    q = rng.standard_normal((heads, D))
    kn = rng.standard_normal((heads, D)).astype(np.float32)
    vn = rng.standard_normal((heads, D)).astype(np.float32)
    rk = rng.standard_normal((heads, R, D)).astype(np.float32)
    rv = rng.standard_normal((heads, R, D)).astype(np.float32)
    cents_k = rng.standard_normal((M, 256, 2)).astype(np.float32)
    cents_v = rng.standard_normal((M, 256, 2)).astype(np.float32)
    out = np.empty((heads, D))
    P = ctypes.c_void_p

    def one_layer():
        rc = lib.oracle_decode_heads_mt(
            q.ctypes.data_as(P), kn.ctypes.data_as(P), vn.ctypes.data_as(P),
            ck_h.ctypes.data_as(P), cv_h.ctypes.data_as(P), n, n, rk.ctypes.data_as(P),
            rv.ctypes.data_as(P), R, cents_k.ctypes.data_as(P), cents_v.ctypes.data_as(P),
            M, NBITS, 2, 1.0 / np.sqrt(D), 8192, out.ctypes.data_as(P), heads, threads)
        assert rc == 0

    one_layer()  # warm-up
    times = []
    t_start = time.perf_counter()
    while True:
        t0 = time.perf_counter()
        for _ in range(layers_per_rep):
            one_layer()
        times.append((time.perf_counter() - t0) / layers_per_rep)
        if time.perf_counter() - t_start > budget_s and len(times) >= 3:
            break
    per_layer = statistics.median(times)
    tok_s = B / (per_layer * L)
    sample = (f"{len(times)} reps x {layers_per_rep} layer(s) of {heads} heads x {n} ctx "
              f"(median {per_layer * 1e3:.1f} ms/layer, scaled x{L} layers)")
    return tok_s, sample


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    threads = len(os.sched_getaffinity(0))
    per_step = []
    sample = ""
    for _ in range(args.warmup):
        cpu_decode_rate(args.config, threads, 0.0)
    for _ in range(args.steps):
        v, sample = cpu_decode_rate(args.config, threads, 0.0)
        per_step.append(v)
    value = statistics.median(per_step)
    L, B, Hq, Hkv, n, R = CONFIGS[args.config]
    line = {"metric": METRIC, "impl": "reference", "value": value, "unit": "tokens/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * B / value, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": config_dict(args.config, args.gpus),
            "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": threads,
                             "kind": "port", "sample": sample},
            "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def config_dict(name, n_gpus):
    L, B, Hq, Hkv, n, R = CONFIGS[name]
    if name in HEAD_SHARD and n_gpus > 1:
        return {"workload": name, "layers": L, "batch_per_gpu": B, "global_batch": B,
                "q_heads": Hq, "kv_heads": Hkv, "q_heads_per_gpu": Hq // n_gpus,
                "kv_heads_per_gpu": Hkv // n_gpus, "head_dim": D, "ctx_quantized": n,
                "recent_rows": R, "pq": "m64b8 (M=64, nbits=8, dsub=2)",
                "code_bytes_per_step_per_gpu": 2 * L * B * (Hkv // n_gpus) * n * M,
                "parallelism": f"kv-head-sharded x{n_gpus} (no collective)",
                "l2": _l2_note(2 * L * B * Hkv * n * M // max(1, n_gpus))}
    if name in SEQ_SPLIT:
        return {"workload": name, "layers": L, "batch_per_gpu": B, "global_batch": B,
                "q_heads": Hq, "kv_heads": Hkv, "head_dim": D, "ctx_quantized": n,
                "recent_rows": R, "pq": "m64b8 (M=64, nbits=8, dsub=2)",
                "code_bytes_per_step_per_gpu": 2 * L * B * Hkv * (n // n_gpus) * M,
                "parallelism": f"sequence-split x{n_gpus} (NCCL all-gather of (m, l, acc) "
                               "records + rank-ordered LSE merge per layer)" if n_gpus > 1
                               else "single GPU (sequence split degenerates)",
                "l2": _l2_note(2 * L * B * Hkv * n * M // max(1, n_gpus))}
    return {"workload": name, "layers": L, "batch_per_gpu": B, "global_batch": B * n_gpus,
            "q_heads": Hq, "kv_heads": Hkv, "head_dim": D, "ctx_quantized": n,
            "recent_rows": R, "pq": "m64b8 (M=64, nbits=8, dsub=2)",
            "code_bytes_per_step_per_gpu": 2 * L * B * Hkv * n * M,
            "parallelism": f"batch-sharded x{n_gpus} (no collective)",
            "l2": _l2_note(2 * L * B * Hkv * n * M)}


def _l2_note(code_bytes: int) -> str:
    if code_bytes > 4 * 126 * 2 ** 20:
        return "inputs > L2 (code stream per step >> 126 MB); no flush needed"
    return ("code stream fits in L2 and is NOT flushed between steps: a latency / "
            "L2-resident figure, not an HBM-bandwidth one (parity configuration)")


# ------------------------------------------------------------------ ours --

def encode_rate(dev, L, Hkv, n, stream):
    """KV encode tok/s (BASELINE config 5): bit-exact nearest-centroid encoding
    of an n-token prefill -- K and V of every KV head of one layer, written
    straight into the decode layout -- timed with CUDA events; tokens/s is
    per model token (all L layers).  Bit-exact with the reference's fp64
    distances (fp32 filter + exact fp64 re-scan of near ties); 98,304 flop
    per vector by the reference's accounting."""
    import torch
    from paper_2504_03661_b200 import kernels as K
    g = torch.Generator(device=dev)
    g.manual_seed(7)
    x = torch.randn((2, Hkv * n, D), generator=g, device=dev)
    cents = torch.randn((2, M, 256, 2), generator=g, device=dev)
    codes = torch.empty((2, Hkv * n, M), dtype=torch.uint8, device=dev)

    def one():
        for kind in range(2):
            K.encode(x[kind], cents[kind], NBITS, out=codes[kind], stream=stream,
                     layout="decode")

    with torch.cuda.stream(stream):
        one()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 3
        e0.record(stream)
        for _ in range(reps):
            one()
        e1.record(stream)
        e1.synchronize()
    t_layer = e0.elapsed_time(e1) / reps * 1e-3
    vectors = 2 * Hkv * n
    # the filter scan's bound: per (vector, centroid pair) 4 packed f32x2 ops
    # (fma pipe) and 7 alu-pipe ops (2 key LOP3 + 5 integer min/max, one of
    # them three-input); the alu pipe retires 64 lanes/clk/SM vs 128 for the
    # fma pipe and issue (scripts/micro/fma_peak.cu): 64 / 3.5 = 18.3
    # candidates/clk/SM
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    cand = vectors * M * 256 / t_layer
    peak = sms * (64 / 3.5) * 1.965e9
    return {"value": n / (t_layer * L), "unit": "tokens/s (all layers, K+V, all KV heads)",
            "workload": f"{n}-token prefill x {Hkv} KV heads x K,V, one layer timed, x{L} layers",
            "ms_per_layer": t_layer * 1e3, "vectors_per_s": vectors / t_layer,
            "tflops_98304_per_vector": vectors * M * 256 * 6 / t_layer / 1e12, "bit_exact": True,
            "roofline": {"bound": "alu pipe (distance-key min/max)", "achieved": cand,
                         "peak": peak, "unit": "candidates/s (vector x centroid)",
                         "frac": cand / peak,
                         "peak_basis": "18.3 candidates/clk/SM (3.5 alu ops each) x SMs x "
                                       "1965 MHz; alu pipe 64 lanes/clk/SM measured "
                                       "(scripts/micro/fma_peak.cu)"}}


def append_overlap(dev, graph, stream, L, B, Hkv, warmup, R_f=32, rounds=3):
    """BASELINE config 5, second part: the per-token append path flushes a
    batch of R_f recent rows (K and V, every layer, sequence and KV head) into
    the code store every R_f decode steps, on a lowest-priority side stream
    (ServingCache(async_flush=True)).  Times R_f decode steps with and without
    one such flush running beside them; reports the slowdown."""
    import torch
    from paper_2504_03661_b200 import kernels as K
    g = torch.Generator(device=dev)
    g.manual_seed(11)
    rows = torch.randn((2, L, B * Hkv * R_f, D), generator=g, device=dev)  # [K|V][layer]
    cents = torch.randn((2, L, M, 256, 2), generator=g, device=dev)
    codes = torch.empty((2, L, B * Hkv * R_f, M), dtype=torch.uint8, device=dev)
    lo, _ = torch.cuda.Stream.priority_range()
    side = torch.cuda.Stream(device=dev, priority=lo)

    def flush():  # ServingCache._encode_all: one batched launch per kind over all layers
        with torch.cuda.stream(side):
            for kind in range(2):
                K.encode_batched(rows[kind], cents[kind], NBITS, out=codes[kind], stream=side,
                                 layout="decode")

    def window(with_flush):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(stream)
        if with_flush:
            side.wait_event(e0)
            flush()
        with torch.cuda.stream(stream):
            for _ in range(R_f):
                graph.replay()
        e1.record(stream)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1)

    for _ in range(max(1, warmup)):
        window(True)
    base = statistics.median(window(False) for _ in range(rounds))
    with_flush = statistics.median(window(True) for _ in range(rounds))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(side)
    flush()
    e1.record(side)
    torch.cuda.synchronize()
    return {"flush_batch": f"{R_f} rows x K,V x {L} layers x {B * Hkv} KV heads "
                           f"({2 * L * B * Hkv * R_f} vectors), every {R_f} steps",
            "flush_alone_ms": e0.elapsed_time(e1),
            "decode_ms_per_step": base / R_f, "decode_ms_per_step_with_flush": with_flush / R_f,
            "slowdown": with_flush / base - 1.0}


def run_ours(args):
    import torch
    import torch.distributed as dist

    rank, world, local = dist_env()
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    from paper_2504_03661_b200 import build as B_
    B_.build()
    from paper_2504_03661_b200 import kernels as K
    from paper_2504_03661_b200 import _native as N
    from paper_2504_03661_b200.engine import PQDecoder, random_codes
    from paper_2504_03661_b200.pq_core import PQConfig

    L, B, Hq, Hkv, n, R = CONFIGS[args.config]
    seq_split = args.config in SEQ_SPLIT and world > 1
    n_full = n
    if seq_split:  # this rank's contiguous token range of every sequence
        from paper_2504_03661_b200.engine import shard_tokens
        a_, b_ = shard_tokens(n_full, rank, world)
        n = b_ - a_
    tail = (not seq_split) or rank == world - 1  # owns the recent window + current token
    head_shard = args.config in HEAD_SHARD and world > 1
    if head_shard:
        if Hkv % world:
            raise SystemExit(f"{args.config}: {Hkv} KV heads do not shard over {world} GPUs")
        Hq, Hkv = Hq // world, Hkv // world
    cfg = PQConfig(D, M, NBITS)
    g = torch.Generator(device=dev)
    g.manual_seed(1234 + rank)
    codes_k = [random_codes((B, Hkv, n, M), NBITS, g, dev) for _ in range(L)]
    codes_v = [random_codes((B, Hkv, n, M), NBITS, g, dev) for _ in range(L)]
    # every layer's codebook layouts in one allocation (kept L2-resident below)
    cb_words = M * 256 * 2
    cb_all = torch.empty((L, 2, cb_words), device=dev)
    cbk = [K.key_codebook_layout(torch.randn((M, 256, 2), generator=g, device=dev), NBITS,
                                 out=cb_all[l, 0]) for l in range(L)]
    cv_raw = [torch.randn((M, 256, 2), generator=g, device=dev) for _ in range(L)]
    cbv32 = [K.value_codebook_layout(cv_raw[l], NBITS, out=cb_all[l, 1]) for l in range(L)]
    cbv16 = [K.value_codebook_layout(cv_raw[l], NBITS, half=True) for l in range(L)]
    cbv = cbv16 if args.f16_value_codebook else cbv32
    rk = torch.randn((L, B, Hkv, R, D), generator=g, device=dev)
    rv = torch.randn((L, B, Hkv, R, D), generator=g, device=dev)
    n_q = torch.full((B,), n, dtype=torch.int32, device=dev)
    n_r = torch.full((B,), R, dtype=torch.int32, device=dev)
    # one step's inputs (q, current k, current v of every layer) in one
    # allocation, so the end-to-end step moves them with a single copy
    nq_, nk_ = L * B * Hq * D, L * B * Hkv * D
    io = torch.randn(nq_ + 2 * nk_, generator=g, device=dev)
    q = io[:nq_].view(L, B, Hq, D)
    kc = io[nq_:nq_ + nk_].view(L, B, Hkv, D)
    vc = io[nq_ + nk_:].view(L, B, Hkv, D)
    out = torch.empty((L, B, Hq, D), device=dev)
    torch.cuda.synchronize()  # codebook layouts are written before any decode launch
    # one fused launch per layer; PDL lets layer l+1 load its value codebook
    # while layer l's last CTAs drain (codebooks are static: prepared above)
    # codebooks (load time) and codes below n_q (appended by earlier steps) are
    # not written by the kernel a launch overlaps: PDL may read them early
    dec = PQDecoder(B, Hq, Hkv, cfg, device=dev, pdl=not args.no_pdl,
                    static_codebooks=not args.no_pdl, early_codes=not args.no_pdl)
    stream = torch.cuda.Stream(device=dev)
    if not args.no_l2_persist:
        N.call("pqkv_l2_persist", N.ptr(cb_all), cb_all.numel() * 4, 1.0, N.stream_ptr(stream))

    rec = torch.empty((L, B * Hq, D + 4), device=dev) if seq_split else None
    gat = torch.empty((L, world, B * Hq, D + 4), device=dev) if seq_split else None

    def capture(cbv_l):
        """one decode step (one fused launch per layer) captured in a CUDA graph"""
        def step():
            for l in range(L):
                if seq_split:
                    # partial record of this rank's token range -> all-gather ->
                    # merge in rank order (engine.sequence_parallel_decode)
                    dec(q[l], codes_k[l], codes_v[l], n_q, cbk[l], cbv_l[l],
                        rk[l] if tail else None, rv[l] if tail else None,
                        n_r if tail else None, kc[l] if tail else None,
                        vc[l] if tail else None, merged=rec[l], finalize=False)
                    dist.all_gather_into_tensor(gat[l], rec[l])
                    K.merge_partials(gat[l], out=out[l])
                else:
                    dec(q[l], codes_k[l], codes_v[l], n_q, cbk[l], cbv_l[l], rk[l], rv[l], n_r,
                        kc[l], vc[l], out=out[l])
        with torch.cuda.stream(stream):
            step()
            step()
        torch.cuda.synchronize()
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr, stream=stream):
            step()
        return gr

    graph = capture(cbv)
    launches_per_step = L

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # ---- device-resident timed region ------------------------------------
    for _ in range(args.warmup):
        graph.replay()
    barrier()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        with torch.cuda.stream(stream):
            ev0.record(stream)
            for _ in range(args.steps):
                graph.replay()
            ev1.record(stream)
        barrier()
    ms = max_over_ranks(ev0.elapsed_time(ev1) / args.steps)
    # ranks serve independent sequences unless they split them (by tokens or heads)
    jobs = 1 if (seq_split or head_shard) else world
    value = jobs * B * 1e3 / ms
    clocks = clk.summary()

    # ---- dominant kernel: per-launch CUDA-event time on its own stream ------
    kev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(L)]
    ktimes = []
    with torch.cuda.stream(stream):
        for rep in range(max(2, min(args.steps, 5))):
            for l in range(L):
                kev[l][0].record(stream)
                K.decode_attention(dec.ws, Hkv, q[l].view(B * Hq, D), 1 / D ** 0.5, cbk[l],
                                   codes_k[l], codes_v[l], n_q, cbv[l], rk[l], rv[l], n_r, kc[l],
                                   vc[l], out=out[l], stream=stream)
                kev[l][1].record(stream)
            stream.synchronize()
            if rep > 0:
                ktimes += [a.elapsed_time(b) for a, b in kev]
    iso_ms = statistics.mean(ktimes)
    # the timed step is L back-to-back launches of this kernel and nothing
    # else (PDL-overlapped), so its average in-step launch duration is ms / L
    k_ms = ms / L
    bytes_per_launch = 2 * B * Hkv * n * M
    hbm_peak, peak_kind = peaks()
    achieved = bytes_per_launch / (k_ms * 1e-3) / 1e9
    share = 1.0

    # ---- end to end through the public API with host buffers --------------
    io_h = torch.randn(io.numel()).pin_memory()  # q, k_cur, v_cur of every layer
    o_h = torch.empty((L, B, Hq, D)).pin_memory()
    h2d = io_h.numel() * 4
    d2h = o_h.numel() * 4

    def e2e_serial():
        io.copy_(io_h, non_blocking=True)
        graph.replay()
        o_h.copy_(out, non_blocking=True)

    def capture_e2e(split=4, tail=4):
        """The same step with its host copies inside the graph, pipelined: the
        first `split` layers' inputs on the launch stream, the rest on a copy
        stream behind them (joined before layer `split`), and the outputs of
        all but the last `tail` layers read back on the copy stream while
        those run.  Every copy stays inside the timed step."""
        cs = torch.cuda.Stream(device=dev)
        qh, kh = io_h[:nq_].view(L, B, Hq, D), io_h[nq_:nq_ + nk_].view(L, B, Hkv, D)
        vh = io_h[nq_ + nk_:].view(L, B, Hkv, D)

        def body():
            for dst, src in ((q, qh), (kc, kh), (vc, vh)):
                dst[:split].copy_(src[:split], non_blocking=True)
            e_fork = torch.cuda.Event()
            e_fork.record(stream)
            cs.wait_event(e_fork)
            with torch.cuda.stream(cs):
                for dst, src in ((q, qh), (kc, kh), (vc, vh)):
                    dst[split:].copy_(src[split:], non_blocking=True)
                e_in = torch.cuda.Event()
                e_in.record(cs)
            e_back = None
            for l in range(L):
                if l == split:
                    stream.wait_event(e_in)
                dec(q[l], codes_k[l], codes_v[l], n_q, cbk[l], cbv[l], rk[l], rv[l], n_r,
                    kc[l], vc[l], out=out[l])
                if l == L - tail - 1:
                    e_mid = torch.cuda.Event()
                    e_mid.record(stream)
                    cs.wait_event(e_mid)
                    with torch.cuda.stream(cs):
                        o_h[:L - tail].copy_(out[:L - tail], non_blocking=True)
                        e_back = torch.cuda.Event()
                        e_back.record(cs)
            o_h[L - tail:].copy_(out[L - tail:], non_blocking=True)
            stream.wait_event(e_back)

        with torch.cuda.stream(stream):
            body()
        torch.cuda.synchronize()
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr, stream=stream):
            body()
        return gr

    e2e_mode = "serial copies around the step graph"
    e2e_step = e2e_serial
    if not seq_split and not args.e2e_serial and L > 8:
        with torch.cuda.stream(stream):
            e2e_serial()
        torch.cuda.synchronize()
        o_ref = o_h.clone()
        g_e2e = capture_e2e()
        with torch.cuda.stream(stream):
            g_e2e.replay()
        torch.cuda.synchronize()
        if not torch.equal(o_h, o_ref):
            raise RuntimeError("pipelined end-to-end step disagrees with the serial one")
        e2e_step = g_e2e.replay
        e2e_mode = "copies pipelined inside the step graph (inputs of layers >= 4 behind " \
                   "layers 0-3, outputs of layers < L-4 behind the last 4)"

    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            e2e_step()
    barrier()
    with torch.cuda.stream(stream):
        ev0.record(stream)
        for _ in range(args.steps):
            e2e_step()
            ev1.record(stream)
            ev1.synchronize()  # the host reads each step's result
        e2e_ms = max_over_ranks(ev0.elapsed_time(ev1) / args.steps)
    barrier()

    # ---- the fp16 value-codebook mode (stated tolerance), same step -------
    f16 = None
    if not args.f16_value_codebook and not args.no_f16_mode:
        g16 = capture(cbv16)
        for _ in range(args.warmup):
            g16.replay()
        barrier()
        with torch.cuda.stream(stream):
            ev0.record(stream)
            for _ in range(args.steps):
                g16.replay()
            ev1.record(stream)
        barrier()
        ms16 = max_over_ranks(ev0.elapsed_time(ev1) / args.steps)
        f16 = {"value": jobs * B * 1e3 / ms16, "unit": "tokens/s", "ms_per_step": ms16,
               "roofline_frac": bytes_per_launch / (ms16 / L * 1e-3) / 1e9 / hbm_peak,
               "tolerance": "rtol 2e-3, atol 2e-4 vs the fp64 reference "
                            "(tests/test_gpu_parity.py::test_f16_value_codebook_mode)"}
        del g16

    enc = None if args.no_encode else encode_rate(dev, L, Hkv, n, stream)
    if enc is not None:
        enc["append_overlap"] = append_overlap(dev, graph, stream, L, B, Hkv, args.warmup)

    line = {"metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True,
            "scaling": "strong" if (seq_split or head_shard) else "weak",
            "vs_baseline": None,
            "dtype": "u8 codes / f32 accumulate" + (" (f16 value codebook)" if args.f16_value_codebook else ""), "data": "synthetic (seeded uniform codes, "
            "N(0,1) codebooks, queries and recent rows)",
            "config": config_dict(args.config, world),
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                         "frac": achieved / hbm_peak, "peak_kind": peak_kind,
                         "frac_of_nominal_8000_gbs": achieved / 8000.0,
                         "traffic": ncu_traffic(args.config),
                         "kernel": "decode_partials_m64b8 (fused pqkv_decode_attention)",
                         "kernel_ms_per_launch": k_ms,
                         "kernel_ms_isolated_launch": iso_ms,
                         "algorithmic_bytes_per_launch": bytes_per_launch,
                         "kernel_share_of_step": share},
            "e2e": {"value": jobs * B * 1e3 / e2e_ms, "unit": "tokens/s",
                    "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "api": "paper_2504_03661_b200.engine.PQDecoder (graph-replayed step)",
                    "copies": e2e_mode},
            "gpu_launches": launches_per_step * args.steps,
            "clocks": clocks,
            "code_stream_gbs_step": 2 * L * B * Hkv * n * M / (ms * 1e-3) / 1e9}
    if enc is not None:
        line["encode"] = enc
    if f16 is not None:
        line["f16_value_codebook_mode"] = f16
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        v, sample = cpu_decode_rate(args.config, 1, args.cpu_budget)
        line["cpu_baseline"] = {"value": v, "unit": "tokens/s", "cores": 1, "kind": "port",
                                "sample": sample}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="llama2-32k", choices=sorted(CONFIGS))
    ap.add_argument("--cpu-budget", type=float, default=10.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-pdl", action="store_true")
    ap.add_argument("--e2e-serial", action="store_true",
                    help="end-to-end copies before / after the step graph, not pipelined")
    ap.add_argument("--no-encode", action="store_true")
    ap.add_argument("--no-l2-persist", action="store_true",
                    help="do not pin the codebooks in L2 (persisting access-policy window)")
    ap.add_argument("--f16-value-codebook", action="store_true",
                    help="headline in the fp16 value-codebook mode (stated tolerance, DESIGN.md)")
    ap.add_argument("--no-f16-mode", action="store_true",
                    help="skip the secondary fp16 value-codebook measurement")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
