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
    # config 4 also reported on the MHA 32/32 shape (Llama-2-7B)
    "llama2-mha-128k": (32, 4, 32, 32, 131072, 31),
}
SEQ_SPLIT = {"llama3-gqa-128k", "llama2-mha-128k"}
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


def ncu_capture(cfg_name):
    """The committed `ncu --set full` capture record of this config's decode
    kernel (profiles/*decode_ncu.json: dram bytes per launch, kernel name,
    shared-load wavefronts per KV token), else {}."""
    pdir = os.path.join(ROOT, "profiles")
    best = {}
    if os.path.isdir(pdir):
        for f in sorted(os.listdir(pdir)):
            if f.endswith("decode_ncu.json"):
                try:
                    with open(os.path.join(pdir, f)) as fh:
                        j = json.load(fh)
                    if j.get("config") == cfg_name:
                        best = j
                except Exception:
                    pass
    return best


def kernel_label(cfg_name, f16_values=False):
    """The decode kernel pqkv_decode_attention dispatches for this config's
    headline mode (decode.cu, pqkv_decode_attention)."""
    _L, _B, Hq, Hkv, _n, _R = CONFIGS[cfg_name]
    group = Hq // Hkv
    if group % 4 == 0 and not f16_values:
        return "decode_gqa_pair (exact fp32 path, clusters of two CTAs)"
    if group % 2 == 0 and f16_values:
        return "decode_partials_m64b8 (two query heads per CTA, fp16 value codebook)"
    return "decode_partials_m64b8 (fused pqkv_decode_attention)"


def ncu_traffic(cfg_name):
    """dram read+write bytes per launch of the decode kernel (ncu_capture), else None."""
    return ncu_capture(cfg_name).get("dram_bytes_per_launch")


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
    # the candidate grids are built once per codebook (load time), like the
    # decode layouts: outside the timed region
    grids = [K.encode_grid(cents[kind], NBITS, stream=stream) for kind in range(2)]

    def one(use_grid=True):
        for kind in range(2):
            K.encode(x[kind], cents[kind], NBITS, out=codes[kind], stream=stream,
                     layout="decode", grid=grids[kind] if use_grid else None)

    def timed(use_grid):
        with torch.cuda.stream(stream):
            one(use_grid)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            reps = 3
            e0.record(stream)
            for _ in range(reps):
                one(use_grid)
            e1.record(stream)
            e1.synchronize()
        return e0.elapsed_time(e1) / reps * 1e-3

    t_full = timed(False)
    t_layer = timed(True)
    vectors = 2 * Hkv * n
    # the filter scan's bound: per (vector, centroid pair) 4 packed f32x2 ops
    # (fma pipe) and 7 alu-pipe ops (2 key LOP3 + 5 integer min/max, one of
    # them three-input); the alu pipe retires 64 lanes/clk/SM vs 128 for the
    # fma pipe and issue (scripts/micro/fma_peak.cu): 64 / 3.5 = 18.3
    # candidates/clk/SM
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    cand = vectors * M * 256 / t_full
    peak = sms * (64 / 3.5) * 1.965e9
    # the grid path reads each row once (fp32, 512 B) and writes its 64 code
    # bytes: an HBM roofline
    hbm = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))).get("hbm_gbs") \
        if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else None
    gbs = vectors * (D * 4 + M) / t_layer / 1e9
    return {"value": n / (t_layer * L), "unit": "tokens/s (all layers, K+V, all KV heads)",
            "workload": f"{n}-token prefill x {Hkv} KV heads x K,V, one layer timed, x{L} layers",
            "kernel": "encode_dsub2_grid (candidate grid per subspace, fp32 filter, exact "
                      "fp64 re-scan of near ties)",
            "ms_per_layer": t_layer * 1e3, "vectors_per_s": vectors / t_layer,
            "bit_exact": True,
            "roofline": {"bound": "hbm", "achieved": gbs, "peak": hbm, "unit": "GB/s",
                         "frac": gbs / hbm if hbm else None,
                         "traffic_basis": "per vector: 512 B of fp32 input + 64 B of codes"},
            "full_scan": {"value": n / (t_full * L), "ms_per_layer": t_full * 1e3,
                          "vectors_per_s": vectors / t_full,
                          "kernel": "encode_dsub2_filter (every centroid)",
                          "roofline": {"bound": "alu pipe (distance-key min/max)",
                                       "achieved": cand, "peak": peak,
                                       "unit": "candidates/s (vector x centroid)",
                                       "frac": cand / peak,
                                       "peak_basis": "18.3 candidates/clk/SM (3.5 alu ops "
                                                     "each) x SMs x 1965 MHz (alu pipe 64 "
                                                     "lanes/clk/SM, scripts/micro/fma_peak.cu)"}}}


def append_overlap(dev, replay, stream, L, B, Hkv, warmup, R_f=32, rounds=3):
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
                replay()
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


def shard_plan(name, rank, world, force_split=False):
    """This rank's share of config `name` on `world` GPUs:
    batch sharding (each rank its own sequences, no collective, weak scaling);
    KV-head sharding for config 3 (rank r serves KV heads [r Hkv/N, (r+1) Hkv/N)
    and their query heads of every sequence, no collective, strong scaling);
    sequence split for config 4 (rank r owns tokens [r n/N, (r+1) n/N) of every
    sequence, the last rank the recent window + current token; one NCCL
    all-gather of (m, l, acc) records + a rank-ordered merge per layer)."""
    L, B, Hq, Hkv, n, R = CONFIGS[name]
    plan = {"workload": name, "rank": rank, "world": world, "L": L, "B": B, "Hq": Hq,
            "Hkv": Hkv, "n": n, "R": R, "tok": [0, n], "kv_heads": [0, Hkv], "tail": True,
            "mode": "batch", "jobs": world}
    if (world > 1 or force_split) and name in SEQ_SPLIT:
        from paper_2504_03661_b200.engine import shard_tokens
        a, b = shard_tokens(n, rank, world)
        plan.update(mode="sequence", n=b - a, tok=[a, b], tail=rank == world - 1, jobs=1)
    elif world > 1 and name in HEAD_SHARD:
        if Hkv % world:
            raise SystemExit(f"{name}: {Hkv} KV heads do not shard over {world} GPUs")
        k = Hkv // world
        plan.update(mode="kv-head", Hq=Hq // world, Hkv=k, kv_heads=[rank * k, (rank + 1) * k],
                    jobs=1)
    return plan


class Workload:
    """One rank's synthetic inputs of a config (HBM-resident) and its decode
    step -- one fused launch per layer, PDL-chained, captured in a CUDA graph."""

    def __init__(self, args, plan, dev, stream, dist_on):
        import torch
        from paper_2504_03661_b200 import kernels as K
        from paper_2504_03661_b200 import _native as N
        from paper_2504_03661_b200.engine import PQDecoder, random_codes
        from paper_2504_03661_b200.pq_core import PQConfig
        self.plan, self.dev, self.stream, self.dist_on = plan, dev, stream, dist_on
        L, B, Hq, Hkv, n, R = (plan[k] for k in ("L", "B", "Hq", "Hkv", "n", "R"))
        self.L, self.B, self.Hq, self.Hkv, self.n, self.R = L, B, Hq, Hkv, n, R
        self.seq_split = plan["mode"] == "sequence"
        self.tail = plan["tail"]
        g = torch.Generator(device=dev)
        g.manual_seed(1234 + plan["rank"])
        self.codes_k = [random_codes((B, Hkv, n, M), NBITS, g, dev) for _ in range(L)]
        self.codes_v = [random_codes((B, Hkv, n, M), NBITS, g, dev) for _ in range(L)]
        # every layer's codebook layouts in one allocation (kept L2-resident)
        cb_words = M * 256 * 2
        self.cb_all = torch.empty((L, 2, cb_words), device=dev)
        self.cbk = [K.key_codebook_layout(torch.randn((M, 256, 2), generator=g, device=dev),
                                          NBITS, out=self.cb_all[l, 0]) for l in range(L)]
        cv_raw = [torch.randn((M, 256, 2), generator=g, device=dev) for _ in range(L)]
        self.cbv32 = [K.value_codebook_layout(cv_raw[l], NBITS, out=self.cb_all[l, 1])
                      for l in range(L)]
        self.cbv16 = [K.value_codebook_layout(cv_raw[l], NBITS, half=True) for l in range(L)]
        self.rk = torch.randn((L, B, Hkv, R, D), generator=g, device=dev)
        self.rv = torch.randn((L, B, Hkv, R, D), generator=g, device=dev)
        self.n_q = torch.full((B,), n, dtype=torch.int32, device=dev)
        self.n_r = torch.full((B,), R, dtype=torch.int32, device=dev)
        # one step's inputs (q, current k, current v of every layer) in one
        # allocation, so the end-to-end step moves them with a single copy
        self.nq_, self.nk_ = L * B * Hq * D, L * B * Hkv * D
        self.io = torch.randn(self.nq_ + 2 * self.nk_, generator=g, device=dev)
        self.q = self.io[:self.nq_].view(L, B, Hq, D)
        self.kc = self.io[self.nq_:self.nq_ + self.nk_].view(L, B, Hkv, D)
        self.vc = self.io[self.nq_ + self.nk_:].view(L, B, Hkv, D)
        self.out = torch.empty((L, B, Hq, D), device=dev)
        torch.cuda.synchronize()  # codebook layouts are written before any decode launch
        # codebooks (load time) and codes below n_q (appended by earlier steps)
        # are not written by the kernel a launch overlaps: PDL may read them
        # early (n_q itself is re-validated after the wait)
        self.dec = PQDecoder(B, Hq, Hkv, PQConfig(D, M, NBITS), device=dev,
                             num_ctas=int(os.environ.get("PQKV_BENCH_CTAS", "0")) or None,
                             pdl=not args.no_pdl, static_codebooks=not args.no_pdl,
                             early_codes=not args.no_pdl)
        if not args.no_l2_persist:
            N.call("pqkv_l2_persist", N.ptr(self.cb_all), self.cb_all.numel() * 4, 1.0,
                   N.stream_ptr(stream))
        self.rec = torch.empty((L, B * Hq, D + 4), device=dev) if self.seq_split else None
        self.gat = (torch.empty((L, plan["world"], B * Hq, D + 4), device=dev)
                    if self.seq_split else None)
        self.bytes_per_launch = 2 * B * Hkv * n * M
        self.graph_mode = "cuda graph"

    def layer(self, l, cbv):
        import torch.distributed as dist
        from paper_2504_03661_b200 import kernels as K
        if self.seq_split:
            # partial record of this rank's token range -> all-gather -> merge
            # in rank order (engine.sequence_parallel_decode)
            t = self.tail
            self.dec(self.q[l], self.codes_k[l], self.codes_v[l], self.n_q, self.cbk[l], cbv[l],
                     self.rk[l] if t else None, self.rv[l] if t else None,
                     self.n_r if t else None, self.kc[l] if t else None,
                     self.vc[l] if t else None, merged=self.rec[l], finalize=False)
            dist.all_gather_into_tensor(self.gat[l], self.rec[l])
            K.merge_partials(self.gat[l], out=self.out[l])
        else:
            self.dec(self.q[l], self.codes_k[l], self.codes_v[l], self.n_q, self.cbk[l], cbv[l],
                     self.rk[l], self.rv[l], self.n_r, self.kc[l], self.vc[l], out=self.out[l])

    def step_fn(self, half=False, keys16=False, pairs=False):
        cbv = self.cbv16 if half else self.cbv32
        self.dec.f16_key_table = keys16  # baked into the captured launches
        self.dec.key_table_pairs = pairs

        def step():
            for l in range(self.L):
                self.layer(l, cbv)
        return step

    def capture(self, half=False, keys16=False, pairs=False):
        """the step captured in a CUDA graph (replay); if capturing the NCCL
        all-gather of a sequence split fails, the step runs eagerly"""
        import torch
        step = self.step_fn(half, keys16, pairs)
        with torch.cuda.stream(self.stream):
            step()
            step()
        torch.cuda.synchronize()
        try:
            gr = torch.cuda.CUDAGraph()
            with torch.cuda.graph(gr, stream=self.stream):
                step()
            return gr.replay
        except Exception as e:  # noqa: BLE001 -- recorded in the JSON line
            if not self.seq_split:
                raise
            torch.cuda.synchronize()
            self.graph_mode = f"eager (graph capture of the all-gather failed: {e!s:.80})"

            def eager():
                with torch.cuda.stream(self.stream):
                    step()
            return eager

    def time(self, fn, steps, warmup, barrier, max_over_ranks):
        import torch
        for _ in range(warmup):
            fn()
        barrier()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(self.stream):
            ev0.record(self.stream)
            for _ in range(steps):
                fn()
            ev1.record(self.stream)
        barrier()
        return max_over_ranks(ev0.elapsed_time(ev1) / steps)


def merge_share(w, steps, barrier, max_over_ranks):
    """Sequence split: device time of the per-layer all-gather + merge alone
    (the step's exchange), captured like the step."""
    import torch
    import torch.distributed as dist
    from paper_2504_03661_b200 import kernels as K

    def ex():
        for l in range(w.L):
            dist.all_gather_into_tensor(w.gat[l], w.rec[l])
            K.merge_partials(w.gat[l], out=w.out[l])
    try:
        with torch.cuda.stream(w.stream):
            ex()
        torch.cuda.synchronize()
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr, stream=w.stream):
            ex()
        fn = gr.replay
    except Exception:  # noqa: BLE001
        torch.cuda.synchronize()

        def fn():
            with torch.cuda.stream(w.stream):
                ex()
    return w.time(fn, steps, 2, barrier, max_over_ranks)


def encode_sample_check(dev, stream, n=2048):
    """bit_exact, measured: a sample of the bench encoder's output against the
    C restatement of assign_codes (oracle/, test infrastructure)."""
    import torch
    from oracle import pqkv_oracle as O
    from paper_2504_03661_b200 import kernels as K
    if O.c_library() is None:
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle")], check=True)
        O._clib = None
    g = torch.Generator(device=dev)
    g.manual_seed(7)
    x = torch.randn((n, D), generator=g, device=dev)
    cents = torch.randn((M, 256, 2), generator=g, device=dev)
    with torch.cuda.stream(stream):
        codes = K.encode(x, cents, NBITS, stream=stream)
        codes_g = K.encode(x, cents, NBITS, stream=stream,
                           grid=K.encode_grid(cents, NBITS, stream=stream))
    stream.synchronize()
    want = O.c_assign_codes(x.cpu().numpy(), cents.cpu().numpy(), NBITS,
                            threads=len(os.sched_getaffinity(0)))
    return bool(np.array_equal(codes.cpu().numpy(), want)
                and np.array_equal(codes_g.cpu().numpy(), want)), n


def run_ours(args):
    import torch
    import torch.distributed as dist

    rank, world, local = dist_env()
    if world != args.gpus:
        raise SystemExit(f"bench.py: WORLD_SIZE={world} but --gpus {args.gpus}")
    if torch.cuda.device_count() < (local + 1):
        raise SystemExit(f"bench.py: rank {rank} needs GPU {local}; "
                         f"{torch.cuda.device_count()} visible")
    force_split = args.seq_split_one and world == 1 and args.config in SEQ_SPLIT
    if world > 1 or force_split:
        if force_split:  # a one-rank NCCL group: the split path's capture and merge on 1 GPU
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", str(29500 + os.getpid() % 1000))
            os.environ.setdefault("RANK", "0")
            os.environ.setdefault("WORLD_SIZE", "1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    from paper_2504_03661_b200 import build as B_
    B_.build()
    from paper_2504_03661_b200 import kernels as K

    stream = torch.cuda.Stream(device=dev)

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

    plan = shard_plan(args.config, rank, world, force_split)
    w = Workload(args, plan, dev, stream, world > 1 or force_split)
    L, B, Hq, Hkv, n = w.L, w.B, w.Hq, w.Hkv, w.n
    seq_split = w.seq_split
    jobs = plan["jobs"]
    replay = w.capture(args.f16_value_codebook)
    launches_per_step = L

    # ---- device-resident timed region ------------------------------------
    for _ in range(args.warmup):
        replay()
    barrier()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        with torch.cuda.stream(stream):
            ev0.record(stream)
            for _ in range(args.steps):
                replay()
            ev1.record(stream)
        barrier()
    ms = max_over_ranks(ev0.elapsed_time(ev1) / args.steps)
    value = jobs * B * 1e3 / ms
    clocks = clk.summary()

    # ---- dominant kernel: per-launch CUDA-event time on its own stream ------
    kev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(L)]
    ktimes = []
    cbv = w.cbv16 if args.f16_value_codebook else w.cbv32
    with torch.cuda.stream(stream):
        for rep in range(max(2, min(args.steps, 5))):
            for l in range(L):
                kev[l][0].record(stream)
                K.decode_attention(w.dec.ws, Hkv, w.q[l].view(B * Hq, D), 1 / D ** 0.5,
                                   w.cbk[l], w.codes_k[l], w.codes_v[l], w.n_q, cbv[l],
                                   w.rk[l], w.rv[l], w.n_r, w.kc[l], w.vc[l], out=w.out[l],
                                   stream=stream)
                kev[l][1].record(stream)
            stream.synchronize()
            if rep > 0:
                ktimes += [a.elapsed_time(b) for a, b in kev]
    iso_ms = statistics.mean(ktimes)
    merge_ms = merge_share(w, args.steps, barrier, max_over_ranks) if seq_split else 0.0
    # the timed step is L back-to-back launches of this kernel (plus, for a
    # sequence split, the all-gather + merge, timed separately)
    k_ms = (ms - merge_ms) / L
    bytes_per_launch = w.bytes_per_launch
    hbm_peak, peak_kind = peaks()
    achieved = bytes_per_launch / (k_ms * 1e-3) / 1e9
    share = (ms - merge_ms) / ms

    # ---- end to end through the public API with host buffers --------------
    io_h = torch.randn(w.io.numel()).pin_memory()  # q, k_cur, v_cur of every layer
    o_h = torch.empty((L, B, Hq, D)).pin_memory()
    h2d = io_h.numel() * 4
    d2h = o_h.numel() * 4

    def e2e_serial():
        w.io.copy_(io_h, non_blocking=True)
        replay()
        o_h.copy_(w.out, non_blocking=True)

    def capture_e2e(split=4, tail=4):
        """The same step with its host copies inside the graph, pipelined: the
        first `split` layers' inputs on the launch stream, the rest on a copy
        stream behind them (joined before layer `split`), and the outputs of
        all but the last `tail` layers read back on the copy stream while
        those run.  Every copy stays inside the timed step."""
        cs = torch.cuda.Stream(device=dev)
        nq_, nk_ = w.nq_, w.nk_
        qh, kh = io_h[:nq_].view(L, B, Hq, D), io_h[nq_:nq_ + nk_].view(L, B, Hkv, D)
        vh = io_h[nq_ + nk_:].view(L, B, Hkv, D)

        def body():
            for dst, src in ((w.q, qh), (w.kc, kh), (w.vc, vh)):
                dst[:split].copy_(src[:split], non_blocking=True)
            e_fork = torch.cuda.Event()
            e_fork.record(stream)
            cs.wait_event(e_fork)
            with torch.cuda.stream(cs):
                for dst, src in ((w.q, qh), (w.kc, kh), (w.vc, vh)):
                    dst[split:].copy_(src[split:], non_blocking=True)
                e_in = torch.cuda.Event()
                e_in.record(cs)
            e_back = None
            for l in range(L):
                if l == split:
                    stream.wait_event(e_in)
                w.layer(l, cbv)
                if l == L - tail - 1:
                    e_mid = torch.cuda.Event()
                    e_mid.record(stream)
                    cs.wait_event(e_mid)
                    with torch.cuda.stream(cs):
                        o_h[:L - tail].copy_(w.out[:L - tail], non_blocking=True)
                        e_back = torch.cuda.Event()
                        e_back.record(cs)
            o_h[L - tail:].copy_(w.out[L - tail:], non_blocking=True)
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
        r16 = w.capture(True)
        ms16 = w.time(r16, args.steps, args.warmup, barrier, max_over_ranks)
        f16 = {"value": jobs * B * 1e3 / ms16, "unit": "tokens/s", "ms_per_step": ms16,
               "roofline_frac": bytes_per_launch / ((ms16 - merge_ms) / L * 1e-3) / 1e9
               / hbm_peak,
               "tolerance": "rtol 2e-3, atol 2e-4 vs the fp64 reference "
                            "(tests/test_gpu_parity.py::test_f16_value_codebook_mode, "
                            "tests/test_gpu_full_shapes.py)"}
        del r16
        if Hq // Hkv >= 2 and (Hq // Hkv) % 2 == 0:
            # GQA: + the query heads of a CTA (four for groups of 4) share one packed fp16 key table
            r16k = w.capture(True, keys16=True)
            ms16k = w.time(r16k, args.steps, args.warmup, barrier, max_over_ranks)
            f16["f16_key_table"] = {
                "value": jobs * B * 1e3 / ms16k, "unit": "tokens/s", "ms_per_step": ms16k,
                "roofline_frac": bytes_per_launch / ((ms16k - merge_ms) / L * 1e-3) / 1e9
                / hbm_peak,
                "tolerance": "rtol 2e-3, atol 2e-4 vs the fp64 reference "
                             "(tests/test_gpu_gqa_tables.py)"}
            del r16k
            if (Hq // Hkv) % 4 == 0:
                # the same with two query heads per CTA (one half2 table per pair)
                r16p = w.capture(True, keys16=True, pairs=True)
                ms16p = w.time(r16p, args.steps, args.warmup, barrier, max_over_ranks)
                f16["f16_key_table"]["two_heads_per_cta"] = {
                    "value": jobs * B * 1e3 / ms16p, "unit": "tokens/s", "ms_per_step": ms16p}
                del r16p
            w.dec.f16_key_table = False
            w.dec.key_table_pairs = False

    enc = None if (args.no_encode or world > 1) else encode_rate(dev, L, Hkv, n, stream)
    if enc is not None:
        enc["append_overlap"] = append_overlap(dev, replay, stream, L, B, Hkv, args.warmup)
        ok, ns = encode_sample_check(dev, stream)
        enc["bit_exact"] = ok
        enc["bit_exact_check"] = (f"{ns} vectors vs the C restatement of assign_codes (the "
                                  "candidate-grid path and the full scan)")

    line = {"metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True,
            "scaling": "strong" if plan["mode"] != "batch" else "weak",
            "vs_baseline": None,
            "dtype": "u8 codes / f32 accumulate" + (" (f16 value codebook)"
                                                    if args.f16_value_codebook else ""),
            "data": "synthetic (seeded uniform codes, N(0,1) codebooks, queries and recent "
                    "rows)",
            "config": config_dict(args.config, world),
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                         "frac": achieved / hbm_peak, "peak_kind": peak_kind,
                         "frac_of_nominal_8000_gbs": achieved / 8000.0,
                         "traffic": ncu_traffic(args.config),
                         "kernel": ncu_capture(args.config).get(
                             "kernel", kernel_label(args.config, args.f16_value_codebook)),
                         "shared_load_wavefronts_per_kv_token": ncu_capture(args.config).get(
                             "shared_load_wavefronts_per_kv_token"),
                         "kernel_ms_per_launch": k_ms,
                         "kernel_ms_isolated_launch": iso_ms,
                         "algorithmic_bytes_per_launch": bytes_per_launch,
                         "kernel_share_of_step": share},
            "e2e": {"value": jobs * B * 1e3 / e2e_ms, "unit": "tokens/s",
                    "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "api": "paper_2504_03661_b200.engine.PQDecoder (graph-replayed step)",
                    "copies": e2e_mode},
            "gpu_launches": launches_per_step * args.steps * (2 if seq_split else 1),
            "clocks": clocks,
            "code_stream_gbs_step": bytes_per_launch * L / (ms * 1e-3) / 1e9}
    if seq_split:
        line["sequence_split"] = {"merge_ms_per_step": merge_ms, "step_mode": w.graph_mode}
    if enc is not None:
        line["encode"] = enc
    if f16 is not None:
        line["f16_value_codebook_mode"] = f16
    del replay, w
    torch.cuda.empty_cache()

    # ---- the GQA configs beside it (N > 1: head-sharded and sequence-split) --
    if args.config == "llama2-32k" and not args.no_extra_configs:
        for extra in ("llama3-gqa-32k", "llama3-gqa-128k") if world > 1 else ("llama3-gqa-32k",):
            try:
                pe = shard_plan(extra, rank, world)
                we = Workload(args, pe, dev, stream, True)
                re_ = we.capture(False)
                mse = we.time(re_, args.steps, args.warmup, barrier, max_over_ranks)
                ent = {"value": pe["jobs"] * we.B * 1e3 / mse, "unit": "tokens/s",
                       "ms_per_step": mse, "config": config_dict(extra, world),
                       "scaling": "strong", "step_mode": we.graph_mode}
                if we.seq_split:
                    ent["merge_ms_per_step"] = merge_share(we, args.steps, barrier,
                                                           max_over_ranks)
                ent["roofline_frac"] = (we.bytes_per_launch * we.L /
                                        ((mse - ent.get("merge_ms_per_step", 0.0)) * 1e-3)
                                        / 1e9 / hbm_peak)
                ent["kernel"] = ("decode_gqa_pair (exact fp32, clusters of two CTAs, four query "
                                 "heads per pair)")
                del re_
                if not args.no_f16_mode:
                    # stated tolerance: fp16 value codebook + one packed fp16 key table
                    # for four query heads per CTA (decode_gqa4_f16)
                    r16 = we.capture(True, keys16=True)
                    ms16 = we.time(r16, args.steps, args.warmup, barrier, max_over_ranks)
                    ent["f16_key_table"] = {
                        "value": pe["jobs"] * we.B * 1e3 / ms16, "unit": "tokens/s",
                        "ms_per_step": ms16,
                        "roofline_frac": (we.bytes_per_launch * we.L /
                                          ((ms16 - ent.get("merge_ms_per_step", 0.0)) * 1e-3)
                                          / 1e9 / hbm_peak),
                        "kernel": "decode_gqa4_f16",
                        "tolerance": "rtol 2e-3, atol 2e-4 vs the fp64 reference "
                                     "(tests/test_gpu_gqa_tables.py)"}
                    del r16
                del we
                torch.cuda.empty_cache()
            except Exception as e:  # noqa: BLE001 -- the headline line still prints
                ent = {"error": f"{type(e).__name__}: {e!s:.200}"}
            line[extra.replace("-", "_")] = ent

    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        v, sample = cpu_decode_rate(args.config, 1, args.cpu_budget)
        line["cpu_baseline"] = {"value": v, "unit": "tokens/s", "cores": 1, "kind": "port",
                                "sample": sample}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist.is_initialized():
        dist.destroy_process_group()


def dry_run(args):
    """--dry-run: the launcher and shard plan without a GPU (gloo when no CUDA
    device is visible) -- every rank's plan gathered to rank 0, one JSON line."""
    import torch
    import torch.distributed as dist
    rank, world, _ = dist_env()
    if world != args.gpus:
        raise SystemExit(f"bench.py: WORLD_SIZE={world} but --gpus {args.gpus}")
    if world > 1:
        dist.init_process_group("gloo")
    plans = [shard_plan(c, rank, world) for c in CONFIGS]
    if world > 1:
        allp = [None] * world
        dist.all_gather_object(allp, plans)
    else:
        allp = [plans]
    if rank == 0:
        print(json.dumps({"dry_run": True, "n_gpus": world, "plans": allp,
                          "configs": {c: config_dict(c, world) for c in CONFIGS}}), flush=True)
    if world > 1:
        dist.destroy_process_group()


def relaunch(args):
    """`python bench.py --gpus N` (N > 1) outside torchrun: re-run this script
    under torch.distributed.run with N ranks (one per GPU), same arguments."""
    import socket
    if not args.dry_run:
        try:
            import torch
            have = torch.cuda.device_count()
        except Exception:  # noqa: BLE001
            have = 0
        if have < args.gpus:
            print(f"bench.py: --gpus {args.gpus} but {have} GPU(s) visible", file=sys.stderr)
            sys.exit(2)
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    sys.exit(subprocess.run(cmd).returncode)


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
    ap.add_argument("--seq-split-one", action="store_true",
                    help="config 4 on one GPU through the sequence-split path (a one-rank NCCL "
                         "group: the captured all-gather + rank-ordered merge, as at N > 1)")
    ap.add_argument("--no-extra-configs", action="store_true",
                    help="N > 1: skip the head-sharded / sequence-split configs beside config 2")
    ap.add_argument("--dry-run", action="store_true",
                    help="launcher + shard plan only (no GPU work; gloo when no GPU)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.gpus < 1:
        raise SystemExit("--gpus must be >= 1")
    if args.impl == "reference":
        run_reference(args)
        return
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        relaunch(args)
    if args.dry_run:
        dry_run(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
