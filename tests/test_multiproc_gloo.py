"""World-size-2 (gloo, CPU) test of the multi-GPU host logic: the sequence split
 -- token sharding, the all-gather of (d+4)-float
partial records and the fixed rank-order merge -- reproduces the unsplit
decode.  The per-rank partials come from the CPU oracle (test-only); on a GPU
box the same records come from PQDecoder(merged=...)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _partial_record(part, d):
    rec = np.zeros(d + 4)
    rec[0], rec[1], rec[4:] = (part.m if part.l else 0.0), part.l, part.acc
    return rec


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import pqkv_oracle as O
        from paper_2504_03661_b200.engine import gather_partials, shard_tokens

        rng = np.random.default_rng(0)  # same data on every rank
        n, d = 5000, 128
        ck = rng.standard_normal((64, 256, 2)).astype(np.float32)
        cv = rng.standard_normal((64, 256, 2)).astype(np.float32)
        codes_k = rng.integers(0, 256, (n, 64), dtype=np.uint8)
        codes_v = rng.integers(0, 256, (n, 64), dtype=np.uint8)
        qv = rng.standard_normal(d)
        rk = rng.standard_normal((5, d)).astype(np.float32)
        rv = rng.standard_normal((5, d)).astype(np.float32)
        kn = rng.standard_normal(d).astype(np.float32)
        vn = rng.standard_normal(d).astype(np.float32)

        a, b = shard_tokens(n, rank, world)
        table = O.key_lut(qv, ck)
        part = O.quantized_partial(table, codes_k[a:b], codes_v[a:b], cv)
        if rank == world - 1:  # the tail rank owns the recent window + current token
            dense = O.dense_partial(qv, np.vstack([rk, kn]), np.vstack([rv, vn]))
            part = O.merge(part, dense)
        rec = torch.from_numpy(_partial_record(part, d)).view(1, -1)
        gathered = gather_partials(rec)
        assert tuple(gathered.shape) == (world, 1, d + 4)
        merged = O.empty(d)
        for r in range(world):  # fixed rank order, as pqkv_merge_partials
            g = gathered[r, 0].numpy()
            merged = O.merge(merged, O.Partial(g[0] if g[1] else -np.inf, g[1], g[4:]))
        full = O.decode_from_snapshot(qv, kn, vn, codes_k, codes_v, rk, rv, ck, cv,
                                      block_size=1 << 30)
        q.put((rank, float(np.max(np.abs(O.finalize(merged) - full)))))
    finally:
        dist.destroy_process_group()


def test_sequence_split_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    errs = dict(q.get(timeout=5) for _ in range(2))
    assert max(errs.values()) < 1e-12


def _gpu_worker(rank, world, port, q):
    """Both ranks on the one GPU of the box: engine.sequence_parallel_decode
    with the real kernels (PQDecoder merged records, all-gather over gloo,
    rank-ordered device merge) == the unsplit decode."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2504_03661_b200 import kernels as K
        from paper_2504_03661_b200.engine import PQDecoder, sequence_parallel_decode, shard_tokens
        from paper_2504_03661_b200.pq_core import PQConfig
        rng = np.random.default_rng(3)  # same data on every rank
        B, Hq, Hkv, n = 2, 8, 2, 9000
        t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
        cbk = K.key_codebook_layout(t(rng.standard_normal((64, 256, 2)).astype(np.float32)), 8)
        cbv = K.value_codebook_layout(t(rng.standard_normal((64, 256, 2)).astype(np.float32)), 8)
        q_ = t(rng.standard_normal((B, Hq, 128)).astype(np.float32))
        ckr = t(rng.integers(0, 256, (B, Hkv, n, 64), dtype=np.uint8))
        cvr = t(rng.integers(0, 256, (B, Hkv, n, 64), dtype=np.uint8))
        rk = t(rng.standard_normal((B, Hkv, 8, 128)).astype(np.float32))
        rv = t(rng.standard_normal((B, Hkv, 8, 128)).astype(np.float32))
        nr = t(np.array([8, 5], np.int32))
        kc = t(rng.standard_normal((B, Hkv, 128)).astype(np.float32))
        vc = t(rng.standard_normal((B, Hkv, 128)).astype(np.float32))
        dec = PQDecoder(B, Hq, Hkv, PQConfig(128, 64, 8))
        full = dec(q_, K.relayout(ckr, True), K.relayout(cvr, True),
                   t(np.array([n, n], np.int32)), cbk, cbv, rk, rv, nr, kc, vc)
        a, b = shard_tokens(n, rank, world)
        tail = rank == world - 1
        out = sequence_parallel_decode(
            dec, None, q_, K.relayout(ckr[:, :, a:b], True), K.relayout(cvr[:, :, a:b], True),
            t(np.array([b - a] * B, np.int32)), cbk, cbv, rk if tail else None,
            rv if tail else None, nr if tail else None, kc if tail else None,
            vc if tail else None)
        torch.cuda.synchronize()
        q.put((rank, float((out - full).abs().max().item())))
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
def test_sequence_parallel_decode_gloo_world2_gpu():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gpu_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(300)
        assert p.exitcode == 0
    errs = dict(q.get(timeout=5) for _ in range(2))
    assert max(errs.values()) < 1e-5, errs
