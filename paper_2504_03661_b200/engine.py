"""Batched decode attention over GPU-resident PQ caches (the serving hot path).

The reference decodes one head of one sequence per call (attention.py:214,
a per-head Python loop in harness.py:195-201).  Here one call covers a whole
layer: every sequence b < B and query head hq < Hq, with GQA (query head hq
reads KV head hq // (Hq // Hkv)).  One launch per layer
(``pqkv_decode_attention``): one persistent CTA per SM builds each head's key
LUT in shared memory (build_key_lut, attention.py:70-83) and streams the codes
of all heads (quantized_partial, attention.py:114-166); the CTA holding a
head's first tokens also computes the dense partial over the recent rows +
current token (dense_partial :169-190), and the last CTA to finish a head
merges its records in a fixed order and finalizes (:193-211, 264-274).
With ``pdl=True`` consecutive layers overlap: a layer's grid starts loading
its value codebook while the previous layer's last CTAs drain.

Lengths are device-resident, so a whole decode step (all layers) can be
captured in a CUDA graph and replayed.

Multi-GPU: head/batch sharding needs no collective -- each
rank runs ``PQDecoder`` on its own heads.  A sequence split (128K context)
runs the same launches on each rank's token range with
``merged=`` records instead of a finalized output, all-gathers the
(d + 4)-float records and merges them in rank order
(``sequence_parallel_decode``), the cross-GPU form of merge_partials.
"""

from __future__ import annotations

import torch

from . import kernels as K
from .pq_core import PQConfig

__all__ = ["PQDecoder", "sequence_parallel_decode", "gather_partials", "shard_tokens",
           "random_codes"]


class PQDecoder:
    """Decode attention for one (B, Hq, Hkv, geometry) launch shape."""

    def __init__(self, B: int, Hq: int, Hkv: int, config: PQConfig, device=None,
                 num_ctas: int | None = None, pdl: bool = False, static_codebooks: bool = False,
                 early_codes: bool = False, f16_key_table: bool = False,
                 key_table_pairs: bool = False):
        if Hq % Hkv:
            raise ValueError(f"Hq={Hq} is not a multiple of Hkv={Hkv}")
        self.B, self.Hq, self.Hkv, self.config = B, Hq, Hkv, config
        self.ws = K.DecodeWorkspace(B, Hq, config.d, config.M, config.nbits, device=device,
                                    num_ctas=num_ctas)
        self.device = self.ws.device
        self.pdl, self.static_codebooks, self.early_codes = pdl, static_codebooks, early_codes
        # stated-tolerance GQA mode (with an fp16 value codebook layout)
        self.f16_key_table = f16_key_table
        self.key_table_pairs = key_table_pairs  # two query heads per CTA even for groups of 4

    @property
    def num_ctas(self) -> int:
        return self.ws.num_ctas

    def __call__(self, q, codes_k, codes_v, n_q, cb_k_layout, cb_v_layout, recent_k=None,
                 recent_v=None, n_recent=None, k_cur=None, v_cur=None, out=None, lse=None,
                 merged=None, scale: float | None = None, stream=None, finalize: bool = True):
        """q (B, Hq, d) f32; codes (B, Hkv, cap, M); n_q (B,) int32 device;
        cb_k_layout / cb_v_layout from kernels.key/value_codebook_layout (or
        Codebook.device_key_layout / device_value_layout);
        recent (B, Hkv, R, d) f32 + n_recent (B,) int32; k_cur/v_cur (B, Hkv, d).
        Returns out (B, Hq, d) f32 (or only fills lse / merged)."""
        cfg = self.config
        B, Hq, d = self.B, self.Hq, cfg.d
        if q.shape != (B, Hq, d):
            raise ValueError(f"q must be {(B, Hq, d)}, got {tuple(q.shape)}")
        sc = K.default_scale(d) if scale is None else float(scale)
        qf = q if (q.dtype == torch.float32 and q.is_contiguous()) else q.float().contiguous()
        if out is None and finalize:
            out = torch.empty((B, Hq, d), dtype=torch.float32, device=q.device)
        K.decode_attention(self.ws, self.Hkv, qf.view(B * Hq, d), sc, cb_k_layout, codes_k,
                           codes_v, n_q, cb_v_layout, recent_k=recent_k, recent_v=recent_v,
                           n_recent=n_recent, k_cur=k_cur, v_cur=v_cur, out=out, lse=lse,
                           merged=merged, pdl=self.pdl, static_codebooks=self.static_codebooks,
                           early_codes=self.early_codes, f16_key_table=self.f16_key_table,
                           key_table_pairs=self.key_table_pairs,
                           stream=stream)
        return out


def sequence_parallel_decode(decoder: PQDecoder, group, q, codes_k, codes_v, n_q, cb_k_layout,
                             cb_v_layout, recent_k=None, recent_v=None, n_recent=None,
                             k_cur=None, v_cur=None, scale: float | None = None, out=None):
    """Context-parallel decode: this rank holds a contiguous token range of
    every head; the rank(s) owning the tail pass the recent rows / current
    token.  One all-gather of (B*Hq, d+4) partial records, merged in rank
    order on the device (merge_partials is associative, attention.py:193-204;
    a fixed order keeps the result identical on every rank)."""
    import torch.distributed as dist

    B, Hq, d = decoder.B, decoder.Hq, decoder.config.d
    rec = torch.empty((B * Hq, d + 4), dtype=torch.float32, device=q.device)
    decoder(q, codes_k, codes_v, n_q, cb_k_layout, cb_v_layout, recent_k, recent_v, n_recent, k_cur,
            v_cur, merged=rec, scale=scale, finalize=False)
    gathered = gather_partials(rec, group)
    if out is None:
        out = torch.empty((B, Hq, d), dtype=torch.float32, device=q.device)
    K.merge_partials(gathered, out=out)
    return out


def gather_partials(rec: torch.Tensor, group=None) -> torch.Tensor:
    """All-gather one (heads, d+4) record per rank -> (world, heads, d+4)."""
    import torch.distributed as dist

    world = dist.get_world_size(group)
    if dist.get_backend(group) == "nccl":
        out = torch.empty((world, *rec.shape), dtype=rec.dtype, device=rec.device)
        dist.all_gather_into_tensor(out, rec.contiguous(), group=group)
        return out
    bufs = [torch.empty_like(rec) for _ in range(world)]
    dist.all_gather(bufs, rec.contiguous(), group=group)
    return torch.stack(bufs)


def shard_tokens(n: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous token range [a, b) of rank in a sequence split of n tokens
    (GPU g owns [g*n/W, (g+1)*n/W); the last rank owns the tail,
    hence the recent window and every appended token)."""
    if world <= 0 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    return (n * rank) // world, (n * (rank + 1)) // world


def random_codes(shape, nbits: int, generator: torch.Generator | None = None, device=None):
    """Uniform random codes (the bank-conflict worst case for table gathers)."""
    hi = 1 << nbits
    dt = K.code_dtype(nbits)
    if dt == torch.uint8:
        return torch.randint(0, hi, shape, dtype=torch.uint8, device=device, generator=generator)
    return torch.randint(0, hi, shape, dtype=torch.int32, device=device,
                         generator=generator).to(torch.uint16)
