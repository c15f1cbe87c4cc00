"""Batched, multi-layer GPU PQ KV cache for the serving path (``PQDecoder``).

The reference keeps one ``LayerKVCache`` per (layer, head) (kv_cache.py:42-302)
and loops over them in Python.  ``ServingCache`` holds every layer, sequence
and KV head of a model in a few HBM tensors laid out for the fused decode
launch, with the reference's semantics per (layer, sequence, head):

* quantized span: ``[L][B][Hkv][cap][M]`` uint8 in the decode layout
  (common.cuh), written by the bit-exact encoder (``pqkv_encode``), in paged
  stores (vstore.py: virtual reservation, pages mapped on growth, no copies);
* full-precision recent rows ``[L][B][Hkv][R_cap][d]`` float32, rows
  ``[0, n_recent[b])`` live;
* device lengths ``n_q[B]`` and ``n_recent[B]`` (one per sequence; every layer
  and head of a sequence holds the same tokens), so a decode step captured in
  a CUDA graph stays valid as the cache grows;
* flush trigger ``n_recent >= flush_threshold`` after an append, whole batches
  of the oldest ``flush_threshold`` rows (kv_cache.py:108-110, 197-215);
* single publication point: ``n_q`` grows (and the batch leaves the recent
  window) only after the batch's codes are written (kv_cache.py:228), so every
  token is covered exactly once by (codes, recent rows) (:269-290).

``async_flush=True`` (the reference's ``worker="thread"``) encodes on a
lowest-priority side stream, overlapping the following decode steps; the
batch stays in the recent window until the encode's event has completed, and
only then is the publication (n_q += batch, shift of the recent rows)
enqueued on the main stream -- ordered with the decodes, never blocking them.
All sequences advance together (one decode step appends one token to each).
"""

from __future__ import annotations

import torch

from . import kernels as K
from .pq_core import PQConfig

__all__ = ["ServingCache"]


class _nullctx:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False


class ServingCache:
    def __init__(self, layers: int, B: int, Hkv: int, config: PQConfig, centroids_k,
                 centroids_v, capacity: int, recent_capacity: int = 32,
                 flush_threshold: int = 32, async_flush: bool = True, device=None):
        """centroids_k / centroids_v: per layer (M, ksub, dsub) float32 tensors
        (or Codebooks).  capacity: maximum quantized tokens per sequence --
        reserved address space; memory is mapped as the cache fills."""
        if not K.is_fast_geometry(config.d, config.M, config.nbits):
            raise ValueError("ServingCache stores the m64b8 decode layout (d=128, M=64, nbits=8)")
        if len(centroids_k) != layers or len(centroids_v) != layers:
            raise ValueError("one key and one value codebook per layer")
        if recent_capacity < 0 or flush_threshold < 1:
            raise ValueError("recent_capacity >= 0 and flush_threshold >= 1 required")
        self.L, self.B, self.Hkv, self.config = layers, B, Hkv, config
        self.R, self.R_f = recent_capacity, flush_threshold
        self.device = torch.device(device) if device is not None else torch.device("cuda")
        dev, M, d = self.device, config.M, config.d

        def cents(c):
            c = c.device_centroids(dev) if hasattr(c, "device_centroids") else c
            return c.to(dev, torch.float32).contiguous()

        self.cents_k = [cents(c) for c in centroids_k]
        self.cents_v = [cents(c) for c in centroids_v]
        self.cents_k_all = torch.stack(self.cents_k)  # (L, M, ksub, dsub): batched flushes
        # the encoder's candidate grids (None for geometries without one)
        self.grid_k = [K.encode_grid(c, config.nbits) for c in self.cents_k]
        self.grid_v = [K.encode_grid(c, config.nbits) for c in self.cents_v]
        self.grid_k_all = (torch.stack(self.grid_k) if self.grid_k[0] is not None else None)
        self.grid_v_all = (torch.stack(self.grid_v) if self.grid_v[0] is not None else None)
        self.cents_v_all = torch.stack(self.cents_v)
        # decode-kernel codebook layouts (static: prepared once, at load time)
        self.cb_k = [K.key_codebook_layout(c, config.nbits) for c in self.cents_k]
        self.cb_v = [K.value_codebook_layout(c, config.nbits) for c in self.cents_v]
        # paged code stores (vstore.py): one region of virtual address space
        # per (layer, sequence, KV head) and kind, `capacity` rows each; pages
        # are mapped as the cache fills, so capacity costs address space only
        # and growth never copies (the decode kernel reads each head's rows
        # as one contiguous run, ld_tok = the region's row capacity)
        from .vstore import PagedCodeStore
        self._stores = [PagedCodeStore(layers * B * Hkv, capacity, (M,), torch.uint8, dev)
                        for _ in range(2)]
        self.capacity = capacity
        self.ld_tok = self._stores[0].max_rows  # row stride of a head: the reservation,
                                                # rounded up to whole pages
        self.codes_k = self._stores[0].tensor.view(layers, B, Hkv, self.ld_tok, M)
        self.codes_v = self._stores[1].tensor.view(layers, B, Hkv, self.ld_tok, M)
        # recent rows: the live window plus one in-flight batch and one step
        self.R_cap = max(1, recent_capacity + 2 * flush_threshold + 1)
        self.recent_k = torch.zeros((layers, B, Hkv, self.R_cap, d), device=dev)
        self.recent_v = torch.zeros_like(self.recent_k)
        self.n_q = torch.zeros(B, dtype=torch.int32, device=dev)
        self.n_recent = torch.zeros(B, dtype=torch.int32, device=dev)
        self._nq = 0          # host mirrors (every sequence holds the same tokens)
        self._nr = 0
        self._pending = None  # (event, batch) of the in-flight flush
        self.async_flush = async_flush
        lo, _ = torch.cuda.Stream.priority_range()
        self._side = torch.cuda.Stream(device=dev, priority=lo) if async_flush else None

    def ensure_rows(self, rows: int) -> None:
        """Back `rows` code rows of every (layer, sequence, head) with pages."""
        for st in self._stores:
            st.ensure(max(rows, 1))

    @property
    def mapped_rows(self) -> int:
        return self._stores[0].mapped_rows

    # -- views for PQDecoder --------------------------------------------------
    def layer(self, l: int) -> dict:
        """Keyword arguments of PQDecoder for layer l (plus q, k_cur, v_cur)."""
        return dict(codes_k=self.codes_k[l], codes_v=self.codes_v[l], n_q=self.n_q,
                    cb_k_layout=self.cb_k[l], cb_v_layout=self.cb_v[l],
                    recent_k=self.recent_k[l], recent_v=self.recent_v[l],
                    n_recent=self.n_recent)

    @property
    def n_quantized(self) -> int:
        return self._nq

    @property
    def n_recent_rows(self) -> int:
        return self._nr

    # -- writes -----------------------------------------------------------------
    def _encode(self, l: int, rows_k, rows_v, t_first: int, stream=None) -> None:
        """rows (B, Hkv, n, d) -> codes[l][:, :, t_first:t_first+n] (decode layout).
        The decode layout rotates bytes by the token index mod 8, so when n is
        a multiple of 8 all B * Hkv heads encode in one launch into a packed
        scratch (row v = (head, t) has index t_first + v == t_first + t mod 8)
        and land with one strided copy; otherwise one launch per head."""
        B, Hkv, n, d = rows_k.shape
        M = self.config.M
        for rows, cents, grid, store in ((rows_k, self.cents_k[l], self.grid_k[l], self.codes_k),
                                         (rows_v, self.cents_v[l], self.grid_v[l], self.codes_v)):
            if n % 8 == 0:
                tmp = K.encode(rows.reshape(B * Hkv * n, d), cents, self.config.nbits,
                               stream=stream, layout="decode", t_first=t_first, grid=grid)
                with torch.cuda.stream(stream) if stream is not None else _nullctx():
                    store[l, :, :, t_first:t_first + n] = tmp.view(B, Hkv, n, M)
            else:
                for b in range(B):
                    for h in range(Hkv):
                        K.encode(rows[b, h], cents, self.config.nbits,
                                 out=store[l, b, h, t_first:t_first + n], stream=stream,
                                 layout="decode", t_first=t_first, grid=grid)

    def _encode_all(self, rows_k, rows_v, t_first: int, stream=None) -> None:
        """rows (L, B, Hkv, n, d), n a multiple of 8 -> codes[:, :, :, t_first:+n]:
        one batched encode launch per kind for every layer (row v = (b, h, t)
        carries index t_first + v == t_first + t mod 8, see _encode), then one
        strided copy into the store."""
        L, B, Hkv, n, d = rows_k.shape
        M = self.config.M
        for rows, cents, grids, store in ((rows_k, self.cents_k_all, self.grid_k_all, self.codes_k),
                                          (rows_v, self.cents_v_all, self.grid_v_all, self.codes_v)):
            tmp = K.encode_batched(rows.reshape(L, B * Hkv * n, d), cents, self.config.nbits,
                                   stream=stream, layout="decode", t_first=t_first, grids=grids)
            with torch.cuda.stream(stream) if stream is not None else _nullctx():
                store[:, :, :, t_first:t_first + n] = tmp.view(L, B, Hkv, n, M)

    def prefill(self, K_rows: torch.Tensor, V_rows: torch.Tensor) -> None:
        """K/V (L, B, Hkv, n, d): encode all but the trailing min(R, n) rows,
        keep those full precision (prefill_ingest, kv_cache.py:152-181)."""
        if self._nq or self._nr:
            raise RuntimeError("prefill into a non-empty cache")
        L, B, Hkv, n, d = K_rows.shape
        if (L, B, Hkv, d) != (self.L, self.B, self.Hkv, self.config.d) or V_rows.shape != K_rows.shape:
            raise ValueError("prefill rows must be (L, B, Hkv, n, d)")
        keep = min(self.R, n)
        n_enc = n - keep
        if n_enc > self.capacity:
            raise ValueError("prefill exceeds the code capacity")
        self.ensure_rows(n_enc)
        if n_enc:
            self._encode_layers(K_rows[:, :, :, :n_enc].float().contiguous(),
                                V_rows[:, :, :, :n_enc].float().contiguous(), 0)
        self.recent_k[:, :, :, :keep] = K_rows[:, :, :, n_enc:]
        self.recent_v[:, :, :, :keep] = V_rows[:, :, :, n_enc:]
        self._nq, self._nr = n_enc, keep
        self.n_q.fill_(n_enc)
        self.n_recent.fill_(keep)

    def append(self, k: torch.Tensor, v: torch.Tensor) -> None:
        """One decode step's KV rows, k/v (L, B, Hkv, d), for every layer and
        sequence (append_decode, kv_cache.py:183-206)."""
        self._publish(block=False)
        if self._nr >= self.R_cap:
            self._publish(block=True)
        r = self._nr
        self.recent_k[:, :, :, r] = k
        self.recent_v[:, :, :, r] = v
        self._nr += 1
        self.n_recent.fill_(self._nr)
        if self._side is None:
            # the reference's sync worker flushes whole batches until the
            # window is below the threshold (append_decode, kv_cache.py:183-206)
            while self._nr >= self.R_f:
                self._flush()
            return
        inflight = self._pending[1] if self._pending else 0
        if self._nr - inflight >= self.R_f and self._pending is None:
            self._flush()

    def drain(self) -> None:
        """Run and publish every due flush (kv_cache.py:229-235)."""
        while True:
            self._publish(block=True)
            if self._nr >= self.R_f:
                self._flush()
            else:
                return

    # -- flush machinery -----------------------------------------------------------
    def _encode_layers(self, rows_k, rows_v, t_first: int, stream=None) -> None:
        if rows_k.shape[3] % 8 == 0:
            self._encode_all(rows_k, rows_v, t_first, stream)
        else:
            for l in range(self.L):
                self._encode(l, rows_k[l], rows_v[l], t_first, stream)

    def _flush(self) -> None:
        batch = self.R_f
        if self._nq + batch > self.capacity:
            raise RuntimeError("code capacity exhausted")
        self.ensure_rows(self._nq + batch)
        main = torch.cuda.current_stream(self.device)
        rows_k = self.recent_k[:, :, :, :batch].clone()  # snapshot on the main stream
        rows_v = self.recent_v[:, :, :, :batch].clone()
        if self._side is None:
            self._encode_layers(rows_k, rows_v, self._nq)
            self._pending = (None, batch)
            self._publish(block=True)
            return
        ready = torch.cuda.Event()
        ready.record(main)
        self._side.wait_event(ready)
        with torch.cuda.stream(self._side):
            rows_k.record_stream(self._side)
            rows_v.record_stream(self._side)
            self._encode_layers(rows_k, rows_v, self._nq, stream=self._side)
        done = torch.cuda.Event()
        done.record(self._side)
        self._pending = (done, batch)

    def _publish(self, block: bool) -> None:
        if self._pending is None:
            return
        done, batch = self._pending
        if done is not None:
            if not block and not done.query():
                return
            torch.cuda.current_stream(self.device).wait_event(done)
        # publication on the main stream, ordered with the decodes: the batch's
        # codes become visible and the rows leave the recent window together
        live = self._nr - batch
        if live:
            self.recent_k[:, :, :, :live] = self.recent_k[:, :, :, batch:self._nr].clone()
            self.recent_v[:, :, :, :live] = self.recent_v[:, :, :, batch:self._nr].clone()
        self._nq += batch
        self._nr = live
        self.n_q.fill_(self._nq)
        self.n_recent.fill_(self._nr)
        self._pending = None

    def _set_lengths(self, n_q: int, n_recent: int) -> None:
        """After a restore (fileio.load_serving_cache): publish the lengths."""
        self._nq, self._nr = n_q, n_recent
        self.n_q.fill_(n_q)
        self.n_recent.fill_(n_recent)

    def snapshot(self, l: int, b: int, h: int):
        """Host copy of (codes_k, codes_v) in the reference row layout and the
        recent rows of (layer, sequence, KV head), as the decodes enqueued so
        far see them (an in-flight flush stays unpublished) -- for checkers."""
        torch.cuda.current_stream(self.device).synchronize()
        n = self._nq
        ck = K.relayout(self.codes_k[l, b, h, :n].contiguous(), False) if n else self.codes_k[l, b, h, :0]
        cv = K.relayout(self.codes_v[l, b, h, :n].contiguous(), False) if n else self.codes_v[l, b, h, :0]
        return (ck.cpu().numpy(), cv.cpu().numpy(), self.recent_k[l, b, h, :self._nr].cpu().numpy(),
                self.recent_v[l, b, h, :self._nr].cpu().numpy())
