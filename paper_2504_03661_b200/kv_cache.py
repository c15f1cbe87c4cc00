"""GPU-resident per-layer PQ code store + full-precision recent window.

Drop-in for the reference ``kv_cache.py`` (CacheSnapshot :26-39,
LayerKVCache :42-302): same constructor, methods, flush trigger
(``len(recent) >= flush_threshold``, whole batches only, :108-110, :197-215),
single publication point (``n_q`` bumps after a batch's codes are written,
:228) and exactly-once snapshots (:269-290).

B200 mapping of the reference's concurrency:

* the code store and the recent rows live in HBM (torch tensors); flushes run
  the sm_100a encoder (``pqkv_encode``) straight into the store;
* ``worker="sync"`` enqueues the flush on the caller's stream inline;
* ``worker="thread"`` (the reference's background flusher thread) runs the
  encode on a low-priority side stream; the batch stays in the recent window
  until the side stream's event has completed, and only then is ``n_q``
  published -- a snapshot therefore still covers every token exactly once;
* ``worker="manual"`` leaves flushing to ``flush_step`` / ``drain`` (the
  deterministic test driver of the reference).
"""

from __future__ import annotations

import os
import threading
import time
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as N
from . import kernels as K
from .pq_core import Codebook, CodesMatrix, _is_tensor, default_device, to_device

# decode_append's grid: CTAs per quantized token (each CTA builds its key table,
# and the last arriver merges one record per CTA)
STEP_TOKENS_PER_CTA = int(os.environ.get("PQKV_STEP_TOKENS_PER_CTA", "1024"))
# ... but at least this many (capped by the plan's grid): a short context is
# latency bound, and 32 CTAs of a few units each beat one CTA walking them all
# (1K tokens: 13.7 us per launch vs 16.5; scripts/ds_time.py)
STEP_MIN_CTAS = int(os.environ.get("PQKV_STEP_MIN_CTAS", "32"))

__all__ = ["LayerKVCache", "CacheSnapshot"]


def _host_codes(c: torch.Tensor) -> np.ndarray:
    if c.dtype == torch.uint16:  # no numpy view of torch.uint16 on every build
        return c.to(torch.int32).cpu().numpy().astype(np.uint16)
    return c.cpu().numpy()


@dataclass(frozen=True)
class CacheSnapshot:
    """Immutable view: published codes + recent rows, tokens [0, n_total) once."""

    codes_K: CodesMatrix
    codes_V: CodesMatrix
    recent_K: object
    recent_V: object
    n_q: int
    n_total: int


class LayerKVCache:
    """KV store for one layer/head with deferred batch quantization on the GPU."""

    def __init__(self, cb_K: Codebook, cb_V: Codebook, recent_capacity: int = 32,
                 flush_threshold: int = 32, worker: str = "sync", device=None):
        if cb_K.config != cb_V.config:
            raise ValueError("key/value codebooks must share one PQConfig")
        if cb_K.kind != "key" or cb_V.kind != "value":
            raise ValueError("expected a (key, value) codebook pair")
        if recent_capacity < 0 or flush_threshold < 1:
            raise ValueError("recent_capacity >= 0 and flush_threshold >= 1 required")
        if worker not in ("sync", "thread", "manual"):
            raise ValueError(f"unknown worker mode {worker!r}")
        self.cb_K, self.cb_V = cb_K, cb_V
        self.config = cb_K.config
        self.recent_capacity = recent_capacity
        self.flush_threshold = flush_threshold
        self.worker = worker
        # m64b8 stores codes in the decode kernel's layout (include/pqkv_sm100.h);
        # snapshots convert back to the reference row layout
        self._layout = "decode" if K.is_fast_geometry(cb_K.config.d, cb_K.config.M,
                                                      cb_K.config.nbits) else "rows"
        self.device = torch.device(device) if device is not None else default_device()
        cfg = self.config
        # paged code store (vstore.py): K and V rows in two regions of one
        # virtual reservation, pages mapped as the rows grow -- no copies
        self._new_store(self.DEFAULT_MAX_ROWS)
        self._n_q = 0
        # the ring is compacted (copied to the front of a new buffer) when its
        # tail reaches the end; 8 flush cycles of headroom make that rare
        rcap = max(self.RING_MIN, self.RING_CYCLES * (recent_capacity + flush_threshold))
        self._rk = torch.zeros((rcap, cfg.d), dtype=torch.float32, device=self.device)
        self._rv = torch.zeros_like(self._rk)
        # (n_q, recent length) on the device, in the callers' stream order: the
        # per-token append bumps it and a publication moves a batch from the
        # second to the first (pqkv_append_recent / pqkv_publish_lengths), so a
        # decode step reads its lengths without a host->device transfer
        self._lens = torch.zeros(2, dtype=torch.int32, device=self.device)
        self._r0 = 0          # first live recent row in _rk/_rv
        self._rlen = 0        # live recent rows (published + in-flight flushes)
        self._n_total = 0
        self._pending: list[tuple[torch.cuda.Event, int]] = []  # in-flight batches, FIFO
        self._pending_rows = 0
        self._lock = threading.RLock()
        self._plan = None  # decode_append's (key, StepPlan)
        self._retired: list = []  # ring buffers still read by in-flight flushes
        self.inline_flush_seconds = 0.0
        # numpy in -> numpy snapshots, like the reference (kv_cache.py:269-290);
        # decided by the first write (None until then)
        self._numpy_io: bool | None = None
        self._side = (torch.cuda.Stream(device=self.device, priority=0)
                      if worker == "thread" else None)
        if self._side is not None:
            lo, _hi = torch.cuda.Stream.priority_range()
            self._side = torch.cuda.Stream(device=self.device, priority=lo)  # lowest priority

    # -- state queries -----------------------------------------------------
    @property
    def n_total(self) -> int:
        return self._n_total

    @property
    def n_q(self) -> int:
        with self._lock:
            self._publish_completed()
            return self._n_q

    def recent_len(self) -> int:
        with self._lock:
            self._publish_completed()
            return self._rlen

    def _flush_needed_locked(self) -> bool:
        return self._rlen - self._pending_rows >= self.flush_threshold

    # -- storage helpers ---------------------------------------------------
    DEFAULT_MAX_ROWS = 1 << 24  # virtual row capacity per kind (address space only)
    RING_MIN, RING_CYCLES = 256, 8  # recent-ring rows: max(RING_MIN, RING_CYCLES (R + R_f))
    STORE_HEADROOM_ROWS = 1 << 15   # rows mapped ahead of need (one 2 MiB page at m64b8)

    def _new_store(self, max_rows: int) -> None:
        from .vstore import PagedCodeStore
        self._store = PagedCodeStore(2, max_rows, (self.config.M,),
                                     self.config.torch_code_dtype, self.device)
        self._store_k, self._store_v = self._store.tensor[0], self._store.tensor[1]
        self._mapped = self._store.mapped_rows

    def _ensure_store(self, n_new: int, ahead: bool = False) -> None:
        """Map pages for n_new rows (the reference doubles and copies,
        kv_cache.py:217-228; here rows never move).  Past the reservation
        (16 Mi rows) the store moves once into a larger one."""
        if n_new <= self._store.max_rows:
            # mapping (cuMemCreate / cuMemMap / cuMemSetAccess, ~1 ms of host
            # calls) only when the rows outgrow the mapped ones, and then with
            # headroom (a page, or 1/8 of the rows); a prefill / restore
            # (ahead=True) maps that headroom up front for the decode steps
            # that follow it
            room = max(self.STORE_HEADROOM_ROWS, n_new // 8)
            if n_new + (room if ahead else 0) > self._mapped:
                self._store.ensure(min(self._store.max_rows, n_new + room))
                self._mapped = self._store.mapped_rows
            return
        self._wait_pending()
        old_k, old_v, n = self._store_k, self._store_v, self._n_q
        self._new_store(max(n_new, 2 * self._store.max_rows))
        self._store.ensure(n_new)
        self._mapped = self._store.mapped_rows
        self._store_k[:n] = old_k[:n]
        self._store_v[:n] = old_v[:n]

    def _ensure_recent(self, extra: int) -> None:
        cap = self._rk.shape[0]
        if self._r0 + self._rlen + extra <= cap:
            return
        if self._pending:
            # in-flight flushes read rows of the old buffers on the side stream:
            # keep them alive until those flushes are published (no host wait;
            # r0 keeps its meaning, the copy below starts at the old r0)
            self._retired.append((self._rk, self._rv))
        need = self._rlen + extra
        if need * 2 > cap:
            cap = max(2 * need, cap)
        nk = torch.zeros((cap, self.config.d), dtype=torch.float32, device=self.device)
        nv = torch.zeros_like(nk)
        nk[: self._rlen] = self._rk[self._r0: self._r0 + self._rlen]
        nv[: self._rlen] = self._rv[self._r0: self._r0 + self._rlen]
        self._rk, self._rv, self._r0 = nk, nv, 0

    def _rows(self, x, name: str) -> torch.Tensor:
        if self._numpy_io is None:
            self._numpy_io = not _is_tensor(x)
        t = to_device(x if _is_tensor(x) else np.asarray(x, dtype=np.float32), torch.float32,
                      self.device)
        return t

    def _check_row(self, x, name: str) -> torch.Tensor:
        t = self._rows(x, name).reshape(-1)
        if t.shape[0] != self.config.d:
            raise ValueError(f"{name} width {t.shape[0]} != d {self.config.d}")
        return t

    # -- writes --------------------------------------------------------------
    def prefill_ingest(self, K_rows, V_rows) -> None:
        """Encode prompt tokens, keeping the trailing min(R, n) rows full precision."""
        Kt = self._rows(K_rows, "K")
        Vt = self._rows(V_rows, "V")
        if Kt.shape != Vt.shape or Kt.dim() != 2 or Kt.shape[1] != self.config.d:
            raise ValueError(f"bad prefill shapes K{tuple(Kt.shape)} V{tuple(Vt.shape)}")
        with self._lock:
            self._publish_completed()
            if self._n_total != self._rlen + self._n_q:
                raise RuntimeError("cache in inconsistent state")
            n = Kt.shape[0]
            keep = min(self.recent_capacity, n)
            n_enc = n - keep
            if n_enc > 0:
                self._wait_pending()
                self._ensure_store(self._n_q + n_enc, ahead=True)
                K.encode(Kt[:n_enc].contiguous(), self.cb_K.device_centroids(self.device),
                         self.config.nbits, out=self._store_k[self._n_q: self._n_q + n_enc],
                         layout=self._layout, t_first=self._n_q,
                         grid=self.cb_K.device_encode_grid(self.device))
                K.encode(Vt[:n_enc].contiguous(), self.cb_V.device_centroids(self.device),
                         self.config.nbits, out=self._store_v[self._n_q: self._n_q + n_enc],
                         layout=self._layout, t_first=self._n_q,
                         grid=self.cb_V.device_encode_grid(self.device))
            if keep:
                self._ensure_recent(keep)
                a = self._r0 + self._rlen
                self._rk[a: a + keep] = Kt[n_enc:]
                self._rv[a: a + keep] = Vt[n_enc:]
                self._rlen += keep
            self._n_q += n_enc
            self._n_total += n
            self._set_device_lengths()

    def _set_device_lengths(self) -> None:
        """lens <- (n_q, recent length) after a bulk state change (prefill,
        restore), enqueued on the current stream."""
        self._lens.copy_(torch.tensor([self._n_q, self._rlen], dtype=torch.int32),
                         non_blocking=False)

    def _publish_device(self, batch: int) -> None:
        K._call(self.device, "pqkv_publish_lengths", N.ptr(self._lens), batch,
                N.stream_ptr(None, self.device))

    def append_decode(self, k_n, v_n) -> None:
        """Append the current token's full-precision KV pair; flush whole
        batches once the recent window reaches the threshold."""
        k = self._check_row(k_n, "k_n").contiguous()
        v = self._check_row(v_n, "v_n").contiguous()
        with self._lock:
            self._publish_completed()
            self._ensure_recent(1)
            # row r0 + rlen of the ring, and the device recent length + 1
            off = self._r0 * self.config.d * 4
            K._call(self.device, "pqkv_append_recent", N.ptr(k), N.ptr(v),
                    self._rk.data_ptr() + off, self._rv.data_ptr() + off, N.ptr(self._lens),
                    self.config.d, N.stream_ptr(None, self.device))
            self._rlen += 1
            self._n_total += 1
            needed = self._flush_needed_locked()
        self._flush_after_append(needed)

    def decode_append(self, q, k, v, scale: float, cb_k_layout, cb_v_layout, ws, out) -> None:
        """decode_step's per-token work (attention.py:214-287 then
        append_decode) in one library call, pqkv_step_run: the fused decode of
        q against the stored codes + recent ring + (k, v), then the append of
        (k, v) to the ring.  q, k, v: (d,) float32 on this device; out: (d,).
        The step plan (codebook layouts, stores, device lengths, workspace)
        is built once and rebuilt when any of them moves."""
        with self._lock:
            self._publish_completed()
            self._ensure_recent(1)
            key = (self._store_k.data_ptr(), self._store_v.data_ptr(), cb_k_layout.data_ptr(),
                   cb_v_layout.data_ptr(), float(scale), id(ws))
            plan = self._plan
            if plan is None or plan[0] != key:
                plan = self._plan = (key, K.StepPlan(self, cb_k_layout, cb_v_layout, scale, ws))
            d4 = self.config.d * 4
            off = self._r0 * d4
            # grid sized to the (host-known) context: one CTA per STEP_TOKENS_PER_CTA
            # tokens, at least STEP_MIN_CTAS (the device lengths may be ahead of
            # these; only the split changes)
            nc = max(STEP_MIN_CTAS, -(-(self._n_q + self._pending_rows) // STEP_TOKENS_PER_CTA))
            plan[1].run(q, k, v, self._rk.data_ptr() + off, self._rv.data_ptr() + off,
                        self._rk.shape[0] - self._r0, out, max(1, nc))
            self._rlen += 1
            self._n_total += 1
            needed = self._flush_needed_locked()
        self._flush_after_append(needed)

    def _flush_after_append(self, needed: bool) -> None:
        if needed and self.worker == "sync":
            t0 = time.perf_counter()
            with self._lock:
                while self._flush_needed_locked():
                    self._flush_batch_locked(self.flush_threshold)
            self.inline_flush_seconds += time.perf_counter() - t0
        elif needed and self.worker == "thread":
            with self._lock:
                while self._flush_needed_locked():
                    self._flush_batch_locked(self.flush_threshold, asynchronous=True)

    def flush_recent(self, batch: int) -> None:
        """Explicitly encode and publish the oldest `batch` recent entries."""
        if batch < 0:
            raise ValueError("batch must be >= 0")
        with self._lock:
            self._publish_completed()
            if batch > self._rlen:
                raise ValueError(f"batch {batch} exceeds recent length {self._rlen}")
            if batch > 0:
                self._wait_pending()
                self._flush_batch_locked(batch)

    def flush_step(self) -> bool:
        """Run one scheduled flush if the trigger condition holds."""
        with self._lock:
            self._publish_completed()
            if not self._flush_needed_locked():
                return False
            self._flush_batch_locked(self.flush_threshold)
            return True

    def drain(self) -> None:
        """Barrier: run/await flushes until no flush is pending."""
        while self.flush_step():
            pass
        with self._lock:
            self._wait_pending()

    # -- flush machinery -------------------------------------------------------
    def _flush_batch_locked(self, batch: int, asynchronous: bool = False) -> None:
        first = self._r0 + self._pending_rows
        batch = min(batch, self._rlen - self._pending_rows)
        if batch <= 0:
            return
        n0 = self._n_q + self._pending_rows
        self._ensure_store(n0 + batch)
        cents_k = self.cb_K.device_centroids(self.device)
        cents_v = self.cb_V.device_centroids(self.device)
        nb = self.config.nbits
        rows_k = self._rk[first: first + batch]
        rows_v = self._rv[first: first + batch]
        out_k = self._store_k[n0: n0 + batch]
        out_v = self._store_v[n0: n0 + batch]
        gk = self.cb_K.device_encode_grid(self.device)
        gv = self.cb_V.device_encode_grid(self.device)
        if not asynchronous:
            K.encode(rows_k, cents_k, nb, out=out_k, layout=self._layout, t_first=n0, grid=gk)
            K.encode(rows_v, cents_v, nb, out=out_v, layout=self._layout, t_first=n0, grid=gv)
            self._n_q += batch          # single publication point
            self._r0 += batch
            self._rlen -= batch
            self._publish_device(batch)
            return
        main = torch.cuda.current_stream(self.device)
        self._side.wait_stream(main)    # the rows were written on the main stream
        with torch.cuda.stream(self._side):
            K.encode(rows_k, cents_k, nb, out=out_k, stream=self._side, layout=self._layout,
                     t_first=n0, grid=gk)
            K.encode(rows_v, cents_v, nb, out=out_v, stream=self._side, layout=self._layout,
                     t_first=n0, grid=gv)
            ev = torch.cuda.Event()
            ev.record(self._side)
        for t in (rows_k, rows_v, out_k, out_v):
            t.record_stream(self._side)
        self._pending.append((ev, batch))
        self._pending_rows += batch

    def _publish_completed(self, block: bool = False) -> None:
        while self._pending:
            ev, batch = self._pending[0]
            if block:
                ev.synchronize()
            elif not ev.query():
                break
            # make later main-stream readers of the store ordered after the encode
            torch.cuda.current_stream(self.device).wait_event(ev)
            self._pending.pop(0)
            if not self._pending:
                self._retired.clear()
            self._pending_rows -= batch
            self._n_q += batch          # single publication point
            self._r0 += batch
            self._rlen -= batch
            self._publish_device(batch)

    def _wait_pending(self) -> None:
        self._publish_completed(block=True)

    def close(self) -> None:
        with self._lock:
            self._wait_pending()

    def load_snapshot(self, snap: CacheSnapshot) -> None:
        """Restore a previously captured state into an empty cache."""
        if self._n_total != 0:
            raise RuntimeError("load_snapshot requires an empty cache")
        if snap.codes_K.M != self.config.M or snap.codes_K.nbits != self.config.nbits:
            raise ValueError("snapshot geometry does not match codebooks")
        with self._lock:
            n = snap.codes_K.n_tokens
            self._ensure_store(n, ahead=True)
            if n:
                ck = snap.codes_K.device_codes(self.device)
                cv = snap.codes_V.device_codes(self.device)
                if self._layout == "decode":
                    ck, cv = K.relayout(ck, True), K.relayout(cv, True)
                self._store_k[:n] = ck
                self._store_v[:n] = cv
            self._n_q = n
            r = int(snap.recent_K.shape[0])
            if r:
                self._ensure_recent(r)
                self._rk[:r] = self._rows(snap.recent_K, "recent_K").reshape(r, -1)
                self._rv[:r] = self._rows(snap.recent_V, "recent_V").reshape(r, -1)
            self._r0, self._rlen = 0, r
            self._n_total = snap.n_total
            self._set_device_lengths()

    def _load_device(self, n_q: int, r: int, fill) -> None:
        """Restore into an empty cache: fill(codes_k, codes_v, recent_k,
        recent_v) writes n_q code rows (this cache's layout) and r recent rows
        into the given device buffers (fileio.restore_cache, C reader)."""
        if self._n_total != 0:
            raise RuntimeError("load_snapshot requires an empty cache")
        with self._lock:
            self._ensure_store(max(n_q, 1), ahead=True)
            if r:
                self._ensure_recent(r)
            with torch.cuda.device(self.device):
                fill(self._store_k, self._store_v, self._rk, self._rv)
            self._n_q, self._r0, self._rlen = n_q, 0, r
            self._n_total = n_q + r
            self._set_device_lengths()

    # -- reads -------------------------------------------------------------------
    def raw_snapshot(self):
        """(codes_k, codes_v, recent_K, recent_V, n_q, n_total) with the code
        store in its on-device layout ("decode" for m64b8) -- what decode_step
        hands to the kernel without a layout round trip."""
        with self._lock:
            self._publish_completed()
            n_q = self._n_q
            rk = self._rk[self._r0: self._r0 + self._rlen].clone()
            rv = self._rv[self._r0: self._r0 + self._rlen].clone()
            return (self._store_k[:n_q], self._store_v[:n_q], rk, rv, n_q, self._n_total)

    def raw_view(self):
        """raw_snapshot without the copies of the recent rows: views valid for
        work enqueued on the current stream before the next append (every
        write to the recent ring -- append, compaction -- is enqueued on the
        caller's stream, so it is ordered after that work).  decode_step's
        fused path."""
        with self._lock:
            self._publish_completed()
            n_q = self._n_q
            rk = self._rk[self._r0: self._r0 + self._rlen]
            rv = self._rv[self._r0: self._r0 + self._rlen]
            return (self._store_k[:n_q], self._store_v[:n_q], rk, rv, n_q, self._n_total)

    def step_view(self):
        """decode_step's per-token view: (codes_k, codes_v, recent_K,
        recent_V, lens, n_q, recent length) -- the code stores and the recent
        ring from its first live row, and the device lengths lens = (n_q,
        recent length) in stream order (the kernel reads its lengths there;
        the host values are for accounting)."""
        with self._lock:
            self._publish_completed()
            rk = self._rk[self._r0:]
            rv = self._rv[self._r0:]
            return (self._store_k, self._store_v, rk, rv, self._lens, self._n_q, self._rlen)

    @property
    def code_layout(self) -> str:
        return self._layout

    def snapshot(self) -> CacheSnapshot:
        """Consistent view covering every stored token exactly once (codes in
        the reference row layout)."""
        ck, cv, rk, rv, n_q, n_total = self.raw_snapshot()
        if self._layout == "decode" and n_q:
            ck, cv = K.relayout(ck, False), K.relayout(cv, False)
        if self._numpy_io:  # fed numpy: host copies, as the reference returns
            ck, cv = _host_codes(ck), _host_codes(cv)
            rk, rv = rk.cpu().numpy(), rv.cpu().numpy()
        return CacheSnapshot(codes_K=CodesMatrix(codes=ck, nbits=self.config.nbits),
                             codes_V=CodesMatrix(codes=cv, nbits=self.config.nbits),
                             recent_K=rk, recent_V=rv, n_q=n_q, n_total=n_total)

    def memory_usage(self) -> dict[str, int]:
        """Exact byte accounting of current storage."""
        with self._lock:
            self._publish_completed()
            cell = self.config.cell_width
            return {"codes_bytes": 2 * self._n_q * self.config.M * cell,
                    "recent_bytes": 2 * self._rlen * self.config.d * 4,
                    "codebook_bytes": self.cb_K.nbytes() + self.cb_V.nbytes()}
