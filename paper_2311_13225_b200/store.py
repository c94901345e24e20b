"""Versioned historical-embedding store with the bounded-staleness contract
(reference store.py:1-146), device-backed.

``EmbeddingStore`` keeps the reference's protocol object-for-object: ``put``
only for super-batch current+1, ``get`` only inside the current window, a hit
asserts ``reading_batch - version <= 2n - 1``, ``advance_super_batch`` swaps
the double buffer in O(1), ``reset_epoch`` drops everything.  Rows live in two
device tables (current / staging) addressed through a vertex -> slot map; the
per-row version and stamp arrays make both promotion and reset O(1): a slot is
readable iff its stamp equals the current super-batch's stamp.

The training engine uses the same layout in bulk (engine.HotBuffers with the
``hg_store_put`` / ``hg_store_lookup`` / ``hg_inject_rows`` kernels); this class
is the reference-shaped front for drop-in use and the protocol tests.
"""

from __future__ import annotations

import threading

import numpy as np
import torch

from . import _lib
from .device import ptr, require_cuda, stream_ptr


class StalenessViolation(RuntimeError):
    """store.py:16-17: a reuse event exceeded the 2n-1 version gap."""


class StoreContractError(ValueError):
    """store.py:20-21: misuse of the staging protocol."""


class FallbackBudgetExceeded(RuntimeError):
    """orchestrator.py:70-71."""


class EmbeddingStore:
    """store.py:24-146 with device tables (capacity grows on demand)."""

    def __init__(self, n: int, emb_dim: int, capacity: int = 1024, device=None):
        if n < 1:
            raise StoreContractError(f"super-batch size must be >= 1, got {n}")
        self.device = require_cuda(device)
        self.n, self.emb_dim = int(n), int(emb_dim)
        self.current_super_batch = 0
        self._window_start, self._window_len = 0, self.n
        self._slot = {}  # vertex -> slot (slots are never reused; table grows)
        self._cap = 0
        self._tab = [None, None]
        self._ver = [None, None]
        self._stamp = [None, None]
        self._cur = 0  # index of the "current" physical table
        self._stamp_serial = 1
        self._cur_stamp, self._stage_stamp = 0, 1
        self._staged = 0
        self._live_cur = 0
        self._lock = threading.RLock()
        self.hits = self.misses = self.puts = 0
        self.max_observed_gap, self.max_gap_batch, self.max_gap_super_batch = 0, -1, -1
        self._grow(max(int(capacity), 1))

    @property
    def gap_bound(self) -> int:
        return 2 * self.n - 1

    def _grow(self, cap):
        if cap <= self._cap:
            return
        dev = self.device
        for k in range(2):
            tab = torch.zeros((cap, self.emb_dim), dtype=torch.float32, device=dev)
            ver = torch.zeros(cap, dtype=torch.int32, device=dev)
            st = torch.full((cap,), -1, dtype=torch.int32, device=dev)
            if self._cap:
                tab[:self._cap] = self._tab[k]
                ver[:self._cap] = self._ver[k]
                st[:self._cap] = self._stamp[k]
            self._tab[k], self._ver[k], self._stamp[k] = tab, ver, st
        self._cap = cap

    def _slot_of(self, v):
        s = self._slot.get(v)
        if s is None:
            s = len(self._slot)
            self._slot[v] = s
            if s >= self._cap:
                self._grow(2 * self._cap)
        return s

    # -- protocol --------------------------------------------------------------
    def put(self, v: int, emb, version: int, target_super_batch: int) -> None:
        """store.py:53-65."""
        self.put_many(np.array([int(v)]), np.asarray(emb).reshape(1, -1), version, target_super_batch)

    def put_many(self, vs, embs, version: int, target_super_batch: int) -> None:
        """``put`` for many vertices at one version (``puts`` counts every call's rows,
        as that many reference ``put`` calls would)."""
        n_calls = int(np.asarray(vs).reshape(-1).shape[0])
        with self._lock:
            if target_super_batch != self.current_super_batch + 1:
                raise StoreContractError(f"put targets super-batch {target_super_batch} but only "
                                         f"{self.current_super_batch + 1} is stageable")
            vs = np.asarray(vs, np.int64).reshape(-1)
            embs = np.asarray(embs, np.float32).reshape(vs.shape[0], -1)
            # a vertex put twice in one call: the last write wins (store.py:64, dict assignment)
            last = vs.shape[0] - 1 - np.unique(vs[::-1], return_index=True)[1]
            if last.shape[0] != vs.shape[0]:
                last.sort()
                vs, embs = vs[last], embs[last]
            slots = np.array([self._slot_of(int(v)) for v in vs], np.int64)
            stg = 1 - self._cur
            idx = torch.as_tensor(slots, device=self.device)
            newly = int((self._stamp[stg][idx] != self._stage_stamp).sum().item())
            self._tab[stg][idx] = torch.as_tensor(embs, device=self.device)
            self._ver[stg][idx] = int(version)
            self._stamp[stg][idx] = self._stage_stamp
            self._staged += newly
            self.puts += n_calls

    def get(self, v: int, reading_batch: int):
        """store.py:67-98: the embedding staged for this super-batch, or None."""
        with self._lock:
            if not (self._window_start <= reading_batch < self._window_start + self._window_len):
                raise StoreContractError(f"read at batch {reading_batch} outside current super-batch window "
                                         f"[{self._window_start}, {self._window_start + self._window_len})")
            s = self._slot.get(int(v))
            if s is None or int(self._stamp[self._cur][s].item()) != self._cur_stamp:
                self.misses += 1
                return None
            gap = reading_batch - int(self._ver[self._cur][s].item())
            if gap > self.gap_bound:
                raise StalenessViolation(f"vertex {v}: version gap {gap} exceeds bound {self.gap_bound} "
                                         f"(read batch {reading_batch})")
            self.hits += 1
            if gap > self.max_observed_gap:
                self.max_observed_gap = gap
                self.max_gap_batch = reading_batch
                self.max_gap_super_batch = self.current_super_batch
            return self._tab[self._cur][s].double().cpu().numpy()

    def advance_super_batch(self, window_start: int | None = None, window_len: int | None = None) -> None:
        """store.py:100-118: promote staging; entries staged two super-batches ago die."""
        with self._lock:
            self._cur = 1 - self._cur
            self._cur_stamp = self._stage_stamp
            self._stamp_serial += 1
            self._stage_stamp = self._stamp_serial
            self._live_cur, self._staged = self._staged, 0
            self.current_super_batch += 1
            if window_start is None:
                window_start = self._window_start + self._window_len
            self._window_start = int(window_start)
            self._window_len = int(window_len) if window_len else self.n
            if self._window_len < 1 or self._window_len > self.n:
                raise StoreContractError(f"super-batch window length {self._window_len} outside [1, {self.n}]")

    def reset_epoch(self, window_start: int) -> None:
        """store.py:120-130."""
        with self._lock:
            self._stamp_serial += 2
            self._cur_stamp = self._stamp_serial - 1
            self._stage_stamp = self._stamp_serial
            self._live_cur = self._staged = 0
            self.current_super_batch = 0
            self._window_start = int(window_start)
            self._window_len = self.n

    def staged_count(self) -> int:
        with self._lock:
            return self._staged

    def live_entries(self) -> int:
        with self._lock:
            return self._live_cur + self._staged

    def memory_bytes(self) -> int:
        """store.py:140-142 accounting view (8-byte reals, as the reference)."""
        return self.live_entries() * self.emb_dim * 8

    def contains_current(self, v: int) -> bool:
        with self._lock:
            s = self._slot.get(int(v))
            return s is not None and int(self._stamp[self._cur][s].item()) == self._cur_stamp
