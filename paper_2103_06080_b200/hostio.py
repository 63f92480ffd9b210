"""Device -> host transfers of fields (results and snapshots of a march).

* ``to_host64`` copies a device field into a fresh ordinary (pageable)
  float64 numpy array through two reusable 32 MB page-locked staging chunks:
  the DMA of chunk i+1 overlaps the host copy (and fp32 -> fp64 widening) of
  chunk i, so a 287 MB C2 field comes back at DMA speed while the process pins
  only 64 MB, whatever the number or size of the results the caller keeps.
* ``SnapshotStreamer`` implements the reference's snapshots
  (``nwave/exprk.py:208-216,301-302``: v_n at the start of step n, kept on the
  host) without holding them on the device: a ring of two device buffers, each
  filled by a c2r of the state on the plan stream and drained to host memory
  by a worker thread on its own copy stream while the march continues.  Device
  memory is two fields, independent of the snapshot count.
"""

from __future__ import annotations

import os
import threading
from concurrent.futures import ThreadPoolExecutor

import numpy as np

STAGE_BYTES = 32 << 20

# host-side copies of a staging chunk run on a few threads: np.copyto releases
# the GIL, and a fresh destination's first-touch page faults then proceed in
# parallel (C2 field, 287 MB into np.empty: ~50 ms serial, ~16 ms on 8 threads)
_COPY_THREADS = max(1, min(8, os.cpu_count() or 1))
_pool = None
_pool_lock = threading.Lock()


def par_copyto(dst: np.ndarray, src: np.ndarray) -> None:
    """np.copyto(dst, src, casting="unsafe") for 1-D arrays, split over threads."""
    global _pool
    n = dst.size
    if _COPY_THREADS == 1 or n < (1 << 18):
        np.copyto(dst, src, casting="unsafe")
        return
    with _pool_lock:
        if _pool is None:
            _pool = ThreadPoolExecutor(_COPY_THREADS, thread_name_prefix="nwb-copy")
    step = (n + _COPY_THREADS - 1) // _COPY_THREADS
    futs = [_pool.submit(np.copyto, dst[a:a + step], src[a:a + step], casting="unsafe")
            for a in range(0, n, step)]
    for f in futs:
        f.result()

_free_pairs: dict = {}  # device index -> list of idle staging pairs
_staging_lock = threading.Lock()


def _torch():
    import torch

    return torch


def _acquire_pair(dev: int):
    """An idle pair of page-locked STAGE_BYTES chunks for device ``dev``
    (allocated on first need; as many exist as copies ever ran at once)."""
    torch = _torch()
    with _staging_lock:
        idle = _free_pairs.setdefault(dev, [])
        if idle:
            return idle.pop()
    return [torch.empty(STAGE_BYTES, dtype=torch.uint8, pin_memory=True) for _ in range(2)]


def _release_pair(dev: int, pair):
    with _staging_lock:
        _free_pairs.setdefault(dev, []).append(pair)


def copy_to_host(src, out: np.ndarray, stream=None) -> np.ndarray:
    """Copy device tensor ``src`` into numpy ``out`` (same element count; dtype
    widened on the host) through a staging pair, on ``stream`` (default: the
    current stream), after the work already queued there.  Each copy holds
    its own pair for its duration, so concurrent copies (studies run several
    marches at once; snapshot drains run beside the march) never share one."""
    torch = _torch()
    flat = src.reshape(-1)
    dst = out.reshape(-1)
    if flat.numel() != dst.size:
        raise ValueError("copy_to_host: element counts differ")
    stream = stream or torch.cuda.current_stream(src.device)
    per = STAGE_BYTES // flat.element_size()
    bufs = _acquire_pair(src.device.index)
    try:
        views = [b.view(flat.dtype) for b in bufs]
        pending = []  # (event, k, start, end)
        with torch.cuda.stream(stream):
            for i, s in enumerate(range(0, flat.numel(), per)):
                e, k = min(flat.numel(), s + per), i & 1
                if len(pending) == 2:  # buffer k is still held by chunk i-2: drain it
                    ev, kk, s0, e0 = pending.pop(0)
                    ev.synchronize()
                    par_copyto(dst[s0:e0], views[kk][: e0 - s0].numpy())
                views[k][: e - s].copy_(flat[s:e], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(stream)
                pending.append((ev, k, s, e))
            for ev, kk, s0, e0 in pending:
                ev.synchronize()
                par_copyto(dst[s0:e0], views[kk][: e0 - s0].numpy())
    finally:
        _release_pair(src.device.index, bufs)
    return out


def to_host64(src, stream=None) -> np.ndarray:
    """Device field -> fresh float64 numpy array (ordinary host memory)."""
    out = np.empty(tuple(src.shape), dtype=np.float64)
    return copy_to_host(src, out, stream)


class SnapshotStreamer:
    """Ring of two device snapshot buffers drained to host by a worker thread."""

    def __init__(self, plan):
        torch = _torch()
        self.plan = plan
        self.slots = []
        self.free = [threading.Event(), threading.Event()]
        for f in self.free:
            f.set()
        self.copy_stream = torch.cuda.Stream(device=plan.device)
        self.results: dict = {}
        self.errors: list = []
        self._threads: list = []
        self._n = 0

    def capture(self, key):
        """Snapshot the plan's current state (v at the start of the next step)."""
        torch = _torch()
        k = self._n & 1
        self._n += 1
        self.free[k].wait()  # the slot's previous drain has finished
        if self.errors:
            raise self.errors[0]
        if len(self.slots) <= k:
            self.slots.append(torch.empty((self.plan.batch, self.plan.n_rho, self.plan.n_theta),
                                          dtype=self.plan.rdt, device=self.plan.device))
        slot = self.slots[k]
        self.plan.store_physical_into(slot)
        ready = torch.cuda.Event()
        ready.record(self.plan.stream)
        self.free[k].clear()
        th = threading.Thread(target=self._drain, args=(k, slot, ready, key), daemon=True)
        th.start()
        self._threads.append(th)

    def _drain(self, k, slot, ready, key):
        torch = _torch()
        try:
            with torch.cuda.device(self.plan.device):
                self.copy_stream.wait_event(ready)
                out = np.empty(tuple(slot.shape), dtype=np.float64)
                copy_to_host(slot, out, self.copy_stream)
                self.results[key] = out
        except BaseException as exc:  # surfaced by capture() / finish()
            self.errors.append(exc)
        finally:
            self.free[k].set()

    def finish(self) -> dict:
        for th in self._threads:
            th.join()
        if self.errors:
            raise self.errors[0]
        return self.results
