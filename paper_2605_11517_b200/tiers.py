"""Host and storage tiers of the feature rows the streaming engine reads
(SSO: PAPER.md:611-621; the ledger's gpu_host / gpu_storage / host_storage
links, hierarchy.py:519-583).

A *row source* hands the streaming engine page-locked host views of feature
row ranges, ready for a DMA to HBM:

* ``HostRows`` — the features live in host memory (the dataset's fp32 array,
  page-locked in place, or a padded pinned copy);
* ``FileRows`` — the features live in a tier file on NVMe (the GRIN feature
  format, ``formats.write_features``); rows in a host-cache window are read
  once into pinned memory, every other range is read per pass with direct
  (page-cache bypassing) I/O into a ring of pinned bounce buffers by a
  reader thread that runs ahead of the GPU, so storage reads, the host link
  and the kernels overlap.  The node has no GPUDirect Storage, so the
  bounce buffer *is* the GPU<->storage bypass: NVMe DMA into the buffer the
  copy engine reads (no page-cache copy).

Protocol (one pass = one sweep over the engine's row chunks):
``begin_pass(ranges)`` with the ranges the pass will ``acquire`` in order;
``acquire(r0, r1) -> (host_view, token)``; after the H2D copy from the view
is enqueued, ``release(token, event)`` with a CUDA event recorded after it;
``end_pass()``.
"""

from __future__ import annotations

import queue
import threading

import numpy as np
import torch

from . import _lib

__all__ = ["FileRows", "HostRows", "file_backing"]


class HostRows:
    """Feature rows in (page-locked) host memory."""

    def __init__(self, host: torch.Tensor):
        self.host = host
        self.n_rows, self.width = host.shape
        self.storage_bytes = 0

    def configure(self, first_row: int) -> None:
        pass

    def describe(self) -> str:
        return "the rest page-locked in host memory"

    def begin_pass(self, ranges) -> None:
        pass

    def acquire(self, r0: int, r1: int):
        return self.host[r0:r1], None

    def release(self, token, event) -> None:
        pass

    def end_pass(self) -> None:
        pass


def file_backing(arr: np.ndarray):
    """(path, byte offset of arr[0, 0]) when ``arr`` is a C-contiguous view
    of a memory-mapped file, else None."""
    if not arr.flags.c_contiguous:
        return None
    base = arr
    while base is not None and not isinstance(base, np.memmap):
        base = base.base if isinstance(base, np.ndarray) else None
    if base is None or getattr(base, "filename", None) is None:
        return None
    off = arr.__array_interface__["data"][0] - base.__array_interface__["data"][0]
    return str(base.filename), int(base.offset) + int(off)


class FileRows:
    """Feature rows in a tier file (NVMe), with a pinned host-cache window.

    ``data_offset`` is the byte offset of row 0 in the file; rows are
    ``width`` fp32 values (width % 4 == 0, so every row range is 16-byte
    aligned for the copy engine).  ``host_rows`` rows after the first row
    the engine asks for (``configure``) are cached in pinned memory."""

    SLOTS = 3

    def __init__(self, path: str, data_offset: int, n_rows: int, width: int, chunk_rows: int,
                 host_cache_bytes: int = 0, threads: int = 16):
        if width % 4:
            raise ValueError("file-backed feature rows need width % 4 == 0")
        L = _lib.lib()
        self.align = int(L.grd_direct_alignment())
        fd = np.zeros(1, np.int32)
        direct = np.zeros(1, np.int32)
        _lib.check(L.grd_direct_open(str(path).encode(), 0, 0, _lib.ptr(fd), _lib.ptr(direct)),
                   "direct_open")
        self.fd, self.direct = int(fd[0]), bool(direct[0])
        self.path, self.data_offset = str(path), int(data_offset)
        self.n_rows, self.width = int(n_rows), int(width)
        self.row_bytes = 4 * self.width
        self.threads = int(threads)
        self.host_cache_rows = min(self.n_rows, int(host_cache_bytes) // self.row_bytes)
        self.host_lo = self.host_hi = 0
        self.host_cache = None
        self.host_valid = False
        span = int(chunk_rows) * self.row_bytes + 2 * self.align
        self.slots = []
        for _ in range(self.SLOTS):
            buf = torch.empty(span + self.align, dtype=torch.uint8, pin_memory=True)
            pad = (-buf.data_ptr()) % self.align
            self.slots.append(buf[pad: pad + span])
        self.slot_free = [threading.Event() for _ in range(self.SLOTS)]
        self.slot_event: list = [None] * self.SLOTS
        self.storage_bytes = 0          # bytes read from the file
        self._thread = None
        self._q: queue.Queue | None = None
        self._error = None

    def __del__(self):
        try:
            if self.fd >= 0:
                _lib.lib().grd_direct_close(self.fd)
                self.fd = -1
        except Exception:
            pass

    def describe(self) -> str:
        return (f"rows {self.host_lo}:{self.host_hi} in a pinned host cache, rows "
                f"{self.host_hi}:{self.n_rows} read per pass from {self.path} "
                f"({'O_DIRECT' if self.direct else 'buffered'} I/O, {self.threads} threads)")

    # -- reads ------------------------------------------------------------
    def _read_into(self, r0: int, r1: int, buf: torch.Tensor) -> int:
        """Read rows [r0, r1) (aligned superset) into ``buf``; returns the
        byte offset of row r0 inside it."""
        start = self.data_offset + r0 * self.row_bytes
        end = self.data_offset + r1 * self.row_bytes
        a0 = start // self.align * self.align
        a1 = -(-end // self.align) * self.align
        if a1 - a0 > buf.numel():
            raise ValueError("bounce buffer too small for the row range")
        _lib.check(_lib.lib().grd_direct_read(self.fd, a0, a1 - a0, buf.data_ptr(), self.threads),
                   "direct_read")
        self.storage_bytes += a1 - a0
        return start - a0

    def _view(self, buf: torch.Tensor, off: int, n: int) -> torch.Tensor:
        return buf[off: off + n * self.row_bytes].view(torch.float32).view(n, self.width)

    def configure(self, first_row: int) -> None:
        """Cache rows [first_row, first_row + host_cache_rows) in pinned memory
        (the rows before first_row are the engine's HBM cache)."""
        lo = int(first_row)
        hi = min(self.n_rows, lo + self.host_cache_rows)
        if (lo, hi) != (self.host_lo, self.host_hi):
            self.host_lo, self.host_hi = lo, hi
            self.host_cache = None
            self.host_valid = False

    def _fill_host_cache(self) -> None:
        n = self.host_hi - self.host_lo
        if n <= 0:
            self.host_valid = True
            return
        span = n * self.row_bytes + 2 * self.align
        raw = torch.empty(span + self.align, dtype=torch.uint8, pin_memory=True)
        pad = (-raw.data_ptr()) % self.align
        buf = raw[pad: pad + span]
        off = self._read_into(self.host_lo, self.host_hi, buf)
        self._host_raw = raw
        self.host_cache = self._view(buf, off, n)
        self.host_valid = True

    def _in_host(self, r0: int, r1: int) -> bool:
        return self.host_lo <= r0 and r1 <= self.host_hi and r1 > r0

    # -- pass protocol ----------------------------------------------------
    def begin_pass(self, ranges) -> None:
        file_ranges = [(r0, r1) for r0, r1 in ranges if not self._in_host(r0, r1)]
        if any(self._in_host(r0, r1) for r0, r1 in ranges) and not self.host_valid:
            self._fill_host_cache()
        self._q = queue.Queue()
        self._error = None
        for e in self.slot_free:
            e.set()
        self._thread = threading.Thread(target=self._reader, args=(file_ranges,), daemon=True)
        self._thread.start()

    def _reader(self, ranges) -> None:
        try:
            for k, (r0, r1) in enumerate(ranges):
                s = k % self.SLOTS
                self.slot_free[s].wait()
                self.slot_free[s].clear()
                if self.slot_event[s] is not None:
                    self.slot_event[s].synchronize()     # the H2D out of this slot is done
                off = self._read_into(r0, r1, self.slots[s])
                self._q.put((r0, r1, s, off))
        except BaseException as exc:    # surfaced by acquire()
            self._error = exc
            self._q.put(None)

    def acquire(self, r0: int, r1: int):
        if self._in_host(r0, r1):
            if not self.host_valid:
                self._fill_host_cache()
            return self.host_cache[r0 - self.host_lo: r1 - self.host_lo], None
        item = self._q.get()
        if item is None:
            raise self._error
        q0, q1, s, off = item
        if (q0, q1) != (r0, r1):
            raise RuntimeError(f"file tier out of order: got rows {q0}:{q1}, wanted {r0}:{r1}")
        return self._view(self.slots[s], off, r1 - r0), s

    def release(self, token, event) -> None:
        if token is None:
            return
        self.slot_event[token] = event
        self.slot_free[token].set()

    def end_pass(self) -> None:
        if self._thread is not None:
            self._thread.join()
            self._thread = None
        if self._error is not None:
            raise self._error
