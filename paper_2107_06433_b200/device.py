"""Device residency: the corpus CSC and the embedding table live in HBM across calls.

The reference passes numpy arrays on every call (solver.py:106-112) and caches
only the CSC view on the corpus object (sparse.py:98-120).  On a GPU the
240 MB fp64 embedding table and the corpus would dominate every solve if
they crossed PCIe each time, so both are uploaded once and cached:

* ``DeviceCorpus.of(corpus)`` — cached on the corpus object (or, for a
  foreign corpus such as the reference's frozen ``CsrMatrix``, in a table
  keyed by object identity and dropped when the object dies);
* ``DeviceEmbeddings.of(E)`` — keyed by buffer identity (address, shape,
  strides, dtype) plus a content hash: every byte of a writeable table is
  hashed on each call (an in-place edit of one element is detected), a
  read-only table is sampled only (it cannot be edited).  torch CUDA tensors
  are used in place (keyed by their version counter).

HBM layout: CSC ``col_ptr`` int64 (N+1), ``rows`` int32 (nnz),
``vals`` f64 (nnz); a longest-column-first work order int32 (N); the list of
vocabulary rows that occur in the corpus int32; E f64 (V, w) row-major with
its row norms f64 (V).
"""

from __future__ import annotations

import os
import warnings
import weakref
import zlib

import numpy as np
import torch

from . import _lib

__all__ = ["DeviceCorpus", "DeviceEmbeddings", "device", "stream_ptr", "DeviceWorkspace"]


_CUDA_OK = False
_DEVICES: dict = {}


def cuda_ok() -> bool:
    """torch.cuda.is_available(), remembered once true (per-call cost matters
    on the per-query path)."""
    global _CUDA_OK
    if not _CUDA_OK:
        _CUDA_OK = torch.cuda.is_available()
    return _CUDA_OK


def device(index: int | None = None) -> torch.device:
    if not cuda_ok():
        raise _lib.NativeUnavailable("no CUDA device is visible; the B200 path has no CPU fallback")
    if index is None:
        index = torch.cuda.current_device()
    d = _DEVICES.get(index)
    if d is None:
        d = _DEVICES[index] = torch.device("cuda", index)
    return d


_RAW_STREAM = getattr(torch._C, "_cuda_getCurrentRawStream", None)


def stream_ptr(dev: torch.device | None = None) -> int:
    """cudaStream_t of the current stream on ``dev`` (the per-query path calls
    this every time: the raw accessor skips torch's Stream object)."""
    if _RAW_STREAM is not None and dev is not None and dev.index is not None:
        return int(_RAW_STREAM(dev.index))
    return torch.cuda.current_stream(dev).cuda_stream


_STAGE_BYTES = 32 << 20
_stage_bufs: list = []


def _h2d_staged(a: np.ndarray, dev: torch.device) -> torch.Tensor:
    """Upload of a large host array through two pinned 32 MB staging buffers:
    the threaded host copy into one buffer overlaps the DMA out of the other
    (pageable copies of a 240 MB embedding table run at a fraction of PCIe)."""
    with warnings.catch_warnings():
        warnings.simplefilter("ignore", UserWarning)
        host = torch.from_numpy(a)
    out = torch.empty(host.shape, dtype=host.dtype, device=dev)
    n = a.nbytes
    src = a.ctypes.data
    dst = out.view(-1).view(torch.uint8)
    if not _stage_bufs:
        _stage_bufs.extend(torch.empty(_STAGE_BYTES, dtype=torch.uint8, pin_memory=True)
                           for _ in range(2))
    stream = torch.cuda.current_stream(dev)
    pending = [None, None]
    threads = min(8, os.cpu_count() or 1)
    for k, off in enumerate(range(0, n, _STAGE_BYTES)):
        b = k % 2
        if pending[b] is not None:
            pending[b].synchronize()          # the DMA out of this buffer is done
        m = min(_STAGE_BYTES, n - off)
        _lib.call("swmd_host_copy", _stage_bufs[b].data_ptr(), src + off, m, threads)
        dst[off: off + m].copy_(_stage_bufs[b][:m], non_blocking=True)
        ev = torch.cuda.Event()
        ev.record(stream)
        pending[b] = ev
    stream.synchronize()
    return out


def _h2d(a: np.ndarray, dev: torch.device, dtype: torch.dtype | None = None) -> torch.Tensor:
    a = np.ascontiguousarray(a)
    if dtype is None and a.nbytes >= 4 * _STAGE_BYTES and _lib.lib_or_none() is not None:
        return _h2d_staged(a, dev)
    with warnings.catch_warnings():   # read-only host arrays: only read here
        warnings.simplefilter("ignore", UserWarning)
        t = torch.from_numpy(a)
    if dtype is not None:
        t = t.to(dtype)
    return t.to(dev, non_blocking=False)


class DeviceCorpus:
    """A corpus (or a contiguous column block of it) resident in HBM as CSC."""

    def __init__(self, n_rows: int, col_ptr: np.ndarray, rows: np.ndarray, vals: np.ndarray,
                 dev: torch.device, col_offset: int = 0, n_key: int | None = None,
                 pos: np.ndarray | None = None):
        self.n_rows = int(n_rows)
        self.n_cols = int(col_ptr.size - 1)
        self.nnz = int(col_ptr[-1] - col_ptr[0])
        self.col_offset = int(col_offset)
        self.n_key = int(n_key if n_key is not None else self.n_cols)
        self.device = dev
        base = int(col_ptr[0])
        cp = np.asarray(col_ptr, dtype=np.int64) - base
        self.col_ptr = _h2d(cp, dev)
        self.rows = _h2d(np.asarray(rows[base: base + self.nnz], dtype=np.int32), dev)
        self.vals = _h2d(np.asarray(vals[base: base + self.nnz], dtype=np.float64), dev)
        present = np.flatnonzero(np.bincount(np.asarray(rows[base: base + self.nnz]),
                                             minlength=self.n_rows) > 0).astype(np.int32)
        self._set_layout(cp, present)
        self._pos_host = pos
        self._pos = None

    HOT_ROWS = 256   # ranks kept in the hot-row index (a launch uses as many as fit its slab)

    def hot_index(self):
        """(hot_slot, hot_ids) of swmd_solve_hot_f64, built on the device at the
        first long-query solve: the corpus's most frequent vocabulary rows by
        nonzero count (ties to the lower row id), or (None, None) for an empty
        corpus."""
        hot = getattr(self, "_hot", None)
        if hot is None:
            if self.nnz == 0 or self.n_rows == 0:
                hot = (None, None)
            else:
                counts = torch.bincount(self.rows.to(torch.int64), minlength=self.n_rows)
                k = int(min(self.HOT_ROWS, self.n_rows))
                # stable: sort by (-count, row id)
                order = torch.argsort(counts, descending=True, stable=True)[:k]
                order = order[counts[order] > 0]
                ids = order.to(torch.int32).contiguous()
                slot = torch.full((self.n_rows,), -1, dtype=torch.int32, device=self.device)
                slot[order] = torch.arange(order.numel(), dtype=torch.int32, device=self.device)
                hot = (slot, ids) if ids.numel() else (None, None)
            self._hot = hot
        return hot

    def _set_layout(self, cp: np.ndarray, present: np.ndarray):
        lens = np.diff(cp)
        self.host_col_ptr = cp
        self.mean_len = float(self.nnz / max(1, self.n_cols))
        self.max_len = int(lens.max()) if lens.size else 0
        self.order = _h2d(claim_order(cp, self.device), self.device)
        self.n_present = int(present.size)
        self.present_rows = _h2d(present, self.device) if present.size else None

    @classmethod
    def from_csr(cls, n_rows: int, n_cols: int, row_ptr: np.ndarray, col_idx: np.ndarray,
                 values: np.ndarray, dev: torch.device) -> "DeviceCorpus":
        """Upload the CSR arrays and transpose them in HBM (swmd_csr_to_csc_f64).

        Replaces the host argsort of ``CsrMatrix.csc_index`` (sparse.py:98-120)
        for a corpus that arrives row-major: the CSC (rows ascending within a
        column, so identical to the host view) and the CSR position of every
        slot are built by the device; only ``col_ptr`` comes back to size the
        launch order.
        """
        rp = np.asarray(row_ptr, dtype=np.int64)
        nnz = int(rp[-1]) if rp.size else 0
        self = cls.__new__(cls)
        self.n_rows, self.n_cols, self.nnz = int(n_rows), int(n_cols), nnz
        self.col_offset, self.n_key, self.device = 0, int(n_cols), dev
        d_rp = _h2d(rp, dev)
        d_ci = _h2d(np.asarray(col_idx, dtype=np.int64), dev)
        d_v = _h2d(np.asarray(values, dtype=np.float64), dev)
        self.col_ptr = torch.empty(self.n_cols + 1, dtype=torch.int64, device=dev)
        self.rows = torch.empty(max(1, nnz), dtype=torch.int32, device=dev)[:nnz]
        self.vals = torch.empty(max(1, nnz), dtype=torch.float64, device=dev)[:nnz]
        pos = torch.empty(max(1, nnz), dtype=torch.int64, device=dev)[:nnz]
        sb = int(_lib.lib().swmd_csr_to_csc_scratch_bytes(self.n_cols))
        scratch = torch.empty(sb, dtype=torch.uint8, device=dev)
        longest = torch.zeros(1, dtype=torch.int32, device=dev)
        _lib.call("swmd_csr_to_csc_f64", d_rp.data_ptr(), d_ci.data_ptr(), d_v.data_ptr(),
                  self.n_rows, self.n_cols, nnz, self.col_ptr.data_ptr(), self.rows.data_ptr(),
                  self.vals.data_ptr(), pos.data_ptr(), scratch.data_ptr(), sb,
                  longest.data_ptr(), stream_ptr(dev))
        cp = self.col_ptr.cpu().numpy()
        if int(longest.item()) > 0:
            # the few columns longer than the warp sort handles: sort their
            # slots by CSR position on the device
            long_cols = np.flatnonzero(np.diff(cp) > 1024)
            for c in long_cols:
                b, e = int(cp[c]), int(cp[c + 1])
                perm = torch.argsort(pos[b:e], stable=True)
                pos[b:e] = pos[b:e][perm]
                self.rows[b:e] = self.rows[b:e][perm]
                self.vals[b:e] = self.vals[b:e][perm]
        present = np.flatnonzero(np.diff(rp) > 0).astype(np.int32)
        self._set_layout(cp, present)
        self._pos_host = None
        self._pos = pos
        return self

    @property
    def pos(self) -> torch.Tensor:
        """CSR storage position of every CSC slot (for the unfused sddmm/spmm)."""
        if self._pos is None:
            if self._pos_host is None:
                raise ValueError("CSR positions are not available for this corpus view")
            self._pos = _h2d(np.asarray(self._pos_host, dtype=np.int64), self.device)
        return self._pos

    # -- cache -------------------------------------------------------------------
    _foreign: dict[int, dict] = {}

    @classmethod
    def _store(cls, corpus) -> dict:
        """The per-corpus cache of resident copies: on the corpus object when it
        has a slot for it (this package's CsrMatrix), else keyed by id and
        dropped when the corpus is collected."""
        store = getattr(corpus, "_device_cache", None)
        if isinstance(store, dict):
            return store
        store = cls._foreign.get(id(corpus))
        if store is None:
            store = {}
            cls._foreign[id(corpus)] = store
            try:
                weakref.finalize(corpus, cls._foreign.pop, id(corpus), None)
            except TypeError:
                pass
        return store

    @classmethod
    def of(cls, corpus, dev: torch.device | None = None) -> "DeviceCorpus":
        dev = dev or device()
        key = (dev.type, dev.index)
        store = cls._store(corpus)
        dc = store.get(key)
        if dc is None and _row_major_only(corpus):
            dc = cls.from_csr(corpus.n_rows, corpus.n_cols, corpus.row_ptr, corpus.col_idx,
                              corpus.values, dev)
            store[key] = dc
        if dc is None:
            if hasattr(corpus, "csc_compact"):
                cp, rows, vals = corpus.csc_compact()
                pos_host = corpus.csc_index()[2] if corpus._csc_cache is not None else None
            else:  # reference CsrMatrix: its own cached column view
                cp, rows, pos_host, vals = corpus.csc_index()
            dc = cls(corpus.n_rows, cp, rows, vals, dev, pos=pos_host)
            if pos_host is None and hasattr(corpus, "csc_index"):
                dc._pos_host_fn = corpus.csc_index
            store[key] = dc
        return dc

    @classmethod
    def block_of(cls, corpus, dev: torch.device, c0: int, c1: int) -> "DeviceCorpus":
        """Columns [c0, c1) of ``corpus`` resident on ``dev`` (a shard of the
        multi-GPU split), cached on the corpus like ``of``."""
        if (c0, c1) == (0, corpus.n_cols):
            return cls.of(corpus, dev)
        store = cls._store(corpus)
        key = (dev.type, dev.index, int(c0), int(c1))
        dc = store.get(key)
        if dc is None:
            if hasattr(corpus, "csc_compact"):
                cp, rows, vals = corpus.csc_compact()
            else:
                cp, rows, _, vals = corpus.csc_index()
            dc = cls(corpus.n_rows, cp[c0: c1 + 1], rows, vals, dev, col_offset=c0,
                     n_key=corpus.n_cols)
            store[key] = dc
        return dc

    def compact_rows(self, de) -> "tuple[torch.Tensor, int] | None":
        """The corpus's vocabulary rows of ``de`` as one contiguous f64 matrix
        (cached per embedding table): the TMA cost build streams it.  The
        table itself when every row occurs."""
        if de.dtype != torch.float64 or de.dim % 2 or de.ld % 2:
            return None
        cache = self.__dict__.setdefault("_compact", {})
        hit = cache.get(id(de))
        if hit is not None and hit[0] is de:
            return hit[1], hit[2]
        if self.present_rows is None or self.n_present >= self.n_rows:
            Ec, ld = de.E, de.ld             # every row occurs: the table itself
        else:
            Ec = de.E.index_select(0, self.present_rows.long())[:, : de.dim].contiguous()
            ld = int(Ec.stride(0))
        cache.clear()
        cache[id(de)] = (de, Ec, ld)
        return Ec, ld

    def ensure_pos(self):
        if self._pos_host is None and hasattr(self, "_pos_host_fn"):
            self._pos_host = self._pos_host_fn()[2]
        return self.pos

# the slot count the claim order is planned for: the persistent solve of a
# v_r <= 20 query (VRP 20, the BASELINE configs); other widths still get a
# valid (nearly longest-first) order
_PLAN_V_R = 19
SCHEDULE_MAX_RATIO = 8


def claim_order(col_ptr: np.ndarray, dev: torch.device) -> np.ndarray:
    """Column claim order of the persistent solve (swmd_schedule_order): a
    planned schedule for the resident warps of ``dev`` when a launch runs
    only a few columns per warp (the tail matters), longest-first otherwise."""
    import ctypes

    cp = np.ascontiguousarray(col_ptr, dtype=np.int64)
    n = cp.size - 1
    order = np.empty(max(n, 1), dtype=np.int32)[:n]
    if n == 0:
        return order
    lib = _lib.lib()
    slots = ctypes.c_int32(0)
    with torch.cuda.device(dev):
        _lib.call("swmd_solve_slots_f64", _PLAN_V_R, ctypes.byref(slots))
    rounds = int(lib.swmd_solve_reg_rounds_f64(_PLAN_V_R))
    _lib.call("swmd_schedule_order", cp.ctypes.data, n, int(slots.value), rounds, 48,
              SCHEDULE_MAX_RATIO, order.ctypes.data)
    return order


def _row_major_only(corpus) -> bool:
    """True for a corpus that holds only its CSR arrays (no column view has
    been built on the host yet): it is transposed on the device."""
    if getattr(corpus, "_csc_cache", None) is not None:
        return False
    if hasattr(corpus, "csc_compact"):
        return corpus._csc_compact is None and corpus._csr is not None
    return hasattr(corpus, "row_ptr") and hasattr(corpus, "col_idx")


def _read_only(a: np.ndarray) -> bool:
    """True when no numpy array can write ``a``'s buffer: ``a`` and every
    ndarray in its ``base`` chain are read-only (a read-only view of a
    writeable array is not enough)."""
    x = a
    while isinstance(x, np.ndarray):
        if x.flags.writeable:
            return False
        x = x.base
    return True


def _fingerprint(a: np.ndarray) -> int:
    """Content key of a host table for the resident cache.

    Read-only tables (``E.flags.writeable = False`` down the base chain)
    cannot be edited in place, so a sampled hash (64 strided elements + the
    last 16) guards only against a recycled address.  A writeable table is
    hashed in full on every call (``swmd_content_hash``, all host threads):
    any in-place edit, even one element, invalidates the device copy — the
    reference reads the table on every call, so must this path.  Callers that
    want the cheap path mark the table read-only or pass a CUDA tensor."""
    ro = _read_only(a)
    if a.flags.c_contiguous and a.size >= 16:
        lib = _lib.lib_or_none()
        if lib is not None:
            if ro:
                return int(lib.swmd_sample_crc(a.ctypes.data, a.size, a.itemsize))
            return int(lib.swmd_content_hash(a.ctypes.data, a.nbytes,
                                             min(8, os.cpu_count() or 1)))
    if ro:
        return _fingerprint_py(a)
    return zlib.crc32(np.ascontiguousarray(a).tobytes())


def _fingerprint_py(a: np.ndarray) -> int:
    """Sampled content check: 256 strided elements plus the last 16, CRC32."""
    flat = a.reshape(-1)
    step = max(1, flat.size // 256)
    return zlib.crc32(flat[::step].tobytes(), zlib.crc32(flat[-16:].tobytes()))


class DeviceEmbeddings:
    """An embedding table resident in HBM, row-major, with its row norms.

    float64 for the reference-precision path; float32 (rows padded to a
    multiple of 4 elements, 16-byte aligned) for the multi-query fp32 path.
    """

    _cache: dict = {}
    _last = None

    def __init__(self, E: torch.Tensor, dim: int | None = None):
        self.E = E
        self.V = int(E.shape[0])
        self.dim = int(dim if dim is not None else E.shape[1])
        self.ld = int(E.stride(0))
        self.dtype = E.dtype
        self._norms = None

    @property
    def norms(self) -> torch.Tensor:
        if self._norms is None:
            n = torch.empty(self.V, dtype=self.dtype, device=self.E.device)
            fn = "swmd_row_norms_f64" if self.dtype == torch.float64 else "swmd_row_norms_f32"
            _lib.call(fn, self.E.data_ptr(), self.V, self.dim, self.ld, n.data_ptr(),
                      stream_ptr(self.E.device))
            self._norms = n
        return self._norms

    @classmethod
    def of(cls, E, dev: torch.device | None = None,
           dtype: torch.dtype = torch.float64) -> "DeviceEmbeddings":
        if isinstance(E, torch.Tensor):
            if E.device.type != "cuda":
                E = E.detach().cpu().numpy()
            elif dtype == torch.float64:
                t = E.detach()
                if t.dtype != torch.float64:
                    t = t.double()
                if t.stride(-1) != 1:
                    t = t.contiguous()
                key = ("torch", t.data_ptr(), tuple(t.shape), t._version, dtype)
                de = cls._cache.get(key)
                if de is None:
                    de = cls(t)
                    cls._cache = {k: v for k, v in cls._cache.items() if k[0] != "torch"}
                    cls._cache[key] = de
                return de
            else:
                E = E.detach().cpu().numpy()
        dev = dev or device()
        arr = np.asarray(E)
        if arr.ndim != 2:
            raise ValueError(f"embeddings must be 2-D, got shape {arr.shape}")
        last = cls._last
        if (last is not None and last[0] is arr and last[1] == arr.shape and last[2] is dev
                and last[3] == dtype and last[4] == _fingerprint(arr)):
            return last[5]            # the same live array object, content unchanged
        key = ("numpy", dev.index, arr.__array_interface__["data"][0], arr.shape,
               arr.strides, arr.dtype.str, _fingerprint(arr), dtype)
        de = cls._cache.get(key)
        if de is None:
            if dtype == torch.float64:
                host = np.ascontiguousarray(arr, dtype=np.float64)
                de = cls(_h2d(host, dev))
            else:
                V, dim = arr.shape
                ld = (dim + 3) // 4 * 4
                host = np.zeros((V, ld), dtype=np.float32)
                host[:, :dim] = arr
                de = cls(_h2d(host, dev), dim=dim)
            # keep one resident table per (device, precision): a new one evicts the old
            cls._cache = {k: v for k, v in cls._cache.items()
                          if k[0] == "torch" or k[-1] != dtype}
            cls._cache[key] = de
        # holding the array keeps its id from being reused while it is cached
        cls._last = (arr, arr.shape, dev, dtype, key[6], de)
        return de


class DeviceWorkspace:
    """Grow-only named device pools (the device twin of SinkhornWorkspace,
    solver.py:59-81)."""

    def __init__(self, dev: torch.device):
        self.device = dev
        self._pools: dict[tuple[str, torch.dtype], torch.Tensor] = {}

    def flat(self, name: str, n: int, dtype=torch.float64) -> torch.Tensor:
        key = (name, dtype)
        p = self._pools.get(key)
        if p is None or p.numel() < n:
            p = torch.empty(max(n, 1), dtype=dtype, device=self.device)
            self._pools[key] = p
        return p[:n]

    def matrix(self, name: str, rows: int, cols: int, dtype=torch.float64) -> torch.Tensor:
        return self.flat(name, rows * cols, dtype).view(rows, cols)
