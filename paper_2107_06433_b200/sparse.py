"""Host-side sparse containers: the boundary types of the drop-in.

Same public names and semantics as the reference's ``sinkwmd.sparse``
(sparse.py:15-276): an immutable vocabulary-by-document ``CsrMatrix`` with a
lazily cached column-major view, the query ``SparseVector``, and the
partition helpers.  Differences that matter to the device path:

* ``CsrMatrix.from_csc`` builds the matrix straight from CSC arrays (the
  layout the kernels consume, and what the synthetic generator emits); the
  CSR arrays are then derived lazily, only if a caller asks for them;
* the column view is cached exactly like the reference's ``_csc_cache``
  (sparse.py:98-120), and the device upload is cached next to it
  (``device.DeviceCorpus``).

Any object with the reference's attributes (``n_rows``, ``n_cols``,
``row_ptr``, ``col_idx``, ``values``, ``csc_index()``) — in particular a
reference ``sinkwmd.CsrMatrix`` — is accepted wherever a corpus is expected.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Iterable, Sequence

import numpy as np

__all__ = [
    "StructuralError",
    "SparseVector",
    "CsrMatrix",
    "NnzPartition",
    "csr_from_triplets",
    "csr_validate",
    "nnz_partition",
    "partitions_to_arrays",
    "column_blocks",
]


class StructuralError(ValueError):
    """Input data violates a container's structural contract (sparse.py:15)."""


def _readonly(a, dtype) -> np.ndarray:
    out = np.array(a, dtype=dtype, copy=True, order="C")
    out.flags.writeable = False
    return out


def _readonly_view(a: np.ndarray, dtype) -> np.ndarray:
    """Read-only C-contiguous array of ``dtype``; copies only when it must."""
    a = np.asarray(a)
    if a.dtype != dtype or not a.flags.c_contiguous or a.flags.writeable:
        a = np.array(a, dtype=dtype, copy=True, order="C")
    a.flags.writeable = False
    return a


class SparseVector:
    """Strictly positive sparse vector (query histograms); sparse.py:27-60."""

    __slots__ = ("length", "indices", "values")

    def __init__(self, length: int, indices, values):
        idx = _readonly(indices, np.int64)
        val = _readonly(values, np.float64)
        if idx.ndim != 1 or idx.shape != val.shape:
            raise StructuralError("indices and values must be 1-D and equally long")
        if idx.size:
            if idx[0] < 0 or idx[-1] >= length:
                raise StructuralError("indices out of range")
            if np.any(idx[1:] <= idx[:-1]):
                raise StructuralError("indices must be strictly increasing")
            if np.any(val <= 0.0):
                raise StructuralError("values must be strictly positive")
        object.__setattr__(self, "length", int(length))
        object.__setattr__(self, "indices", idx)
        object.__setattr__(self, "values", val)

    def __setattr__(self, name, value):
        raise AttributeError("SparseVector is immutable")

    def __repr__(self) -> str:
        return f"SparseVector(length={self.length}, nnz={self.nnz})"

    @property
    def nnz(self) -> int:
        return int(self.indices.size)

    def to_dense(self) -> np.ndarray:
        d = np.zeros(self.length, dtype=np.float64)
        d[self.indices] = self.values
        return d


class CsrMatrix:
    """Immutable vocabulary x document matrix; sparse.py:63-133.

    Construct from CSR arrays (``CsrMatrix(n_rows, n_cols, row_ptr, col_idx,
    values)``, columns strictly increasing per row) or from CSC arrays with
    ``CsrMatrix.from_csc`` (rows strictly increasing per column).
    """

    def __init__(self, n_rows: int, n_cols: int, row_ptr=None, col_idx=None, values=None,
                 _csc_cache: tuple | None = None):
        self.__dict__["n_rows"] = int(n_rows)
        self.__dict__["n_cols"] = int(n_cols)
        self.__dict__["_csr"] = None
        self.__dict__["_csc_cache"] = None
        self.__dict__["_csc_compact"] = None   # (col_ptr i64, rows i32, vals f64)
        self.__dict__["_device_cache"] = {}
        if row_ptr is not None:
            self.__dict__["_csr"] = (_readonly(row_ptr, np.int64), _readonly(col_idx, np.int64),
                                     _readonly(values, np.float64))
        if _csc_cache is not None:
            self.__dict__["_csc_cache"] = _csc_cache

    @classmethod
    def from_csc(cls, n_rows: int, n_cols: int, col_ptr, rows, values) -> "CsrMatrix":
        m = cls(n_rows, n_cols)
        cp = _readonly_view(col_ptr, np.int64)
        rw = _readonly_view(rows, np.int32)
        vl = _readonly_view(values, np.float64)
        if cp.size != n_cols + 1 or rw.size != vl.size or int(cp[-1]) != rw.size:
            raise StructuralError("inconsistent CSC arrays")
        m.__dict__["_csc_compact"] = (cp, rw, vl)
        return m

    def __setattr__(self, name, value):
        raise AttributeError("CsrMatrix is immutable")

    def __repr__(self) -> str:
        return f"CsrMatrix(n_rows={self.n_rows}, n_cols={self.n_cols}, nnz={self.nnz})"

    # -- CSR view (derived on demand when built from CSC) ----------------------
    def _csr_arrays(self):
        if self._csr is None:
            cp, rw, vl = self._csc_compact
            cols = np.repeat(np.arange(self.n_cols, dtype=np.int64), np.diff(cp))
            perm = np.argsort(rw, kind="stable")      # stable keeps columns ascending
            row_ptr = np.zeros(self.n_rows + 1, dtype=np.int64)
            np.cumsum(np.bincount(rw, minlength=self.n_rows), out=row_ptr[1:])
            self.__dict__["_csr"] = (_readonly(row_ptr, np.int64), _readonly(cols[perm], np.int64),
                                     _readonly(vl[perm], np.float64))
            # CSR position of every CSC slot: inverse permutation
            if self._csc_cache is None:
                pos = np.empty_like(perm)
                pos[perm] = np.arange(perm.size, dtype=np.int64)
                pos.flags.writeable = False
                self.__dict__["_csc_cache"] = (cp, _readonly(rw, np.int64), pos, vl)
        return self._csr

    @property
    def row_ptr(self) -> np.ndarray:
        return self._csr_arrays()[0]

    @property
    def col_idx(self) -> np.ndarray:
        return self._csr_arrays()[1]

    @property
    def values(self) -> np.ndarray:
        return self._csr_arrays()[2]

    @property
    def nnz(self) -> int:
        if self._csc_compact is not None:
            return int(self._csc_compact[1].size)
        return int(self._csr[1].size)

    @property
    def shape(self) -> tuple[int, int]:
        return (self.n_rows, self.n_cols)

    def row_of_nnz(self) -> np.ndarray:
        return np.repeat(np.arange(self.n_rows, dtype=np.int64), np.diff(self.row_ptr))

    def csc_index(self) -> tuple[np.ndarray, np.ndarray, np.ndarray, np.ndarray]:
        """``(col_ptr, rows, pos, values)``: the column-major view (sparse.py:98-120).

        Rows ascend within a column; ``pos`` maps each column slot to its CSR
        position.  Cached after the first call.
        """
        if self._csc_cache is None:
            if self._csc_compact is not None:
                self._csr_arrays()
            else:
                row_ptr, col_idx, values = self._csr
                perm = np.argsort(col_idx, kind="stable")
                col_ptr = np.zeros(self.n_cols + 1, dtype=np.int64)
                np.cumsum(np.bincount(col_idx, minlength=self.n_cols), out=col_ptr[1:])
                rows = np.repeat(np.arange(self.n_rows, dtype=np.int64), np.diff(row_ptr))[perm]
                self.__dict__["_csc_cache"] = (_readonly(col_ptr, np.int64),
                                               _readonly(rows, np.int64),
                                               _readonly(perm, np.int64),
                                               _readonly(values[perm], np.float64))
        return self._csc_cache

    def csc_compact(self) -> tuple[np.ndarray, np.ndarray, np.ndarray]:
        """``(col_ptr int64, rows int32, values f64)`` — the device upload layout."""
        if self._csc_compact is None:
            cp, rows, _, vals = self.csc_index()
            self.__dict__["_csc_compact"] = (cp, _readonly(rows, np.int32), vals)
        return self._csc_compact

    def to_triplets(self) -> list[tuple[int, int, float]]:
        return [(int(i), int(j), float(v))
                for i, j, v in zip(self.row_of_nnz(), self.col_idx, self.values)]

    def to_dense(self) -> np.ndarray:
        d = np.zeros((self.n_rows, self.n_cols), dtype=np.float64)
        d[self.row_of_nnz(), self.col_idx] = self.values
        return d


@dataclass(frozen=True)
class NnzPartition:
    """A worker's contiguous nonzero range (sparse.py:136-151)."""

    worker_id: int
    nnz_begin: int
    nnz_end: int
    start_row: int

    @property
    def size(self) -> int:
        return self.nnz_end - self.nnz_begin


def csr_from_triplets(entries: Iterable[tuple[int, int, float]], n_rows: int,
                      n_cols: int) -> CsrMatrix:
    """CSR from (row, col, value) triplets; duplicates summed, zero sums dropped
    (sparse.py:154-188)."""
    trip = list(entries)
    if not trip:
        return CsrMatrix(n_rows, n_cols, np.zeros(n_rows + 1, np.int64),
                         np.zeros(0, np.int64), np.zeros(0))
    arr_r = np.array([t[0] for t in trip], dtype=np.int64)
    arr_c = np.array([t[1] for t in trip], dtype=np.int64)
    arr_v = np.array([t[2] for t in trip], dtype=np.float64)
    oob = (arr_r < 0) | (arr_r >= n_rows) | (arr_c < 0) | (arr_c >= n_cols)
    if oob.any():
        k = int(np.argmax(oob))
        raise StructuralError(
            f"triplet out of bounds: ({arr_r[k]}, {arr_c[k]}, {arr_v[k]}) "
            f"for shape ({n_rows}, {n_cols})")
    key = arr_r * n_cols + arr_c
    order = np.argsort(key, kind="stable")
    key, arr_v = key[order], arr_v[order]
    uniq, first = np.unique(key, return_index=True)
    sums = np.add.reduceat(arr_v, first)
    nz = sums != 0.0
    uniq, sums = uniq[nz], sums[nz]
    r, c = np.divmod(uniq, n_cols)
    row_ptr = np.zeros(n_rows + 1, dtype=np.int64)
    np.cumsum(np.bincount(r, minlength=n_rows), out=row_ptr[1:])
    return CsrMatrix(n_rows, n_cols, row_ptr, c, sums)


def csr_validate(m) -> list[str]:
    """All CSR structural violations as messages (sparse.py:191-223)."""
    out: list[str] = []
    rp, ci, vals = np.asarray(m.row_ptr), np.asarray(m.col_idx), np.asarray(m.values)
    if rp.size != m.n_rows + 1:
        return [f"row_ptr length {rp.size} != n_rows + 1 = {m.n_rows + 1}"]
    if rp[0] != 0:
        out.append(f"row_ptr[0] == {rp[0]}, expected 0")
    bad_rows = np.flatnonzero(rp[1:] < rp[:-1])
    out.extend(f"row_ptr non-decreasing at row {int(r)}" for r in bad_rows)
    if rp[-1] != ci.size:
        out.append(f"row_ptr[n_rows] == {rp[-1]}, expected nnz == {ci.size}")
    if ci.size != vals.size:
        out.append(f"col_idx length {ci.size} != values length {vals.size}")
    if bad_rows.size == 0 and rp[-1] == ci.size == vals.size:
        for r in range(m.n_rows):
            seg = ci[rp[r]:rp[r + 1]]
            if seg.size == 0:
                continue
            if seg.min() < 0 or seg.max() >= m.n_cols:
                out.append(f"col_idx out of range in row {r}")
            if np.any(seg[1:] <= seg[:-1]):
                out.append(f"col_idx strictly increasing violated in row {r}")
        neg = np.flatnonzero(vals < 0.0)
        if neg.size:
            out.append(f"negative value at nonzero {int(neg[0])}")
    return out


def nnz_partition(row_ptr, nnz: int, p: int) -> list[NnzPartition]:
    """``p`` contiguous nonzero ranges, sizes within one (sparse.py:226-246)."""
    if p < 1:
        raise ValueError(f"worker count must be >= 1, got {p}")
    rp = np.asarray(row_ptr, dtype=np.int64)
    q, rem = divmod(int(nnz), p)
    sizes = np.array([q + (1 if w < rem else 0) for w in range(p)], dtype=np.int64)
    edges = np.concatenate(([0], np.cumsum(sizes)))
    starts = np.searchsorted(rp, edges[:-1], side="right") - 1
    return [NnzPartition(w, int(edges[w]), int(edges[w + 1]), int(starts[w])) for w in range(p)]


def partitions_to_arrays(parts: Sequence[NnzPartition]) -> tuple[np.ndarray, np.ndarray]:
    """(bounds, start_rows) kernel inputs of a partition list (sparse.py:249-258)."""
    bounds = np.zeros(len(parts) + 1, dtype=np.int64)
    starts = np.zeros(len(parts), dtype=np.int64)
    for k, part in enumerate(parts):
        if part.nnz_begin != bounds[k]:
            raise ValueError("partitions must be contiguous and ordered")
        bounds[k + 1] = part.nnz_end
        starts[k] = part.start_row
    return bounds, starts


def column_blocks(col_ptr, p: int) -> np.ndarray:
    """``p + 1`` nnz-balanced column boundaries that never split a column
    (sparse.py:261-276).  Also the multi-GPU shard split."""
    if p < 1:
        raise ValueError(f"worker count must be >= 1, got {p}")
    cp = np.asarray(col_ptr, dtype=np.int64)
    n_cols, total = cp.size - 1, int(cp[-1])
    cuts = np.searchsorted(cp, (np.arange(1, p, dtype=np.int64) * total) // p, side="left")
    b = np.concatenate(([0], cuts, [n_cols])).astype(np.int64)
    return np.maximum.accumulate(b)
