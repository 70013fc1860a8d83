"""Seeded synthetic Sinkhorn-WMD instances shaped like the BASELINE.json configs.

The paper's datasets (crawl-300d-2M subset, dbpedia) are not
available, so every benchmark and parity case runs on seeded synthetic data
(SURVEY.md §8d):

* embeddings ``E ~ N(0,1)^{V x w}``, every row L2-normalised;
* documents: ``k`` unique word ids per document drawn Zipf(s) over ids
  ``0..V-1`` (id order is rank order), ``k`` uniform in ``[k_min, k_max]``,
  counts ``1 + Poisson(1)`` normalised to column sum 1, stored as CSC with
  rows ascending inside each column;
* query: ``v_r`` unique Zipf ids; weights uniform ``1/v_r`` (c1) or
  normalised ``1 + Poisson(1)`` counts (c2..c5).

The generator emits CSC directly (the layout the device path consumes) and
is vectorised in document chunks so the N=1M config builds in seconds.  The
reference's own ``synth.random_instance`` (``sinkwmd/synth.py:61-73``) draws
uniform words with a density and is not used for the Zipf configs.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np

__all__ = [
    "ZipfConfig",
    "CONFIGS",
    "ZipfInstance",
    "zipf_instance",
    "zipf_corpus_csc",
    "zipf_query",
    "normal_embeddings",
    "csc_to_csr",
]


@dataclass(frozen=True)
class ZipfConfig:
    """One BASELINE.json config (`configs[k]` is ``c{k+1}``)."""

    name: str
    n_vocab: int
    n_docs: int
    k_min: int
    k_max: int
    v_r: int | tuple[int, int]          # tuple = uniform range per query (c4)
    n_queries: int = 1
    dim: int = 300
    lam: float = 10.0
    max_iter: int = 15
    uniform_weights: bool = False
    dtype: str = "f64"
    zipf_s: float = 1.1
    seed: int = 0


CONFIGS: dict[str, ZipfConfig] = {
    "c1": ZipfConfig("c1", 10_000, 500, 20, 60, 20, uniform_weights=True, seed=1),
    "c2": ZipfConfig("c2", 100_000, 5_000, 10, 80, 19, seed=2),
    "c3": ZipfConfig("c3", 100_000, 1_000_000, 10, 80, 19, seed=3),
    "c4": ZipfConfig("c4", 100_000, 100_000, 10, 80, (8, 64), n_queries=64,
                     max_iter=20, dtype="f32", seed=4),
    "c5": ZipfConfig("c5", 200_000, 200_000, 50, 300, 256, seed=5),
}


@dataclass
class ZipfInstance:
    """CSC corpus (V x N), embeddings and one or more dense query histograms."""

    config: ZipfConfig
    embeddings: np.ndarray            # (V, w) float64 (or float32 for c4)
    col_ptr: np.ndarray               # (N+1,) int64
    rows: np.ndarray                  # (nnz,) int32, ascending within a column
    vals: np.ndarray                  # (nnz,) float64
    queries: list[np.ndarray] = field(default_factory=list)  # dense (V,) float64

    @property
    def n_vocab(self) -> int:
        return self.config.n_vocab

    @property
    def n_docs(self) -> int:
        return int(self.col_ptr.size - 1)

    @property
    def nnz(self) -> int:
        return int(self.rows.size)

    @property
    def query(self) -> np.ndarray:
        return self.queries[0]

    def corpus(self):
        """The corpus as this package's ``CsrMatrix`` with its CSC view pre-cached."""
        from .sparse import CsrMatrix

        return CsrMatrix.from_csc(self.n_vocab, self.n_docs, self.col_ptr,
                                  self.rows, self.vals)


class _Alias:
    """Walker alias table for the finite Zipf law P(id = k) ∝ (k + 1)^-s, k < V.

    O(1) vectorised sampling (one uniform per draw); the table construction
    is deterministic, so a seed fixes every draw.
    """

    def __init__(self, n_vocab: int, s: float):
        w = np.arange(1, n_vocab + 1, dtype=np.float64) ** (-s)
        p = w * (n_vocab / w.sum())
        prob = np.ones(n_vocab)
        alias = np.arange(n_vocab, dtype=np.int64)
        small = list(np.flatnonzero(p < 1.0)[::-1])
        large = list(np.flatnonzero(p >= 1.0)[::-1])
        while small and large:
            lo, hi = small.pop(), large.pop()
            prob[lo] = p[lo]
            alias[lo] = hi
            p[hi] = (p[hi] + p[lo]) - 1.0
            (small if p[hi] < 1.0 else large).append(hi)
        self.n = n_vocab
        self.prob = prob
        self.alias = alias

    def draw(self, rng: np.random.Generator, shape) -> np.ndarray:
        x = rng.random(shape) * self.n
        col = np.minimum(x.astype(np.int64), self.n - 1)
        frac = x - col
        return np.where(frac < self.prob[col], col, self.alias[col])


_ALIAS_CACHE: dict[tuple[int, float], _Alias] = {}


def _zipf_table(n_vocab: int, s: float) -> _Alias:
    key = (n_vocab, s)
    if key not in _ALIAS_CACHE:
        _ALIAS_CACHE[key] = _Alias(n_vocab, s)
    return _ALIAS_CACHE[key]


def _unique_draws(rng: np.random.Generator, table: _Alias, k: np.ndarray) -> np.ndarray:
    """For each entry of ``k``: the first ``k[d]`` distinct Zipf ids in draw order.

    Sequential sampling without replacement, implemented as "draw with
    replacement, keep first occurrences"; rows that come up short are
    redrawn with a larger candidate budget.  Returns an ``(n, max k)`` int64
    array whose row ``d`` holds its ids in draw order in the first ``k[d]``
    slots and ``-1`` after them.
    """
    n = k.size
    kmax_all = int(k.max()) if n else 0
    out = np.full((n, kmax_all), -1, dtype=np.int64)
    todo = np.arange(n)
    budget = int(max(8, 2 * kmax_all + 16))
    while todo.size:
        kk = k[todo]
        cand = table.draw(rng, (todo.size, budget))
        # sort (id, draw position) pairs; the first of each id run is its first draw
        key = np.sort(cand * budget + np.arange(budget)[None, :], axis=1)
        ids_sorted = key // budget
        first = np.ones(key.shape, dtype=bool)
        first[:, 1:] = ids_sorted[:, 1:] != ids_sorted[:, :-1]
        pos = np.where(first, key % budget, budget)
        pos.sort(axis=1)
        pos = pos[:, :kmax_all]
        short = pos[np.arange(todo.size), kk - 1] >= budget
        ok = np.flatnonzero(~short)
        if ok.size:
            p = pos[ok]
            keep = np.arange(kmax_all)[None, :] < kk[ok, None]
            ids = np.take_along_axis(cand[ok], np.minimum(p, budget - 1), axis=1)
            out[todo[ok]] = np.where(keep, ids, -1)
        todo = todo[short]
        budget *= 2
    return out


def normal_embeddings(rng: np.random.Generator, n_vocab: int, dim: int,
                      dtype=np.float64) -> np.ndarray:
    e = rng.standard_normal((n_vocab, dim))
    e /= np.linalg.norm(e, axis=1, keepdims=True)
    return np.ascontiguousarray(e.astype(dtype, copy=False))


def zipf_corpus_csc(rng: np.random.Generator, n_vocab: int, n_docs: int,
                    k_min: int, k_max: int, s: float = 1.1,
                    chunk: int = 25_000) -> tuple[np.ndarray, np.ndarray, np.ndarray]:
    """Column-normalised V x N corpus in CSC form (col_ptr int64, rows int32, vals f64)."""
    table = _zipf_table(n_vocab, s)
    k_max = min(k_max, n_vocab)
    k_min = min(k_min, k_max)
    lens = rng.integers(k_min, k_max + 1, size=n_docs)
    col_ptr = np.zeros(n_docs + 1, dtype=np.int64)
    np.cumsum(lens, out=col_ptr[1:])
    nnz = int(col_ptr[-1])
    rows = np.empty(nnz, dtype=np.int32)
    vals = np.empty(nnz, dtype=np.float64)
    starts = list(range(0, n_docs, chunk))
    # one child generator per chunk: the result is independent of how many
    # threads fill the chunks (numpy releases the GIL in the heavy kernels)
    children = rng.spawn(len(starts))

    def fill(ci: int) -> None:
        crng = children[ci]
        c0 = starts[ci]
        c1 = min(n_docs, c0 + chunk)
        k = lens[c0:c1]
        ids = _unique_draws(crng, table, k)                   # (n, kmax), -1 padded
        valid = ids >= 0
        counts = np.where(valid, 1.0 + crng.poisson(1.0, size=ids.shape), 0.0)
        counts /= counts.sum(axis=1, keepdims=True)
        key = np.where(valid, ids, n_vocab)                   # padding sorts last
        srt = np.argsort(key, axis=1, kind="stable")
        ids_s = np.take_along_axis(key, srt, axis=1)
        cnt_s = np.take_along_axis(counts, srt, axis=1)
        m = np.take_along_axis(valid, srt, axis=1)
        lo, hi = col_ptr[c0], col_ptr[c1]
        rows[lo:hi] = ids_s[m]
        vals[lo:hi] = cnt_s[m]

    workers = max(1, min(len(starts), os.cpu_count() or 1, 16))
    if workers == 1:
        for ci in range(len(starts)):
            fill(ci)
    else:
        with ThreadPoolExecutor(workers) as ex:
            list(ex.map(fill, range(len(starts))))
    return col_ptr, rows, vals


def zipf_query(rng: np.random.Generator, n_vocab: int, v_r: int,
               uniform: bool = False, s: float = 1.1) -> np.ndarray:
    """Dense normalised histogram with exactly ``v_r`` positive (Zipf-drawn) words."""
    table = _zipf_table(n_vocab, s)
    sel = _unique_draws(rng, table, np.array([min(v_r, n_vocab)]))[0]
    sel = sel[sel >= 0]
    if uniform:
        w = np.full(sel.size, 1.0)
    else:
        w = 1.0 + rng.poisson(1.0, size=sel.size).astype(np.float64)
    q = np.zeros(n_vocab, dtype=np.float64)
    q[sel] = w / w.sum()
    return q


def zipf_instance(cfg: ZipfConfig | str, seed: int | None = None,
                  n_docs: int | None = None) -> ZipfInstance:
    """Build the seeded instance for a config (``n_docs`` overrides N, same generator)."""
    if isinstance(cfg, str):
        cfg = CONFIGS[cfg]
    rng = np.random.default_rng(cfg.seed if seed is None else seed)
    edtype = np.float32 if cfg.dtype == "f32" else np.float64
    emb = normal_embeddings(rng, cfg.n_vocab, cfg.dim, edtype)
    nd = cfg.n_docs if n_docs is None else n_docs
    col_ptr, rows, vals = zipf_corpus_csc(rng, cfg.n_vocab, nd, cfg.k_min,
                                          cfg.k_max, cfg.zipf_s)
    queries = []
    for _ in range(cfg.n_queries):
        if isinstance(cfg.v_r, tuple):
            v_r = int(rng.integers(cfg.v_r[0], cfg.v_r[1] + 1))
        else:
            v_r = cfg.v_r
        queries.append(zipf_query(rng, cfg.n_vocab, v_r, cfg.uniform_weights, cfg.zipf_s))
    return ZipfInstance(cfg, emb, col_ptr, rows, vals, queries)


def csc_to_csr(n_rows: int, n_cols: int, col_ptr: np.ndarray, rows: np.ndarray,
               vals: np.ndarray) -> tuple[np.ndarray, np.ndarray, np.ndarray]:
    """CSR arrays (row_ptr, col_idx int64, values) of a CSC matrix; columns ascend per row."""
    cols = np.repeat(np.arange(n_cols, dtype=np.int64), np.diff(col_ptr))
    order = np.argsort(rows, kind="stable")      # stable: columns stay ascending
    row_ptr = np.zeros(n_rows + 1, dtype=np.int64)
    np.cumsum(np.bincount(rows, minlength=n_rows), out=row_ptr[1:])
    return row_ptr, cols[order], vals[order]
