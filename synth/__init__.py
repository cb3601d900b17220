"""Seeded synthetic workload generator — shared INPUT GENERATION only.

Holds none of the method's arithmetic: it produces ASCII query/target pairs (uppercase ACGT,
optionally N), their byte offsets, lengths and the per-pair initial score h0.  Both the CUDA
path (tests, bench.py) and the CPU oracle consume these arrays; neither imports the other.

The generator itself is native (``synth/synth.c``, SplitMix64 per-pair streams, pthreads) so
that the 1M-10M pair configs of BASELINE.json are produced in seconds.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None

#: BASELINE.json configs (1-based) -> default pair counts
CONFIG_PAIRS = {1: 1_000, 2: 1_000_000, 3: 500_000, 4: 100_000, 5: 10_000_000}


def _lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "libsynth.so")
        if not os.path.exists(path):
            raise RuntimeError(f"{path} missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
        lib = ctypes.CDLL(path)
        i64, i32p, i64p, u8p = ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p
        lib.synth_lengths.argtypes = [ctypes.c_int, ctypes.c_uint64, i64, i64, i64, ctypes.c_int,
                                      i32p, i32p, i32p, ctypes.c_int]
        lib.synth_bases.argtypes = [ctypes.c_int, ctypes.c_uint64, i64, i64, i64, ctypes.c_int,
                                    ctypes.c_double, i64p, i64p, u8p, u8p, ctypes.c_int]
        lib.synth_lengths_idx.argtypes = [ctypes.c_int, ctypes.c_uint64, i64p, i64, i64, ctypes.c_int,
                                          i32p, i32p, i32p, ctypes.c_int]
        lib.synth_bases_idx.argtypes = [ctypes.c_int, ctypes.c_uint64, i64p, i64, i64, ctypes.c_int,
                                        ctypes.c_double, i64p, i64p, u8p, u8p, ctypes.c_int]
        _LIB = lib
    return _LIB


def _ptr(a: np.ndarray) -> ctypes.c_void_p:
    return ctypes.c_void_p(a.ctypes.data)


@dataclass
class Batch:
    """A batch of pairs as flat ASCII buffers + offsets (pair k's query is
    ``q_ascii[q_off[k]:q_off[k+1]]``)."""

    q_ascii: np.ndarray  # uint8
    q_off: np.ndarray  # int64 [n+1]
    t_ascii: np.ndarray
    t_off: np.ndarray
    h0: np.ndarray  # int32 [n]

    @property
    def n(self) -> int:
        return len(self.q_off) - 1

    @property
    def qlen(self) -> np.ndarray:
        return np.diff(self.q_off).astype(np.int32)

    @property
    def tlen(self) -> np.ndarray:
        return np.diff(self.t_off).astype(np.int32)

    def cells(self) -> int:
        return int(np.dot(self.qlen.astype(np.int64), self.tlen.astype(np.int64)))

    def pair(self, k: int) -> tuple[bytes, bytes]:
        return (self.q_ascii[self.q_off[k]:self.q_off[k + 1]].tobytes(),
                self.t_ascii[self.t_off[k]:self.t_off[k + 1]].tobytes())

    def subset(self, idx) -> "Batch":
        return from_pairs([self.pair(int(k)) for k in idx], self.h0[np.asarray(idx)])


def shapes(cfg: int, n: int, seed: int | None = None, first: int = 0, n_total: int | None = None,
           grouped: bool = False, threads: int | None = None):
    """(qlen, tlen, h0) int32 arrays for pairs [first, first+n) without generating bases."""
    seed = cfg if seed is None else seed
    n_total = n if n_total is None else n_total
    q = np.empty(n, np.int32)
    t = np.empty(n, np.int32)
    h = np.empty(n, np.int32)
    _lib().synth_lengths(cfg, seed, first, n, n_total, int(grouped), _ptr(q), _ptr(t), _ptr(h),
                         threads or os.cpu_count() or 1)
    return q, t, h


def offsets(lens: np.ndarray) -> np.ndarray:
    off = np.zeros(len(lens) + 1, np.int64)
    np.cumsum(lens, out=off[1:])
    return off


def generate(cfg: int, n: int | None = None, seed: int | None = None, first: int = 0,
             n_total: int | None = None, grouped: bool = False, p_n: float = 0.0,
             threads: int | None = None, out=None) -> Batch:
    """Generate pairs [first, first+n) of config `cfg` (1..5) with `seed` (default: cfg id).

    `out`, if given, is a callable ``out(name, nbytes) -> np.ndarray[uint8]`` used to allocate
    the two ASCII buffers (e.g. views of pinned host memory)."""
    n = CONFIG_PAIRS[cfg] if n is None else n
    seed = cfg if seed is None else seed
    n_total = n if n_total is None else n_total
    ql, tl, h0 = shapes(cfg, n, seed, first, n_total, grouped, threads)
    qo, to = offsets(ql), offsets(tl)
    if out is None:
        qa = np.empty(int(qo[-1]), np.uint8)
        ta = np.empty(int(to[-1]), np.uint8)
    else:
        qa = out("q", int(qo[-1]))
        ta = out("t", int(to[-1]))
    _lib().synth_bases(cfg, seed, first, n, n_total, int(grouped), float(p_n), _ptr(qo), _ptr(to),
                       _ptr(qa), _ptr(ta), threads or os.cpu_count() or 1)
    return Batch(qa, qo, ta, to, h0)


def generate_idx(cfg: int, idx: np.ndarray, n_total: int, seed: int | None = None, grouped: bool = False,
                 p_n: float = 0.0, threads: int | None = None, out=None) -> Batch:
    """Pairs idx[0], idx[1], ... of the n_total-pair batch of config `cfg` (a rank's shard of a
    partitioned batch); identical to the same pairs of generate(cfg, n_total)."""
    idx = np.ascontiguousarray(idx, np.int64)
    n = len(idx)
    seed = cfg if seed is None else seed
    th = threads or os.cpu_count() or 1
    ql, tl, h0 = (np.empty(n, np.int32) for _ in range(3))
    _lib().synth_lengths_idx(cfg, seed, _ptr(idx), n, n_total, int(grouped), _ptr(ql), _ptr(tl), _ptr(h0), th)
    qo, to = offsets(ql), offsets(tl)
    qa = out("q", int(qo[-1])) if out else np.empty(int(qo[-1]), np.uint8)
    ta = out("t", int(to[-1])) if out else np.empty(int(to[-1]), np.uint8)
    _lib().synth_bases_idx(cfg, seed, _ptr(idx), n, n_total, int(grouped), float(p_n), _ptr(qo), _ptr(to),
                           _ptr(qa), _ptr(ta), th)
    return Batch(qa, qo, ta, to, h0)


def from_pairs(pairs, h0=None) -> Batch:
    """Build a Batch from an explicit list of (query, target) byte strings."""
    qs = [p[0].encode() if isinstance(p[0], str) else bytes(p[0]) for p in pairs]
    ts = [p[1].encode() if isinstance(p[1], str) else bytes(p[1]) for p in pairs]
    qo = offsets(np.array([len(x) for x in qs], np.int64))
    to = offsets(np.array([len(x) for x in ts], np.int64))
    qa = np.frombuffer(b"".join(qs), np.uint8).copy() if qs else np.empty(0, np.uint8)
    ta = np.frombuffer(b"".join(ts), np.uint8).copy() if ts else np.empty(0, np.uint8)
    if h0 is None:
        h0 = np.full(len(pairs), 20, np.int32)
    return Batch(qa, qo, ta, to, np.asarray(h0, np.int32).copy())


def random_pairs(n: int, lo: int, hi: int, seed: int, alphabet: bytes = b"ACGT", p_mut: float = 0.0,
                 tlo: int | None = None, thi: int | None = None) -> Batch:
    """Small randomized pair sets for parity tests (numpy Generator; independent lengths in
    [lo, hi]; with p_mut > 0 the target is a mutated copy of the query plus random flanks)."""
    rng = np.random.default_rng(seed)
    tlo = lo if tlo is None else tlo
    thi = hi if thi is None else thi
    al = np.frombuffer(alphabet, np.uint8)
    pairs = []
    for _ in range(n):
        ql = int(rng.integers(lo, hi + 1))
        q = al[rng.integers(0, len(al), ql)]
        if p_mut > 0:
            t = q.copy()
            m = rng.random(ql) < p_mut
            t[m] = al[rng.integers(0, len(al), int(m.sum()))]
            ops = rng.random(ql)
            keep = ops >= p_mut / 2
            t = t[keep]
            fl = int(rng.integers(0, max(1, ql // 2)))
            left = al[rng.integers(0, len(al), fl // 2)]
            right = al[rng.integers(0, len(al), fl - fl // 2)]
            t = np.concatenate([left, t, right])
            if len(t) == 0:
                t = al[rng.integers(0, len(al), 1)]
        else:
            tl = int(rng.integers(tlo, thi + 1))
            t = al[rng.integers(0, len(al), tl)]
        pairs.append((q.tobytes(), t.tobytes()))
    h0 = rng.integers(1, 40, n).astype(np.int32)
    return from_pairs(pairs, h0)
