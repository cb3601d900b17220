"""CPU oracle — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product path
(``paper_2301_09310_b200``) never imports, links or executes it, and the two share no code.

The arithmetic lives in ``oracle/oracle.c`` (plain full-matrix Gotoh, Eqs. 1-3,
P:132-149; the seed-anchored EXTEND reading of SURVEY §8(c)); this module only marshals
arguments through ctypes.
"""
from __future__ import annotations

import ctypes
import os
import time

import numpy as np

LOCAL, EXTEND = 0, 1
OK, EINVALID_BASE, EEMPTY, ETOO_LARGE, EBAD_H0 = 0, -1, -2, -3, -4

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None


def _lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "liboracle.so")
        if not os.path.exists(path):
            raise RuntimeError(f"{path} missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
        lib = ctypes.CDLL(path)
        p, i, i32, i64 = ctypes.c_void_p, ctypes.c_int, ctypes.c_int32, ctypes.c_int64
        one = [p, i, p, i, i32, i32, i32, i32, i, i32, p]
        lib.oracle_align_full.argtypes = one
        lib.oracle_align_rows.argtypes = one
        lib.oracle_tables.argtypes = [p, i, p, i, i32, i32, i32, i32, i, i32, p, p, p, p]
        lib.oracle_align_batch.argtypes = [p, p, p, p, p, i64, i32, i32, i32, i32, i, p, p, p, p, i, i]
        lib.oracle_align_banded.argtypes = [p, i, p, i, i32, i32, i32, i32, i, i32, i32, p]
        lib.oracle_banded_batch.argtypes = [p, p, p, p, p, p, i64, i32, i32, i32, i32, i, p, p, p, p, i]
        lib.oracle_start.argtypes = [p, i, p, i, i32, i32, i32, i32, p]
        lib.oracle_start_batch.argtypes = [p, p, p, p, i64, i32, i32, i32, i32, p, p, p, p, p, p, i]
        ksw = [p, i, p, i] + [i32] * 11 + [p]
        lib.oracle_ksw_extend.argtypes = ksw
        lib.oracle_ksw_table.argtypes = ksw + [p]
        lib.oracle_ksw_batch.argtypes = [p, p, p, p, p, i64, p, i32, p, p, i]
        lib.oracle_traceback.argtypes = [p, i, p, i, i32, i32, i32, i32, i32, i32, i32, i32, p, i, p]
        _LIB = lib
    return _LIB


def _b(s) -> bytes:
    return s.encode() if isinstance(s, str) else bytes(s)


def _buf(s: bytes):
    return ctypes.c_char_p(s) if s else ctypes.c_char_p(b"\0")


def align(q, t, match=1, mismatch=-4, alpha=7, beta=1, mode=LOCAL, h0=0, rows=False):
    """(score, q_end, t_end) of one pair, or raises ValueError with the oracle status."""
    q, t = _b(q), _b(t)
    out = (ctypes.c_int32 * 3)()
    fn = _lib().oracle_align_rows if rows else _lib().oracle_align_full
    st = fn(_buf(q), len(q), _buf(t), len(t), match, mismatch, alpha, beta, mode, h0, out)
    if st != OK:
        raise ValueError(st)
    return int(out[0]), int(out[1]), int(out[2])


def tables(q, t, match=1, mismatch=-4, alpha=7, beta=1, mode=LOCAL, h0=0):
    """Full H, E, F tables with the boundary: arrays of shape (m+1, n+1), index [i+1, j+1]."""
    q, t = _b(q), _b(t)
    n, m = len(q), len(t)
    H = np.zeros((m + 1, n + 1), np.int32)
    E = np.zeros_like(H)
    F = np.zeros_like(H)
    out = (ctypes.c_int32 * 3)()
    st = _lib().oracle_tables(_buf(q), n, _buf(t), m, match, mismatch, alpha, beta, mode, h0,
                              H.ctypes.data, E.ctypes.data, F.ctypes.data, out)
    if st != OK:
        raise ValueError(st)
    return H, E, F, (int(out[0]), int(out[1]), int(out[2]))


def align_batch(batch, match=1, mismatch=-4, alpha=7, beta=1, mode=LOCAL, threads=None, rows=False):
    """Oracle over a synth.Batch-like object (q_ascii, q_off, t_ascii, t_off, h0).

    Returns (score, q_end, t_end, status, threads_used) as numpy int32 arrays."""
    n = len(batch.q_off) - 1
    score = np.empty(n, np.int32)
    qe = np.empty(n, np.int32)
    te = np.empty(n, np.int32)
    st = np.empty(n, np.int32)
    threads = threads or os.cpu_count() or 1
    qa = np.ascontiguousarray(batch.q_ascii)
    ta = np.ascontiguousarray(batch.t_ascii)
    qo = np.ascontiguousarray(batch.q_off, np.int64)
    to = np.ascontiguousarray(batch.t_off, np.int64)
    h0 = np.ascontiguousarray(batch.h0, np.int32)
    used = _lib().oracle_align_batch(qa.ctypes.data, qo.ctypes.data, ta.ctypes.data, to.ctypes.data,
                                     h0.ctypes.data, n, match, mismatch, alpha, beta, mode,
                                     score.ctypes.data, qe.ctypes.data, te.ctypes.data, st.ctypes.data,
                                     threads, int(rows))
    return score, qe, te, st, used


def align_banded(q, t, w, match=1, mismatch=-4, alpha=7, beta=1, mode=LOCAL, h0=0):
    """(score, q_end, t_end) with only the cells |i - j| <= w in the table (oracle.c header)."""
    q, t = _b(q), _b(t)
    out = (ctypes.c_int32 * 3)()
    st = _lib().oracle_align_banded(_buf(q), len(q), _buf(t), len(t), match, mismatch, alpha, beta, mode, h0, w, out)
    if st != OK:
        raise ValueError(st)
    return int(out[0]), int(out[1]), int(out[2])


def banded_batch(batch, w, match=1, mismatch=-4, alpha=7, beta=1, mode=LOCAL, threads=None):
    """Banded oracle over a synth.Batch-like object; w: int32[n] bands.  (score, q_end, t_end, status)."""
    n = len(batch.q_off) - 1
    outs = [np.empty(n, np.int32) for _ in range(4)]
    threads = threads or os.cpu_count() or 1
    qa = np.ascontiguousarray(batch.q_ascii)
    ta = np.ascontiguousarray(batch.t_ascii)
    qo = np.ascontiguousarray(batch.q_off, np.int64)
    to = np.ascontiguousarray(batch.t_off, np.int64)
    h0 = np.ascontiguousarray(batch.h0, np.int32)
    ww = np.ascontiguousarray(w, np.int32)
    _lib().oracle_banded_batch(qa.ctypes.data, qo.ctypes.data, ta.ctypes.data, to.ctypes.data, h0.ctypes.data,
                               ww.ctypes.data, n, match, mismatch, alpha, beta, mode, *[o.ctypes.data for o in outs],
                               threads)
    return tuple(outs)


def start(q, t, match=1, mismatch=-4, alpha=7, beta=1):
    """(score, q_end, t_end, q_start, t_start) of one pair, LOCAL mode: the start by the reverse DP
    over the prefixes ending at the end cell (oracle.c header; reading 15)."""
    q, t = _b(q), _b(t)
    out = (ctypes.c_int32 * 5)()
    st = _lib().oracle_start(_buf(q), len(q), _buf(t), len(t), match, mismatch, alpha, beta, out)
    if st != OK:
        raise ValueError(st)
    return tuple(int(x) for x in out)


def start_batch(batch, match=1, mismatch=-4, alpha=7, beta=1, threads=None):
    """LOCAL start coordinates over a synth.Batch-like object.

    Returns (score, q_end, t_end, q_start, t_start, status, threads_used)."""
    n = len(batch.q_off) - 1
    outs = [np.empty(n, np.int32) for _ in range(6)]
    threads = threads or os.cpu_count() or 1
    qa = np.ascontiguousarray(batch.q_ascii)
    ta = np.ascontiguousarray(batch.t_ascii)
    qo = np.ascontiguousarray(batch.q_off, np.int64)
    to = np.ascontiguousarray(batch.t_off, np.int64)
    used = _lib().oracle_start_batch(qa.ctypes.data, qo.ctypes.data, ta.ctypes.data, to.ctypes.data, n,
                                     match, mismatch, alpha, beta, *[o.ctypes.data for o in outs], threads)
    return (*outs, used)


def timed_sample(batch, seconds=10.0, mode=LOCAL, threads=None, **sc):
    """Time the oracle, as it stands, over a bounded prefix of `batch`, growing the prefix until
    about `seconds` of wall time are spent.  Returns dict(gcups, cells, pairs, seconds, threads)."""
    from synth import Batch  # shared input module only

    threads = threads or os.cpu_count() or 1
    n_total = len(batch.q_off) - 1
    k = min(n_total, 64 * threads)
    cells_tot, pairs_tot, t_tot = 0, 0, 0.0
    start = 0
    while t_tot < seconds:
        if start >= n_total:  # wrap around: the sample is re-used until the time budget is spent
            start = 0
        end = min(n_total, start + k)
        sub = Batch(batch.q_ascii, batch.q_off[start:end + 1], batch.t_ascii, batch.t_off[start:end + 1],
                    batch.h0[start:end])
        t0 = time.perf_counter()
        _, _, _, _, used = align_batch(sub, mode=mode, threads=threads, **sc)
        dt = time.perf_counter() - t0
        ql = np.diff(sub.q_off).astype(np.int64)
        tl = np.diff(sub.t_off).astype(np.int64)
        cells_tot += int(np.dot(ql, tl))
        pairs_tot += end - start
        t_tot += dt
        start = end
        if dt < seconds / 8:
            k *= 2
    return dict(gcups=cells_tot / t_tot / 1e9 if t_tot > 0 else 0.0, cells=cells_tot, pairs=pairs_tot,
                seconds=t_tot, threads=threads)


# ---- BWA-MEM-compatible extension (oracle/ksw.c, reading 17) ----
KSW_NO_TRIM = 1
#: BWA-MEM defaults: a=1, b=4, o_del=e_del... (o=6, e=1), band w=100, end_bonus=5, zdrop=100
KSW_BWA = dict(a=1, b=4, o_del=6, e_del=1, o_ins=6, e_ins=1, w=100, end_bonus=5, zdrop=100)
KSW_FIELDS = ("score", "qle", "tle", "gtle", "gscore", "max_off", "clip")


def _ksw_params(kw):
    p = dict(KSW_BWA)
    p.update(kw)
    return [p[k] for k in ("a", "b", "o_del", "e_del", "o_ins", "e_ins", "w", "end_bonus", "zdrop")]


def ksw_extend(q, t, h0, flags=0, table=False, **kw):
    """BWA-MEM ksw_extend2 of one pair: dict of KSW_FIELDS (+ 'H': m x n table, -1 = not computed,
    when table=True).  Raises ValueError with the oracle status on invalid input."""
    q, t = _b(q), _b(t)
    out = (ctypes.c_int32 * 7)()
    args = [_buf(q), len(q), _buf(t), len(t), *_ksw_params(kw), h0, flags, out]
    if table:
        H = np.full((max(len(t), 1), max(len(q), 1)), -1, np.int32)
        st = _lib().oracle_ksw_table(*args, H.ctypes.data)
    else:
        st = _lib().oracle_ksw_extend(*args)
    if st != OK:
        raise ValueError(st)
    r = dict(zip(KSW_FIELDS, (int(x) for x in out)))
    if table:
        r["H"] = H
    return r


def ksw_batch(batch, flags=0, threads=None, **kw):
    """ksw_extend2 over a synth.Batch-like object: (out int32[7, n] rows = KSW_FIELDS, status int32[n])."""
    n = len(batch.q_off) - 1
    out = np.empty((7, max(n, 1)), np.int32)
    st = np.empty(max(n, 1), np.int32)
    threads = threads or os.cpu_count() or 1
    qa = np.ascontiguousarray(batch.q_ascii)
    ta = np.ascontiguousarray(batch.t_ascii)
    qo = np.ascontiguousarray(batch.q_off, np.int64)
    to = np.ascontiguousarray(batch.t_off, np.int64)
    h0 = np.ascontiguousarray(batch.h0, np.int32)
    par = np.array(_ksw_params(kw), np.int32)
    _lib().oracle_ksw_batch(qa.ctypes.data, qo.ctypes.data, ta.ctypes.data, to.ctypes.data, h0.ctypes.data, n,
                            par.ctypes.data, flags, out.ctypes.data, st.ctypes.data, threads)
    return out[:, :n], st[:n]


# ---- CIGAR traceback (oracle/traceback.c, reading 18) ------------
CIGAR_OPS = "MID"


def traceback(q, t, t_start, t_end, q_start, q_end, match=1, mismatch=-4, alpha=7, beta=1, cap=4096):
    """(cigar string, global score of t[t_start..t_end] x q[q_start..q_end]) of one pair."""
    q, t = _b(q), _b(t)
    ops = (ctypes.c_uint32 * cap)()
    out = (ctypes.c_int32 * 2)()
    st = _lib().oracle_traceback(_buf(q), len(q), _buf(t), len(t), match, mismatch, alpha, beta, t_start, t_end,
                                 q_start, q_end, ops, cap, out)
    if st != OK:
        raise ValueError(st)
    return "".join(f"{ops[k] >> 4}{CIGAR_OPS[ops[k] & 15]}" for k in range(out[0])), int(out[1])


def traceback_ops(q, t, t_start, t_end, q_start, q_end, match=1, mismatch=-4, alpha=7, beta=1, cap=4096):
    """Raw BAM-encoded CIGAR elements ((len << 4) | op) of one pair, and the global score."""
    q, t = _b(q), _b(t)
    ops = (ctypes.c_uint32 * cap)()
    out = (ctypes.c_int32 * 2)()
    st = _lib().oracle_traceback(_buf(q), len(q), _buf(t), len(t), match, mismatch, alpha, beta, t_start, t_end,
                                 q_start, q_end, ops, cap, out)
    if st != OK:
        raise ValueError(st)
    return [int(ops[k]) for k in range(out[0])], int(out[1])
