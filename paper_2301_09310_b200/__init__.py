"""paper_2301_09310_b200 — B200-native batched affine-gap seed extension (SALoBa hot path).

Thin Python binding over the C ABI in ``include/saloba.h`` (``libsaloba.so``, built in-tree for
sm_100a).  Argument marshalling only: every step of the path (packing, scheduling, DP, write-back)
runs in the library's CUDA kernels.  PyTorch supplies device memory and streams.  There is no CPU
fallback: if the library is missing or no sm_100 device is present, calls raise.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import torch

__all__ = [
    "LOCAL", "EXTEND", "PACK4", "PACK2", "Scoring", "Options", "BWA_MEM", "SalobaError", "lib", "lib_path",
    "packed_words", "pack", "workspace_bytes", "align_batch", "align", "align_banded", "start_workspace_bytes", "locate_start", "partition", "scatter_results",
    "KswParams", "BWA_KSW", "ksw_extend", "ksw_align", "KSW_FIELDS", "traceback", "cigar_strings",
    "align_host", "version", "EXPORTS",
]

LOCAL, EXTEND = 0, 1
PACK2, PACK4 = 2, 4
OK, EINVAL, ECUDA, EWORKSPACE, EUNSUPPORTED = 0, -1, -2, -3, -4

#: every symbol include/saloba.h declares
EXPORTS = ("saloba_packed_words", "saloba_pack", "saloba_workspace_bytes", "saloba_align_batch",
           "saloba_align_banded", "saloba_start_workspace_bytes", "saloba_locate_start",
           "saloba_partition_workspace_bytes", "saloba_partition", "saloba_scatter_results",
           "saloba_ksw_workspace_bytes", "saloba_ksw_extend", "saloba_traceback_workspace_bytes",
           "saloba_traceback",
           "saloba_host_ctx_create", "saloba_host_ctx_destroy", "saloba_align_host_ctx", "saloba_align_host",
           "saloba_stream_create", "saloba_stream_destroy", "saloba_stream_submit", "saloba_stream_wait",
           "saloba_strerror", "saloba_version", "saloba_kernel_launches")

_HERE = os.path.dirname(os.path.abspath(__file__))
# SALOBA_LIB: an alternative build of the same library (kernel A/B experiments, tools/variants.py)
lib_path = os.environ.get("SALOBA_LIB") or os.path.join(_HERE, "libsaloba.so")
_LIB = None


class SalobaError(RuntimeError):
    def __init__(self, code: int, what: str = ""):
        self.code = code
        msg = lib().saloba_strerror(code).decode() if _LIB is not None else str(code)
        super().__init__(f"{what}: {msg} ({code})" if what else f"{msg} ({code})")


class _Scoring(ctypes.Structure):
    _fields_ = [("match", ctypes.c_int32), ("mismatch", ctypes.c_int32), ("gap_open", ctypes.c_int32),
                ("gap_extend", ctypes.c_int32)]


class _KswParams(ctypes.Structure):
    _fields_ = [(k, ctypes.c_int32) for k in ("a", "b", "o_del", "e_del", "o_ins", "e_ins", "w", "end_bonus", "zdrop")]


class _Options(ctypes.Structure):
    _fields_ = [("force_group", ctypes.c_int32), ("force_path", ctypes.c_int32), ("keep_order", ctypes.c_int32),
                ("i16_rows", ctypes.c_int32), ("ev_dp_begin", ctypes.c_void_p), ("ev_dp_end", ctypes.c_void_p),
                ("bin_counts", ctypes.c_void_p), ("long_group", ctypes.c_void_p),
                ("counters", ctypes.c_void_p), ("reserved", ctypes.c_int32 * 2)]


@dataclass(frozen=True)
class Scoring:
    """match >= 1, mismatch <= -1, gap_open = alpha (first gap base) >= gap_extend = beta >= 1."""

    match: int = 1
    mismatch: int = -4
    gap_open: int = 7
    gap_extend: int = 1

    def _c(self) -> _Scoring:
        return _Scoring(self.match, self.mismatch, self.gap_open, self.gap_extend)


#: BWA-MEM-style scoring of the BASELINE configs: match 1, mismatch -4, o=6 e=1 -> alpha 7, beta 1
BWA_MEM = Scoring(1, -4, 7, 1)


@dataclass(frozen=True)
class KswParams:
    """BWA-MEM extension parameters (saloba_ksw_params): b is the mismatch PENALTY (> 0); a gap of k
    bases costs o + k*e; zdrop 0 disables the z-drop."""

    a: int = 1
    b: int = 4
    o_del: int = 6
    e_del: int = 1
    o_ins: int = 6
    e_ins: int = 1
    w: int = 100
    end_bonus: int = 5
    zdrop: int = 100

    def _c(self) -> _KswParams:
        return _KswParams(self.a, self.b, self.o_del, self.e_del, self.o_ins, self.e_ins, self.w, self.end_bonus,
                          self.zdrop)


#: BWA-MEM's defaults (mem_opt_init)
BWA_KSW = KswParams()
#: rows of saloba_ksw_extend's output
KSW_FIELDS = ("score", "qle", "tle", "gtle", "gscore", "max_off", "clip")


@dataclass(frozen=True)
class Options:
    force_group: int = 0  # 0 = scheduler; else G in {1,2,4,8,16,32}
    force_path: int = 0  # 0 auto, 1 int32 exact, 2 prefer int16x2
    keep_order: int = 0  # 1 = no length sort
    dp_events: tuple | None = None  # (torch.cuda.Event, torch.cuda.Event) bracketing the DP kernels
    bin_counts: torch.Tensor | None = None  # cuda int32[16] <- pairs per bin (path*8 + log2 G)
    i16_rows: int = 0  # 0 default (16); 8 = 8 target rows per lane in the int16x2 kernel
    long_group: torch.Tensor | None = None  # cuda int32[1] <- log2 G the long bin (13) ran with
    counters: torch.Tensor | None = None  # cuda int64[8] += NEXT-4 counters (saloba.h saloba_options.counters)

    def _c(self) -> _Options:
        o = _Options(self.force_group, self.force_path, self.keep_order, self.i16_rows)
        if self.dp_events is not None:
            o.ev_dp_begin = ctypes.c_void_p(self.dp_events[0].cuda_event)
            o.ev_dp_end = ctypes.c_void_p(self.dp_events[1].cuda_event)
        if self.bin_counts is not None:
            o.bin_counts = ctypes.c_void_p(self.bin_counts.data_ptr())
        if self.long_group is not None:
            o.long_group = ctypes.c_void_p(self.long_group.data_ptr())
        if self.counters is not None:
            o.counters = ctypes.c_void_p(self.counters.data_ptr())
        return o


def lib() -> ctypes.CDLL:
    """The loaded C-ABI library (raises if it was not built)."""
    global _LIB
    if _LIB is None:
        if not os.path.exists(lib_path):
            raise ImportError(f"{lib_path} is missing; build it with `python build_native.py` "
                              "(or __graft_entry__.build()). There is no CPU fallback.")
        L = ctypes.CDLL(lib_path)
        vp, i32, i64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64
        L.saloba_packed_words.argtypes = [i64, i64, ctypes.c_int]
        L.saloba_packed_words.restype = i64
        L.saloba_pack.argtypes = [vp, vp, i64, ctypes.c_int, vp, i64, vp, vp, vp, vp]
        L.saloba_pack.restype = ctypes.c_int
        L.saloba_workspace_bytes.argtypes = [i64, i32, i32, ctypes.c_int]
        L.saloba_workspace_bytes.restype = ctypes.c_size_t
        L.saloba_align_batch.argtypes = [vp, vp, vp, vp, vp, vp, vp, i64, _Scoring, ctypes.c_int, ctypes.c_int,
                                         vp, vp, vp, vp, ctypes.c_size_t, vp, ctypes.POINTER(_Options), vp]
        L.saloba_align_batch.restype = ctypes.c_int
        L.saloba_align_banded.argtypes = [vp, vp, vp, vp, vp, vp, vp, vp, i64, _Scoring, ctypes.c_int, ctypes.c_int,
                                          vp, vp, vp, vp, ctypes.c_size_t, vp, ctypes.POINTER(_Options), vp]
        L.saloba_align_banded.restype = ctypes.c_int
        L.saloba_partition_workspace_bytes.argtypes = [i64]
        L.saloba_partition_workspace_bytes.restype = ctypes.c_size_t
        L.saloba_partition.argtypes = [vp, vp, i64, i32, vp, vp, ctypes.c_size_t, vp]
        L.saloba_partition.restype = ctypes.c_int
        L.saloba_ksw_workspace_bytes.argtypes = [i64, i32, ctypes.c_int]
        L.saloba_ksw_workspace_bytes.restype = ctypes.c_size_t
        L.saloba_ksw_extend.argtypes = [vp, vp, vp, vp, vp, vp, vp, i64, ctypes.POINTER(_KswParams), ctypes.c_int, i32,
                                        vp, vp, ctypes.c_size_t, vp, vp]
        L.saloba_ksw_extend.restype = ctypes.c_int
        L.saloba_traceback_workspace_bytes.argtypes = [i64, i32, i32, ctypes.c_int]
        L.saloba_traceback_workspace_bytes.restype = ctypes.c_size_t
        L.saloba_traceback.argtypes = [vp, vp, vp, vp, i64, _Scoring, ctypes.c_int, vp, vp, vp, vp, vp, i32, i32, vp,
                                       i32, vp, vp, ctypes.c_size_t, vp, vp]
        L.saloba_traceback.restype = ctypes.c_int
        L.saloba_scatter_results.argtypes = [vp, vp, i64, i32, i64, vp, vp, vp, vp, vp]
        L.saloba_scatter_results.restype = ctypes.c_int
        L.saloba_start_workspace_bytes.argtypes = [i64, i64, i64, i32, ctypes.c_int]
        L.saloba_start_workspace_bytes.restype = ctypes.c_size_t
        L.saloba_locate_start.argtypes = [vp, vp, i64, vp, vp, i64, i64, _Scoring, ctypes.c_int, vp, vp, vp, vp, vp,
                                          vp, ctypes.c_size_t, vp, ctypes.POINTER(_Options), vp]
        L.saloba_locate_start.restype = ctypes.c_int
        L.saloba_align_host.argtypes = [vp, vp, vp, vp, vp, i64, _Scoring, ctypes.c_int, vp, vp, vp, vp,
                                        ctypes.POINTER(_Options), vp]
        L.saloba_align_host.restype = ctypes.c_int
        L.saloba_host_ctx_create.argtypes = [i64, i64, i64, i32, ctypes.c_int]
        L.saloba_host_ctx_create.restype = vp
        L.saloba_host_ctx_destroy.argtypes = [vp]
        L.saloba_host_ctx_destroy.restype = None
        L.saloba_align_host_ctx.argtypes = [vp] + list(L.saloba_align_host.argtypes)
        L.saloba_align_host_ctx.restype = ctypes.c_int
        L.saloba_stream_create.argtypes = [i64, i64, i64, i32, ctypes.c_int]
        L.saloba_stream_create.restype = vp
        L.saloba_stream_destroy.argtypes = [vp]
        L.saloba_stream_destroy.restype = None
        L.saloba_stream_submit.argtypes = [vp, vp, vp, vp, vp, vp, i64, _Scoring, ctypes.c_int, vp, vp, vp, vp,
                                           ctypes.POINTER(_Options)]
        L.saloba_stream_submit.restype = ctypes.c_int
        L.saloba_stream_wait.argtypes = [vp]
        L.saloba_stream_wait.restype = ctypes.c_int
        L.saloba_strerror.argtypes = [ctypes.c_int]
        L.saloba_strerror.restype = ctypes.c_char_p
        L.saloba_version.restype = ctypes.c_int
        L.saloba_kernel_launches.restype = ctypes.c_int64
        _LIB = L
    return _LIB


def version() -> int:
    return lib().saloba_version()


def kernel_launches() -> int:
    """Process-wide count of this library's own kernel launches (diagnostics; bench gpu_launches)."""
    return int(lib().saloba_kernel_launches())


def _check(rc: int, what: str) -> None:
    if rc != OK:
        raise SalobaError(rc, what)


def _p(t) -> ctypes.c_void_p:
    return ctypes.c_void_p(0 if t is None else t.data_ptr())


def _stream(stream) -> ctypes.c_void_p:
    s = torch.cuda.current_stream() if stream is None else stream
    return ctypes.c_void_p(s.cuda_stream)


def _dev_tensor(t: torch.Tensor, dtype, name: str) -> torch.Tensor:
    if not (isinstance(t, torch.Tensor) and t.is_cuda):
        raise TypeError(f"{name} must be a CUDA tensor")
    if t.dtype != dtype:
        raise TypeError(f"{name} must be {dtype}, got {t.dtype}")
    return t.contiguous()


def packed_words(total_bases: int, n_seqs: int, fmt: int = PACK4) -> int:
    return int(lib().saloba_packed_words(total_bases, n_seqs, fmt))


def pack(ascii: torch.Tensor, byte_off: torch.Tensor, fmt: int = PACK4, total_bases: int | None = None,
         stream=None):
    """ASCII (uint8, cuda) + byte offsets (int64[n+1], cuda) -> (words, word_off, lens, status).

    ``status`` is a 1-element int64 cuda tensor: -1 or the first invalid byte index."""
    ascii = _dev_tensor(ascii, torch.uint8, "ascii")
    byte_off = _dev_tensor(byte_off, torch.int64, "byte_off")
    n = byte_off.numel() - 1
    total = ascii.numel() if total_bases is None else total_bases
    cap = packed_words(total, n, fmt)
    dev = ascii.device
    words = torch.empty(max(cap, 1), dtype=torch.int32, device=dev)
    word_off = torch.empty(n + 1, dtype=torch.int64, device=dev)
    lens = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
    status = torch.empty(1, dtype=torch.int64, device=dev)
    _check(lib().saloba_pack(_p(ascii), _p(byte_off), n, fmt, _p(words), cap, _p(word_off), _p(lens), _p(status),
                             _stream(stream)), "saloba_pack")
    return words, word_off, lens[:n], status


def workspace_bytes(n_pairs: int, max_qlen: int, max_tlen: int = 0, device: int | None = None) -> int:
    dev = torch.cuda.current_device() if device is None else device
    b = int(lib().saloba_workspace_bytes(n_pairs, max_qlen, max_tlen, dev))
    if b == 0:
        raise SalobaError(ECUDA, "saloba_workspace_bytes")
    return b


def align_batch(q_words, q_word_off, q_len, t_words, t_word_off, t_len, h0=None, scoring: Scoring = BWA_MEM,
                mode: int = LOCAL, fmt: int = PACK4, out=None, workspace: torch.Tensor | None = None,
                options: Options | None = None, max_qlen: int | None = None, stream=None):
    """Align packed pairs on the GPU. Returns (score, q_end, t_end, status) cuda int32/int64 tensors.

    `workspace` (uint8 cuda tensor) is allocated when omitted (sized from max_qlen, or from
    q_len.max() with a device sync)."""
    n = q_len.numel()
    dev = q_len.device
    if out is None:
        out = torch.empty((3, max(n, 1)), dtype=torch.int32, device=dev)
    score, q_end, t_end = out[0], out[1], out[2]
    if workspace is None:
        mq = int(q_len.max().item()) if (max_qlen is None and n > 0) else (max_qlen or 1)
        workspace = torch.empty(workspace_bytes(n, mq, 0, dev.index), dtype=torch.uint8, device=dev)
    status = torch.empty(1, dtype=torch.int64, device=dev)
    opt = ctypes.byref(options._c()) if options is not None else None
    if mode == EXTEND and h0 is None:
        raise ValueError("EXTEND mode needs h0")
    args = [q_words, q_word_off, q_len, t_words, t_word_off, t_len]
    names = ["q_words", "q_word_off", "q_len", "t_words", "t_word_off", "t_len"]
    dts = [torch.int32, torch.int64, torch.int32, torch.int32, torch.int64, torch.int32]
    args = [_dev_tensor(a, d, nm) for a, d, nm in zip(args, dts, names)]
    if h0 is not None:
        h0 = _dev_tensor(h0, torch.int32, "h0")
    rc = lib().saloba_align_batch(*[_p(a) for a in args], _p(h0), n, scoring._c(), mode, fmt, _p(score),
                                  _p(q_end), _p(t_end), _p(workspace), workspace.numel(), _p(status), opt,
                                  _stream(stream))
    _check(rc, "saloba_align_batch")
    return score[:n], q_end[:n], t_end[:n], status


def align_banded(q_words, q_word_off, q_len, t_words, t_word_off, t_len, band_w, h0=None,
                 scoring: Scoring = BWA_MEM, mode: int = LOCAL, fmt: int = PACK4, out=None,
                 workspace: torch.Tensor | None = None, options: Options | None = None, max_qlen: int | None = None,
                 stream=None):
    """Banded alignment (saloba_align_banded): only cells |i - j| <= band_w[k] are in pair k's table.
    Returns (score, q_end, t_end, status) like align_batch."""
    n = q_len.numel()
    dev = q_len.device
    if out is None:
        out = torch.empty((3, max(n, 1)), dtype=torch.int32, device=dev)
    score, q_end, t_end = out[0], out[1], out[2]
    if workspace is None:
        mq = int(q_len.max().item()) if (max_qlen is None and n > 0) else (max_qlen or 1)
        workspace = torch.empty(workspace_bytes(n, mq, 0, dev.index), dtype=torch.uint8, device=dev)
    status = torch.empty(1, dtype=torch.int64, device=dev)
    opt = ctypes.byref(options._c()) if options is not None else None
    if mode == EXTEND and h0 is None:
        raise ValueError("EXTEND mode needs h0")
    args = [q_words, q_word_off, q_len, t_words, t_word_off, t_len]
    names = ["q_words", "q_word_off", "q_len", "t_words", "t_word_off", "t_len"]
    dts = [torch.int32, torch.int64, torch.int32, torch.int32, torch.int64, torch.int32]
    args = [_dev_tensor(a, d, nm) for a, d, nm in zip(args, dts, names)]
    band_w = _dev_tensor(band_w, torch.int32, "band_w")
    if h0 is not None:
        h0 = _dev_tensor(h0, torch.int32, "h0")
    rc = lib().saloba_align_banded(*[_p(a) for a in args], _p(h0), _p(band_w), n, scoring._c(), mode, fmt,
                                   _p(score), _p(q_end), _p(t_end), _p(workspace), workspace.numel(), _p(status),
                                   opt, _stream(stream))
    _check(rc, "saloba_align_banded")
    return score[:n], q_end[:n], t_end[:n], status


def partition(q_len: torch.Tensor, t_len: torch.Tensor, world: int, stream=None) -> torch.Tensor:
    """Length-balanced rank of each pair (saloba_partition): int32 cuda tensor in 0..world-1."""
    q_len = _dev_tensor(q_len, torch.int32, "q_len")
    t_len = _dev_tensor(t_len, torch.int32, "t_len")
    n = q_len.numel()
    owner = torch.empty(max(n, 1), dtype=torch.int32, device=q_len.device)
    ws = torch.empty(int(lib().saloba_partition_workspace_bytes(n)), dtype=torch.uint8, device=q_len.device)
    _check(lib().saloba_partition(_p(q_len), _p(t_len), n, world, _p(owner), _p(ws), ws.numel(), _stream(stream)),
           "saloba_partition")
    return owner[:n]


def scatter_results(parts: torch.Tensor, index: torch.Tensor, n_total: int, out: torch.Tensor | None = None,
                    stream=None):
    """A5 reassembly (saloba_scatter_results): parts (world, 3, stride) int32 as gathered, index
    (world, stride) int32 global input index per column (-1 = padding) -> (out (3, n_total), status)."""
    parts = _dev_tensor(parts, torch.int32, "parts")
    index = _dev_tensor(index, torch.int32, "index")
    if parts.dim() != 3 or parts.shape[1] != 3 or index.shape != (parts.shape[0], parts.shape[2]):
        raise ValueError("parts must be (world, 3, stride) and index (world, stride)")
    world, stride = int(index.shape[0]), int(index.shape[1])
    if out is None:
        out = torch.full((3, max(n_total, 1)), -9, dtype=torch.int32, device=parts.device)
    status = torch.empty(1, dtype=torch.int64, device=parts.device)
    _check(lib().saloba_scatter_results(_p(parts), _p(index), stride, world, n_total, _p(out[0]), _p(out[1]),
                                        _p(out[2]), _p(status), _stream(stream)), "saloba_scatter_results")
    return out, status


def ksw_extend(q_words, q_word_off, q_len, t_words, t_word_off, t_len, h0, params: KswParams = BWA_KSW,
               fmt: int = PACK4, max_qlen: int | None = None, out=None, workspace=None, stream=None):
    """BWA-MEM-compatible extension of packed pairs (saloba_ksw_extend): returns (out int32[7, n]
    with rows KSW_FIELDS, status)."""
    n = q_len.numel()
    dev = q_len.device
    args = [_dev_tensor(a_, d_, nm) for a_, d_, nm in zip(
        (q_words, q_word_off, q_len, t_words, t_word_off, t_len, h0),
        (torch.int32, torch.int64, torch.int32, torch.int32, torch.int64, torch.int32, torch.int32),
        ("q_words", "q_word_off", "q_len", "t_words", "t_word_off", "t_len", "h0"))]
    if max_qlen is None:
        max_qlen = int(args[2].max().item()) if n > 0 else 1
    if out is None:
        out = torch.empty((7, max(n, 1)), dtype=torch.int32, device=dev)
    if workspace is None:
        b = int(lib().saloba_ksw_workspace_bytes(n, max_qlen, dev.index))
        if b == 0:
            raise SalobaError(ECUDA, "saloba_ksw_workspace_bytes")
        workspace = torch.empty(b, dtype=torch.uint8, device=dev)
    status = torch.empty(1, dtype=torch.int64, device=dev)
    pc = params._c()
    rc = lib().saloba_ksw_extend(*[_p(a_) for a_ in args], n, ctypes.byref(pc), fmt, max_qlen, _p(out), _p(workspace),
                                 workspace.numel(), _p(status), _stream(stream))
    _check(rc, "saloba_ksw_extend")
    return out[:, :n], status


def ksw_align(q_ascii, q_off, t_ascii, t_off, h0, params: KswParams = BWA_KSW, fmt: int = PACK4,
              max_qlen: int | None = None, stream=None):
    """Device-resident ASCII pairs -> (out int32[7, n], status, q pack status, t pack status)."""
    qw, qwo, ql, qst = pack(q_ascii, q_off, fmt, stream=stream)
    tw, two, tl, tst = pack(t_ascii, t_off, fmt, stream=stream)
    out, st = ksw_extend(qw, qwo[:-1], ql, tw, two[:-1], tl, h0, params, fmt, max_qlen=max_qlen, stream=stream)
    return out, st, qst, tst


def traceback(q_words, q_word_off, t_words, t_word_off, score, q_start, q_end, t_start, t_end,
              scoring: Scoring = BWA_MEM, fmt: int = PACK4, cigar_cap: int = 64, max_qlen: int | None = None,
              max_tlen: int | None = None, stream=None):
    """CIGARs of LOCAL results (saloba_traceback): returns (cigar uint32[n, cap], n_ops int32[n], status)."""
    n = score.numel()
    dev = score.device
    args = [_dev_tensor(x, d_, nm) for x, d_, nm in zip(
        (q_words, q_word_off, t_words, t_word_off, score, q_start, q_end, t_start, t_end),
        (torch.int32, torch.int64, torch.int32, torch.int64) + (torch.int32,) * 5,
        ("q_words", "q_word_off", "t_words", "t_word_off", "score", "q_start", "q_end", "t_start", "t_end"))]
    if max_qlen is None:
        max_qlen = int((args[6] - args[5]).max().item()) + 1 if n > 0 else 1
    if max_tlen is None:
        max_tlen = int((args[8] - args[7]).max().item()) + 1 if n > 0 else 1
    cigar = torch.empty((max(n, 1), cigar_cap), dtype=torch.int32, device=dev)
    n_ops = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
    ws = torch.empty(int(lib().saloba_traceback_workspace_bytes(n, max_qlen, max_tlen, dev.index)), dtype=torch.uint8,
                     device=dev)
    status = torch.empty(1, dtype=torch.int64, device=dev)
    rc = lib().saloba_traceback(*[_p(x) for x in args[:4]], n, scoring._c(), fmt, *[_p(x) for x in args[4:]],
                                max_qlen, max_tlen, _p(cigar), cigar_cap, _p(n_ops), _p(ws), ws.numel(), _p(status),
                                _stream(stream))
    _check(rc, "saloba_traceback")
    return cigar[:n], n_ops[:n], status


def cigar_strings(cigar, n_ops) -> list:
    """Host-side formatting of saloba_traceback's output: CIGAR strings ("" for 0 ops, None for -1)."""
    c = cigar.cpu().numpy().view("uint32")
    k = n_ops.cpu().numpy()
    out = []
    for r in range(len(k)):
        if k[r] < 0:
            out.append(None)
        else:
            out.append("".join(f"{int(x) >> 4}{'MID'[int(x) & 15]}" for x in c[r, :k[r]]))
    return out


def start_workspace_bytes(n_pairs: int, q_words_total: int, t_words_total: int, max_qlen: int,
                          device: int | None = None) -> int:
    dev = torch.cuda.current_device() if device is None else device
    b = int(lib().saloba_start_workspace_bytes(n_pairs, q_words_total, t_words_total, max_qlen, dev))
    if b == 0:
        raise SalobaError(ECUDA, "saloba_start_workspace_bytes")
    return b


def locate_start(q_words, q_word_off, t_words, t_word_off, score, q_end, t_end, scoring: Scoring = BWA_MEM,
                 fmt: int = PACK4, out=None, workspace: torch.Tensor | None = None, options: Options | None = None,
                 max_qlen: int | None = None, stream=None):
    """Start coordinates of LOCAL results (saloba_locate_start): returns (q_start, t_start, status).

    q_words / t_words are the packed buffers the forward call used (their numel is the capacity);
    score / q_end / t_end are its results."""
    n = score.numel()
    dev = score.device
    if out is None:
        out = torch.empty((2, max(n, 1)), dtype=torch.int32, device=dev)
    q_start, t_start = out[0], out[1]
    args = [_dev_tensor(a, d, nm) for a, d, nm in zip(
        (q_words, q_word_off, t_words, t_word_off, score, q_end, t_end),
        (torch.int32, torch.int64, torch.int32, torch.int64, torch.int32, torch.int32, torch.int32),
        ("q_words", "q_word_off", "t_words", "t_word_off", "score", "q_end", "t_end"))]
    qw, qwo, tw, two, sc_, qe, te = args
    if workspace is None:
        mq = int(qe.max().item()) + 1 if (max_qlen is None and n > 0) else (max_qlen or 1)
        workspace = torch.empty(start_workspace_bytes(n, qw.numel(), tw.numel(), mq, dev.index), dtype=torch.uint8,
                                device=dev)
    status = torch.empty(1, dtype=torch.int64, device=dev)
    opt = ctypes.byref(options._c()) if options is not None else None
    rc = lib().saloba_locate_start(_p(qw), _p(qwo), qw.numel(), _p(tw), _p(two), tw.numel(), n, scoring._c(), fmt,
                                   _p(sc_), _p(qe), _p(te), _p(q_start), _p(t_start), _p(workspace),
                                   workspace.numel(), _p(status), opt, _stream(stream))
    _check(rc, "saloba_locate_start")
    return q_start[:n], t_start[:n], status


def align(q_ascii, q_off, t_ascii, t_off, h0=None, scoring: Scoring = BWA_MEM, mode: int = LOCAL,
          fmt: int = PACK4, options: Options | None = None, max_qlen: int | None = None, workspace=None,
          stream=None):
    """Device-resident ASCII pairs -> (score, q_end, t_end, status): pack (A1) then align (A2-A4).
    status: -1, or the first bad pair index from alignment; pack errors raise after a sync."""
    qw, qwo, ql, qst = pack(q_ascii, q_off, fmt, stream=stream)
    tw, two, tl, tst = pack(t_ascii, t_off, fmt, stream=stream)
    res = align_batch(qw, qwo[:-1], ql, tw, two[:-1], tl, h0, scoring, mode, fmt, workspace=workspace,
                      options=options, max_qlen=max_qlen, stream=stream)
    return (*res[:3], res[3], qst, tst)


def align_host(batch, scoring: Scoring = BWA_MEM, mode: int = LOCAL, options: Options | None = None,
               out=None, stream=None, ctx: "HostContext | None" = None):
    """End-to-end from host buffers (numpy / pinned CPU tensors): returns numpy-like int32 arrays
    (score, q_end, t_end) and the host status (-1 or first bad pair).  The library pipelines the
    upload in slices; copies overlap compute only for page-locked (pinned) host memory, so the
    default `out` is pinned (pass pinned inputs too, e.g. torch tensors with pin_memory=True)."""
    import numpy as np

    def host_ptr(a):
        if isinstance(a, torch.Tensor):
            assert not a.is_cuda
            return ctypes.c_void_p(a.data_ptr())
        return ctypes.c_void_p(a.ctypes.data)

    n = len(batch.q_off) - 1
    if out is None:
        out = torch.empty((3, max(n, 1)), dtype=torch.int32, pin_memory=torch.cuda.is_available()).numpy()
    st = ctypes.c_int64(0)
    opt = ctypes.byref(options._c()) if options is not None else None
    qo = np.ascontiguousarray(batch.q_off, np.int64)
    to = np.ascontiguousarray(batch.t_off, np.int64)
    h0 = np.ascontiguousarray(batch.h0, np.int32) if mode == EXTEND else None
    o = out if isinstance(out, np.ndarray) else out.numpy()
    args = (host_ptr(batch.q_ascii), host_ptr(qo), host_ptr(batch.t_ascii), host_ptr(to),
            host_ptr(h0) if h0 is not None else None, n, scoring._c(), mode,
            ctypes.c_void_p(o[0].ctypes.data), ctypes.c_void_p(o[1].ctypes.data),
            ctypes.c_void_p(o[2].ctypes.data), ctypes.byref(st), opt, _stream(stream))
    if ctx is not None:
        rc = lib().saloba_align_host_ctx(ctypes.c_void_p(ctx.handle), *args)
    else:
        rc = lib().saloba_align_host(*args)
    _check(rc, "saloba_align_host")
    return o[0, :n], o[1, :n], o[2, :n], int(st.value)


class Aligner:
    """Preallocated device pipeline for repeated batches of the same capacity (the hot path the
    bench times): pack (A1) -> schedule + DP + write-back (A2-A4), all on one stream, no host sync.

    Capacity: n_pairs pairs, total_q / total_t ASCII bytes, queries up to max_qlen bases."""

    def __init__(self, n_pairs: int, total_q: int, total_t: int, max_qlen: int, scoring: Scoring = BWA_MEM,
                 mode: int = LOCAL, fmt: int = PACK4, options: Options | None = None, device=None):
        self.dev = torch.device("cuda", torch.cuda.current_device() if device is None else device)
        self.n, self.scoring, self.mode, self.fmt = n_pairs, scoring, mode, fmt
        self.options = options
        d = self.dev
        qcap, tcap = packed_words(total_q, n_pairs, fmt), packed_words(total_t, n_pairs, fmt)
        self.qcap, self.tcap = qcap, tcap
        self.q_words = torch.empty(max(qcap, 1), dtype=torch.int32, device=d)
        self.t_words = torch.empty(max(tcap, 1), dtype=torch.int32, device=d)
        self.q_word_off = torch.empty(n_pairs + 1, dtype=torch.int64, device=d)
        self.t_word_off = torch.empty(n_pairs + 1, dtype=torch.int64, device=d)
        self.q_len = torch.empty(max(n_pairs, 1), dtype=torch.int32, device=d)
        self.t_len = torch.empty(max(n_pairs, 1), dtype=torch.int32, device=d)
        self.out = torch.empty((3, max(n_pairs, 1)), dtype=torch.int32, device=d)
        self.status = torch.empty(4, dtype=torch.int64, device=d)  # [pack q, pack t, align, -]
        self.ws = torch.empty(workspace_bytes(n_pairs, max_qlen, 0, d.index), dtype=torch.uint8, device=d)

    def run(self, q_ascii, q_off, t_ascii, t_off, h0=None, options: Options | None = None, stream=None):
        """Returns views (score, q_end, t_end) of the preallocated output (valid after sync)."""
        L, st = lib(), _stream(stream)
        n = self.n
        _check(L.saloba_pack(_p(q_ascii), _p(q_off), n, self.fmt, _p(self.q_words), self.qcap, _p(self.q_word_off),
                             _p(self.q_len), ctypes.c_void_p(self.status.data_ptr()), st), "saloba_pack")
        _check(L.saloba_pack(_p(t_ascii), _p(t_off), n, self.fmt, _p(self.t_words), self.tcap, _p(self.t_word_off),
                             _p(self.t_len), ctypes.c_void_p(self.status.data_ptr() + 8), st), "saloba_pack")
        o = options if options is not None else self.options
        opt = ctypes.byref(o._c()) if o is not None else None
        rc = L.saloba_align_batch(_p(self.q_words), _p(self.q_word_off), _p(self.q_len), _p(self.t_words),
                                  _p(self.t_word_off), _p(self.t_len), _p(h0) if self.mode == EXTEND else None, n,
                                  self.scoring._c(), self.mode, self.fmt, _p(self.out[0]), _p(self.out[1]),
                                  _p(self.out[2]), _p(self.ws), self.ws.numel(),
                                  ctypes.c_void_p(self.status.data_ptr() + 16), opt, st)
        _check(rc, "saloba_align_batch")
        return self.out[0, :n], self.out[1, :n], self.out[2, :n]


    def capture(self, q_ascii, q_off, t_ascii, t_off, h0=None, options: Options | None = None):
        """Capture one run() on these (fixed) input buffers as a CUDA graph and return it; replay()
        re-runs pack + schedule + DP on whatever the buffers hold, with no per-launch host work
        (launch-bound small batches gain ~25%).  The kernels' auxiliary streams join the capture
        through the library's fork/join events."""
        g = torch.cuda.CUDAGraph()
        cap = torch.cuda.Stream(device=self.dev)
        cap.wait_stream(torch.cuda.current_stream(self.dev))
        with torch.cuda.stream(cap):
            self.run(q_ascii, q_off, t_ascii, t_off, h0, options)  # warm on the capture stream
            torch.cuda.synchronize(self.dev)
            with torch.cuda.graph(g, stream=cap):
                self.run(q_ascii, q_off, t_ascii, t_off, h0, options)
        torch.cuda.current_stream(self.dev).wait_stream(cap)
        return g


class HostContext:
    """Reusable device buffers/streams for the host-buffer entry point (saloba_host_ctx)."""

    def __init__(self, max_pairs: int, max_q_bytes: int, max_t_bytes: int, max_qlen: int, device=None):
        dev = torch.cuda.current_device() if device is None else device
        self.handle = lib().saloba_host_ctx_create(max_pairs, max_q_bytes, max_t_bytes, max_qlen, dev)
        if not self.handle:
            raise SalobaError(ECUDA, "saloba_host_ctx_create")

    def close(self):
        if self.handle:
            lib().saloba_host_ctx_destroy(ctypes.c_void_p(self.handle))
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class HostStream:
    """Streaming host batches (saloba_stream_*): submit() enqueues a host batch and returns at once
    (it only finishes the batch submitted two calls earlier), so a batch's upload overlaps the
    previous batch's alignment.  Results land in the given host arrays (pinned: numpy views of
    torch pin_memory tensors) and are valid after wait() or two submits later."""

    def __init__(self, max_pairs: int, max_q_bytes: int, max_t_bytes: int, max_qlen: int, device=None):
        dev = torch.cuda.current_device() if device is None else device
        self.handle = lib().saloba_stream_create(max_pairs, max_q_bytes, max_t_bytes, max_qlen, dev)
        if not self.handle:
            raise SalobaError(ECUDA, "saloba_stream_create")
        self._keep = []  # host arrays of the batches in flight (kept alive until finished)

    def submit(self, batch, out, status, scoring: Scoring = BWA_MEM, mode: int = LOCAL,
               options: Options | None = None):
        """out: int32 host array (3, n) (score, q_end, t_end); status: ctypes.c_int64 receiving -1 or
        the first bad pair once the batch is finished."""
        import numpy as np

        n = len(batch.q_off) - 1
        qo = np.ascontiguousarray(batch.q_off, np.int64)
        to = np.ascontiguousarray(batch.t_off, np.int64)
        h0 = np.ascontiguousarray(batch.h0, np.int32) if mode == EXTEND else None
        o = out if isinstance(out, np.ndarray) else out.numpy()
        opt = ctypes.byref(options._c()) if options is not None else None
        keep = (batch.q_ascii, batch.t_ascii, qo, to, h0, o)
        self._keep = (self._keep + [keep])[-2:]
        rc = lib().saloba_stream_submit(
            ctypes.c_void_p(self.handle), ctypes.c_void_p(batch.q_ascii.ctypes.data), ctypes.c_void_p(qo.ctypes.data),
            ctypes.c_void_p(batch.t_ascii.ctypes.data), ctypes.c_void_p(to.ctypes.data),
            ctypes.c_void_p(h0.ctypes.data) if h0 is not None else None, n, scoring._c(), mode,
            ctypes.c_void_p(o[0].ctypes.data), ctypes.c_void_p(o[1].ctypes.data), ctypes.c_void_p(o[2].ctypes.data),
            ctypes.byref(status), opt)
        _check(rc, "saloba_stream_submit")

    def wait(self):
        _check(lib().saloba_stream_wait(ctypes.c_void_p(self.handle)), "saloba_stream_wait")

    def close(self):
        if self.handle:
            lib().saloba_stream_destroy(ctypes.c_void_p(self.handle))
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
