"""C-ABI library: loads, exports every symbol include/saloba.h declares, host-side validation
(CPU-only: no compute call reaches the GPU here)."""
import ctypes
import os
import re

import pytest

import build_native

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def L():
    build_native.build_saloba()
    import paper_2301_09310_b200 as sb

    return sb.lib()


def header_functions():
    txt = open(os.path.join(ROOT, "include", "saloba.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(saloba_[a-z_0-9]+)\s*\(", txt)))


def test_exports_every_declared_symbol(L):
    import paper_2301_09310_b200 as sb

    declared = header_functions()
    assert declared == sorted(sb.EXPORTS)
    for name in declared:
        assert hasattr(L, name), name


def test_version_and_strerror(L):
    assert L.saloba_version() == 2
    for code in (0, -1, -2, -3, -4, 7):
        assert isinstance(L.saloba_strerror(code), bytes)


def test_packed_words_closed_form(L):
    import paper_2301_09310_b200 as sb

    # ceil(len/8) words per sequence always fit in total/8 + n + 1
    assert sb.packed_words(0, 0) == 1
    assert sb.packed_words(150, 1) == 150 // 8 + 2
    assert sb.packed_words(160, 1, sb.PACK2) == 160 // 16 + 2
    assert L.saloba_packed_words(-1, 0, 4) == -1
    assert L.saloba_packed_words(10, 1, 3) == -1


def test_host_checked_errors_launch_nothing(L):
    import paper_2301_09310_b200 as sb

    sc = sb.BWA_MEM._c()
    nul = ctypes.c_void_p(0)
    dummy = ctypes.c_void_p(256)  # never dereferenced: validation fails first
    # negative n / null status / bad scheme / bad enums
    assert L.saloba_align_batch(nul, nul, nul, nul, nul, nul, nul, -1, sc, 0, 4, nul, nul, nul, dummy, 0, dummy,
                                None, nul) == sb.EINVAL
    assert L.saloba_align_batch(dummy, dummy, dummy, dummy, dummy, dummy, nul, 5, sc, 0, 4, dummy, dummy, dummy,
                                dummy, 1 << 20, nul, None, nul) == sb.EINVAL
    bad = sb.Scoring(1, -4, 1, 2)._c()  # alpha < beta
    assert L.saloba_align_batch(dummy, dummy, dummy, dummy, dummy, dummy, nul, 5, bad, 0, 4, dummy, dummy, dummy,
                                dummy, 1 << 20, dummy, None, nul) == sb.EINVAL
    for badsc in (sb.Scoring(0, -4, 7, 1), sb.Scoring(1, 0, 7, 1), sb.Scoring(1, -4, 7, 0), sb.Scoring(1, -4, 2000, 1)):
        assert L.saloba_align_batch(dummy, dummy, dummy, dummy, dummy, dummy, nul, 5, badsc._c(), 0, 4, dummy, dummy,
                                    dummy, dummy, 1 << 20, dummy, None, nul) == sb.EINVAL
    assert L.saloba_align_batch(dummy, dummy, dummy, dummy, dummy, dummy, nul, 5, sc, 2, 4, dummy, dummy, dummy,
                                dummy, 1 << 20, dummy, None, nul) == sb.EINVAL  # bad mode
    assert L.saloba_align_batch(dummy, dummy, dummy, dummy, dummy, dummy, nul, 5, sc, 0, 3, dummy, dummy, dummy,
                                dummy, 1 << 20, dummy, None, nul) == sb.EINVAL  # bad fmt
    # EXTEND without h0
    assert L.saloba_align_batch(dummy, dummy, dummy, dummy, dummy, dummy, nul, 5, sc, 1, 4, dummy, dummy, dummy,
                                dummy, 1 << 20, dummy, None, nul) == sb.EINVAL
    # unaligned workspace
    assert L.saloba_align_batch(dummy, dummy, dummy, dummy, dummy, dummy, nul, 5, sc, 0, 4, dummy, dummy, dummy,
                                ctypes.c_void_p(257), 1 << 20, dummy, None, nul) == sb.EINVAL
    # bad forced group
    opt = sb.Options(force_group=3)._c()
    assert L.saloba_align_batch(dummy, dummy, dummy, dummy, dummy, dummy, nul, 5, sc, 0, 4, dummy, dummy, dummy,
                                dummy, 1 << 20, dummy, ctypes.byref(opt), nul) == sb.EINVAL
    # pack
    assert L.saloba_pack(nul, nul, 3, 4, nul, 0, nul, nul, nul, nul) == sb.EINVAL
    assert L.saloba_pack(dummy, dummy, 3, 5, dummy, 10, dummy, nul, dummy, nul) == sb.EINVAL
    assert L.saloba_pack(dummy, dummy, -1, 4, dummy, 10, dummy, nul, dummy, nul) == sb.EINVAL
    # capacity below the layout's minimum (n_seqs + 1 words): EWORKSPACE before any launch
    assert L.saloba_pack(dummy, dummy, 10, 4, dummy, 10, dummy, nul, dummy, nul) == sb.EWORKSPACE
    # host entry: null status
    assert L.saloba_align_host(dummy, dummy, dummy, dummy, nul, 1, sc, 0, dummy, dummy, dummy, nul, None,
                               nul) == sb.EINVAL


def test_no_oracle_in_product_path():
    """The product package never imports/links the oracle (independence of the parity check)."""
    pkg = os.path.join(ROOT, "paper_2301_09310_b200")
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dp, f)).read()
                assert "oracle" not in txt.lower().replace("oracle-independent", ""), f


def test_host_checked_errors_new_entry_points(L):
    """saloba_align_banded / saloba_locate_start / saloba_partition: argument errors are returned
    synchronously, before any CUDA call (so they are checkable without a GPU)."""
    import paper_2301_09310_b200 as sb

    sc = sb.BWA_MEM._c()
    nul = ctypes.c_void_p(0)
    dummy = ctypes.c_void_p(256)
    # banded: band array missing for n > 0
    assert L.saloba_align_banded(dummy, dummy, dummy, dummy, dummy, dummy, nul, nul, 5, sc, 0, 4, dummy, dummy,
                                 dummy, dummy, 1 << 20, dummy, None, nul) == sb.EINVAL
    # start: null status, missing forward results, bad fmt, bad scheme, unaligned workspace
    args = [dummy, dummy, 100, dummy, dummy, 100, 5, sc, 4, dummy, dummy, dummy, dummy, dummy, dummy, 1 << 20, dummy,
            None, nul]
    a = list(args); a[16] = nul
    assert L.saloba_locate_start(*a) == sb.EINVAL
    a = list(args); a[9] = nul
    assert L.saloba_locate_start(*a) == sb.EINVAL
    a = list(args); a[8] = 3
    assert L.saloba_locate_start(*a) == sb.EINVAL
    a = list(args); a[7] = sb.Scoring(1, -4, 1, 2)._c()
    assert L.saloba_locate_start(*a) == sb.EINVAL
    a = list(args); a[14] = ctypes.c_void_p(300)
    assert L.saloba_locate_start(*a) == sb.EINVAL
    a = list(args); a[15] = 16  # workspace smaller than the reversed-prefix buffers
    assert L.saloba_locate_start(*a) == sb.EWORKSPACE
    # partition: bad world, null workspace, too small workspace, negative n
    assert L.saloba_partition_workspace_bytes(-1) == 0
    need = L.saloba_partition_workspace_bytes(1000)
    assert need >= 1000 * 24
    assert L.saloba_partition(dummy, dummy, 1000, 0, dummy, dummy, need, nul) == sb.EINVAL
    assert L.saloba_partition(dummy, dummy, 1000, 4, dummy, nul, need, nul) == sb.EINVAL
    assert L.saloba_partition(dummy, dummy, 1000, 4, dummy, dummy, need - 1, nul) == sb.EWORKSPACE
    assert L.saloba_partition(dummy, dummy, -1, 4, dummy, dummy, need, nul) == sb.EINVAL
    assert L.saloba_partition(nul, nul, 0, 4, nul, dummy, need, nul) == sb.OK  # empty batch: nothing to do


def test_host_checked_errors_scatter_results(L):
    """saloba_scatter_results (A5 reassembly): argument errors are returned before any CUDA call."""
    import paper_2301_09310_b200 as sb

    nul = ctypes.c_void_p(0)
    dummy = ctypes.c_void_p(256)
    assert L.saloba_scatter_results(dummy, dummy, 10, 2, 20, dummy, dummy, dummy, nul, nul) == sb.EINVAL  # no status
    assert L.saloba_scatter_results(nul, dummy, 10, 2, 20, dummy, dummy, dummy, dummy, nul) == sb.EINVAL  # no parts
    assert L.saloba_scatter_results(dummy, nul, 10, 2, 20, dummy, dummy, dummy, dummy, nul) == sb.EINVAL  # no index
    assert L.saloba_scatter_results(dummy, dummy, 10, 0, 20, dummy, dummy, dummy, dummy, nul) == sb.EINVAL  # world 0
    assert L.saloba_scatter_results(dummy, dummy, -1, 2, 20, dummy, dummy, dummy, dummy, nul) == sb.EINVAL
    assert L.saloba_scatter_results(dummy, dummy, 10, 2, 20, nul, dummy, dummy, dummy, nul) == sb.EINVAL  # no output
    assert L.saloba_scatter_results(dummy, dummy, 10, 2, 1 << 31, dummy, dummy, dummy, dummy, nul) == sb.EINVAL


def test_host_checked_errors_ksw(L):
    """saloba_ksw_extend (NEXT-1): argument errors are returned before any CUDA call."""
    import paper_2301_09310_b200 as sb

    nul = ctypes.c_void_p(0)
    dummy = ctypes.c_void_p(256)
    good = sb.BWA_KSW._c()
    args = [dummy] * 7 + [10, ctypes.byref(good), 4, 150, dummy, dummy, 1 << 20, dummy, nul]
    a = list(args); a[14] = nul  # status
    assert L.saloba_ksw_extend(*a) == sb.EINVAL
    a = list(args); a[6] = nul  # h0
    assert L.saloba_ksw_extend(*a) == sb.EINVAL
    a = list(args); a[9] = 3  # fmt
    assert L.saloba_ksw_extend(*a) == sb.EINVAL
    a = list(args); a[12] = ctypes.c_void_p(300)  # unaligned workspace
    assert L.saloba_ksw_extend(*a) == sb.EINVAL
    for bad in (sb.KswParams(a=0), sb.KswParams(b=0), sb.KswParams(e_ins=0), sb.KswParams(w=-1),
                sb.KswParams(zdrop=-1), sb.KswParams(o_del=2000)):
        a = list(args); a[8] = ctypes.byref(bad._c())
        assert L.saloba_ksw_extend(*a) == sb.EINVAL, bad
    a = list(args); a[8] = None
    assert L.saloba_ksw_extend(*a) == sb.EINVAL
