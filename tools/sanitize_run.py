"""Small workload that launches every kernel of libsaloba.so once or twice, for compute-sanitizer
(memcheck / racecheck / synccheck).  Checks results against the oracle on the way, so a
sanitizer run is also a parity run.

    compute-sanitizer --tool racecheck python tools/sanitize_run.py
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402  (tool, not product)
import paper_2301_09310_b200 as sb  # noqa: E402
import synth  # noqa: E402


def dev(b):
    return [torch.from_numpy(x).cuda() for x in (b.q_ascii, b.q_off, b.t_ascii, b.t_off, b.h0)]


def check(b, got, mode, label, sc=sb.BWA_MEM):
    ref = oracle.align_batch(b, sc.match, sc.mismatch, sc.gap_open, sc.gap_extend, mode)
    for g, r in zip(got[:3], ref[:3]):
        assert np.array_equal(g.cpu().numpy(), r), label
    print("ok", label, flush=True)


def main():
    torch.cuda.set_device(0)
    kernels0 = sb.kernel_launches()
    short = synth.generate(2, 3000, seed=5)                      # G = 1 kernel (dp_g1)
    mixed = synth.generate(3, 1500, seed=6)                      # G = 1 / 2 bins
    qn = synth.generate(2, 3000, seed=7, p_n=0.01)               # query-N variant
    longr = synth.generate(4, 12, seed=8)                        # long bin (cooperative kernel)
    longm = synth.generate(4, 600, seed=9)                       # cooperative kernel, several duos per block
    for mode in (sb.LOCAL, sb.EXTEND):
        for name, b, opt in (("short", short, None), ("mixed", mixed, None), ("qn", qn, None),
                             ("long", longr, None), ("long_stream", longm, None),
                             ("long_onewarp", longr, sb.Options(force_group=32)),
                             ("int32", mixed, sb.Options(force_path=1)),
                             ("G4", mixed, sb.Options(force_group=4))):
            s, qe, te, st, qst, tst = sb.align(*dev(b)[:4], dev(b)[4] if mode else None, sb.BWA_MEM, mode,
                                               options=opt)
            torch.cuda.synchronize()
            assert int(st.item()) == -1
            check(b, (s, qe, te), mode, f"{name} mode={mode}")
    # PACK2
    d = dev(mixed)
    s, qe, te, st, _, _ = sb.align(*d[:4], None, sb.BWA_MEM, sb.LOCAL, fmt=sb.PACK2)
    torch.cuda.synchronize()
    check(mixed, (s, qe, te), sb.LOCAL, "pack2")
    # banded (int32 BAND kernel) and start coordinates
    qw, qwo, ql, _ = sb.pack(d[0], d[1])
    tw, two, tl, _ = sb.pack(d[2], d[3])
    w = torch.full((mixed.n,), 40, dtype=torch.int32, device="cuda")
    bs, bq, bt, bst = sb.align_banded(qw, qwo[:-1], ql, tw, two[:-1], tl, w, None, sb.BWA_MEM, sb.LOCAL)
    torch.cuda.synchronize()
    ref = oracle.banded_batch(mixed, np.full(mixed.n, 40, np.int32))
    assert np.array_equal(bs.cpu().numpy(), ref[0]) and int(bst.item()) == -1
    print("ok banded", flush=True)
    s, qe, te, _ = sb.align_batch(qw, qwo[:-1], ql, tw, two[:-1], tl, None, sb.BWA_MEM, sb.LOCAL)
    q0, t0, sst = sb.locate_start(qw, qwo[:-1], tw, two[:-1], s, qe, te)
    torch.cuda.synchronize()
    assert int(sst.item()) == -1
    print("ok start", flush=True)
    # A5: partition + reassembly
    owner = sb.partition(ql, tl, 3)
    parts = torch.stack([torch.stack([s, qe, te])] * 3)
    idx = torch.full((3, mixed.n), -1, dtype=torch.int32, device="cuda")
    for r in range(3):
        m = torch.nonzero(owner == r).flatten()
        idx[r, :m.numel()] = m.int()
        parts[r, :, :m.numel()] = torch.stack([s, qe, te])[:, m]
    out, sst = sb.scatter_results(parts, idx, mixed.n)
    torch.cuda.synchronize()
    assert int(sst.item()) == -1 and torch.equal(out, torch.stack([s, qe, te]))
    print("ok partition + scatter", flush=True)
    # NEXT-1 ksw: shared-memory rows (short) and global rows (queries > 1023 bp)
    for name, b in (("ksw short", short), ("ksw long", synth.random_pairs(20, 1100, 1500, seed=3, p_mut=0.05))):
        out, kst, _, _ = sb.ksw_align(*dev(b))
        torch.cuda.synchronize()
        ref, _ = oracle.ksw_batch(b)
        assert int(kst.item()) == -1 and np.array_equal(out.cpu().numpy(), ref), name
        print("ok", name, flush=True)
    # host entry point (pipelined slices, copy streams)
    hs, hq, ht, hst = sb.align_host(short, sb.BWA_MEM, sb.LOCAL)
    assert hst == -1
    print("ok host", flush=True)
    print("kernels launched:", sb.kernel_launches() - kernels0)


if __name__ == "__main__":
    main()
