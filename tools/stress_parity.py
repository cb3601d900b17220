"""Randomised parity stress on the GPU box (not part of the pytest suite: minutes of oracle time).
Every round draws a random workload (config shape, N rate, scheme, mode, forced G / path, band,
PACK2) and compares the CUDA path with the oracle on every pair; prints one line per round and
exits non-zero on the first mismatch.   python tools/stress_parity.py [seconds]"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402  (test infrastructure)
import paper_2301_09310_b200 as sb  # noqa: E402
import synth  # noqa: E402

budget = float(sys.argv[1]) if len(sys.argv) > 1 else 240.0
rng = np.random.default_rng(int(time.time()) & 0xFFFF)
t_end = time.time() + budget
rounds = 0
d = "cuda"
while time.time() < t_end:
    rounds += 1
    cfg = int(rng.choice([1, 2, 3, 4]))
    n = {1: 1000, 2: 20000, 3: 5000, 4: 60}[cfg]
    p_n = float(rng.choice([0.0, 0.0, 0.002, 0.02]))
    b = synth.generate(cfg, n, seed=int(rng.integers(1 << 30)), p_n=p_n)
    beta = int(rng.integers(1, 4))
    sc = sb.Scoring(int(rng.integers(1, 5)), int(rng.integers(-6, 0)), int(rng.integers(beta, 9)), beta)
    mode = int(rng.integers(0, 2))
    b.h0[:] = rng.integers(1, 80, b.n).astype(np.int32)
    G = int(rng.choice([0, 0, 1, 2, 4, 8, 16, 32]))
    fp = int(rng.choice([0, 0, 0, 1, 2]))
    fmt = 2 if (p_n == 0.0 and rng.random() < 0.2) else 4
    band = int(rng.choice([-1, -1, -1, 0, 5, 16, 40, 100])) if cfg <= 3 else -1  # banded oracle is full-matrix
    qa, qo = torch.from_numpy(b.q_ascii).to(d), torch.from_numpy(b.q_off).to(d)
    ta, to = torch.from_numpy(b.t_ascii).to(d), torch.from_numpy(b.t_off).to(d)
    qw, qwo, ql, _ = sb.pack(qa, qo, fmt)
    tw, two, tl, _ = sb.pack(ta, to, fmt)
    h0 = torch.from_numpy(b.h0).to(d) if mode else None
    opt = sb.Options(force_group=G, force_path=fp)
    if band >= 0:
        w = np.full(b.n, band, np.int32)
        s, qe, te, st = sb.align_banded(qw, qwo[:-1], ql, tw, two[:-1], tl, torch.from_numpy(w).to(d), h0, sc, mode,
                                        fmt, options=opt)
        ref = oracle.banded_batch(b, w, sc.match, sc.mismatch, sc.gap_open, sc.gap_extend, mode)
    else:
        s, qe, te, st = sb.align_batch(qw, qwo[:-1], ql, tw, two[:-1], tl, h0, sc, mode, fmt, options=opt)
        ref = oracle.align_batch(b, sc.match, sc.mismatch, sc.gap_open, sc.gap_extend, mode)
    torch.cuda.synchronize()
    got = [x.cpu().numpy() for x in (s, qe, te)]
    bad = np.nonzero((got[0] != ref[0]) | (got[1] != ref[1]) | (got[2] != ref[2]))[0]
    desc = f"cfg{cfg} n={n} pN={p_n} {sc.match},{sc.mismatch},{sc.gap_open},{sc.gap_extend} mode={mode} G={G} path={fp} fmt={fmt} band={band}"
    if len(bad) or int(st.item()) != -1:
        k = int(bad[0]) if len(bad) else -1
        print(f"MISMATCH round {rounds}: {desc} status={int(st.item())} bad={len(bad)} first={k}", flush=True)
        if k >= 0:
            print("  gpu", [int(x[k]) for x in got], "oracle", [int(x[k]) for x in ref[:3]], b.pair(k), int(b.h0[k]))
        sys.exit(1)
    # start coordinates for LOCAL unbanded rounds
    if mode == 0 and band < 0:
        qs, ts, st2 = sb.locate_start(qw, qwo[:-1], tw, two[:-1], s, qe, te, sc, fmt, options=opt)
        torch.cuda.synchronize()
        rs = oracle.start_batch(b, sc.match, sc.mismatch, sc.gap_open, sc.gap_extend)
        if not (np.array_equal(qs.cpu().numpy(), rs[3]) and np.array_equal(ts.cpu().numpy(), rs[4])):
            print(f"START MISMATCH round {rounds}: {desc}", flush=True)
            sys.exit(1)
    print(f"ok round {rounds}: {desc}", flush=True)
print(f"stress: {rounds} rounds, no mismatch")
