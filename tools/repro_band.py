"""Search seeds of one stress configuration for a banded-parity mismatch and dump the failing batch.
python tools/repro_band.py <seconds> [cfg n pN match mismatch go ge mode G path band]"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
import paper_2301_09310_b200 as sb  # noqa: E402
import synth  # noqa: E402

budget = float(sys.argv[1])
cfg, n, pn, ma, mm, go, ge, mode, G, fp, band = (2, 20000, 0.002, 3, -2, 7, 3, 1, 32, 2, 40)
if len(sys.argv) > 2:
    a = sys.argv[2:]
    cfg, n, pn, ma, mm, go, ge, mode, G, fp, band = (int(a[0]), int(a[1]), float(a[2]), int(a[3]), int(a[4]),
                                                     int(a[5]), int(a[6]), int(a[7]), int(a[8]), int(a[9]), int(a[10]))
sc = sb.Scoring(ma, mm, go, ge)
d = "cuda"
t_end = time.time() + budget
seed = 0
while time.time() < t_end:
    seed += 1
    rng = np.random.default_rng(seed)
    b = synth.generate(cfg, n, seed=seed, p_n=pn)
    b.h0[:] = rng.integers(1, 80, b.n).astype(np.int32)
    qa, qo = torch.from_numpy(b.q_ascii).to(d), torch.from_numpy(b.q_off).to(d)
    ta, to = torch.from_numpy(b.t_ascii).to(d), torch.from_numpy(b.t_off).to(d)
    qw, qwo, ql, _ = sb.pack(qa, qo, 4)
    tw, two, tl, _ = sb.pack(ta, to, 4)
    h0 = torch.from_numpy(b.h0).to(d) if mode else None
    w = np.full(b.n, band, np.int32)
    s, qe, te, st = sb.align_banded(qw, qwo[:-1], ql, tw, two[:-1], tl, torch.from_numpy(w).to(d), h0, sc, mode, 4,
                                    options=sb.Options(force_group=G, force_path=fp))
    torch.cuda.synchronize()
    ref = oracle.banded_batch(b, w, ma, mm, go, ge, mode)
    got = [x.cpu().numpy() for x in (s, qe, te)]
    bad = np.nonzero((got[0] != ref[0]) | (got[1] != ref[1]) | (got[2] != ref[2]))[0]
    print(f"seed {seed}: bad {len(bad)}", flush=True)
    if len(bad):
        for k in bad[:8]:
            print("  k", int(k), "gpu", [int(x[k]) for x in got], "oracle", [int(x[k]) for x in ref[:3]], "h0", int(b.h0[k]))
        os.makedirs("gpurun_out", exist_ok=True)
        np.savez("gpurun_out/repro_band.npz", q_ascii=b.q_ascii, q_off=b.q_off, t_ascii=b.t_ascii, t_off=b.t_off,
                 h0=b.h0, bad=bad, seed=seed)
        break
