"""Replay gpurun_out/repro_band.npz (tools/repro_band.py) under variations to isolate a mismatch."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
import paper_2301_09310_b200 as sb  # noqa: E402
import synth  # noqa: E402

z = np.load(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "build", "repro_band.npz"))
b = synth.Batch(z["q_ascii"], z["q_off"], z["t_ascii"], z["t_off"], z["h0"])
bad0 = [int(x) for x in z["bad"]]
sc = sb.Scoring(3, -2, 7, 3)
d = "cuda"


def run(batch, kw, band=40):
    qa, qo = torch.from_numpy(batch.q_ascii).to(d), torch.from_numpy(batch.q_off).to(d)
    ta, to = torch.from_numpy(batch.t_ascii).to(d), torch.from_numpy(batch.t_off).to(d)
    qw, qwo, ql, _ = sb.pack(qa, qo, 4)
    tw, two, tl, _ = sb.pack(ta, to, 4)
    w = np.full(batch.n, band, np.int32)
    bins = torch.zeros(16, dtype=torch.int32, device=d)
    opt = sb.Options(bin_counts=bins, **kw)
    s, qe, te, st = sb.align_banded(qw, qwo[:-1], ql, tw, two[:-1], tl, torch.from_numpy(w).to(d),
                                    torch.from_numpy(batch.h0).to(d), sc, 1, 4, options=opt)
    torch.cuda.synchronize()
    ref = oracle.banded_batch(batch, w, 3, -2, 7, 3, 1)
    got = [x.cpu().numpy() for x in (s, qe, te)]
    bad = np.nonzero((got[0] != ref[0]) | (got[1] != ref[1]) | (got[2] != ref[2]))[0]
    return [int(k) for k in bad], bins.cpu().tolist(), got, ref


for name, opt in (("G32 path2", dict(force_group=32, force_path=2)), ("auto", dict()),
                  ("path2", dict(force_path=2)), ("keep_order path2", dict(force_path=2, keep_order=1))):
    bad, bins, got, ref = run(b, opt)
    print(name, "bad", bad[:6], "bins", bins, flush=True)
k = bad0[0]
print("pair", k, "qlen", len(b.pair(k)[0]), "tlen", len(b.pair(k)[1]), "h0", int(b.h0[k]))
# the pair with each neighbour in input order (keep_order: duo = (2i, 2i+1) of the bin)
for lo in (k - 1, k):
    idx = [lo, lo + 1]
    sub = b.subset(idx)
    bad, bins, got, ref = run(sub, dict(force_path=2, keep_order=1))
    print("duo", idx, "bad", bad, "got", [list(map(int, x)) for x in got], "ref", [list(map(int, x)) for x in ref[:3]],
          "h0", [int(b.h0[i]) for i in idx], "bins", bins)
sub = b.subset([k])
bad, bins, got, ref = run(sub, dict(force_path=2))
print("alone bad", bad, "got", [list(map(int, x)) for x in got], "ref", [list(map(int, x)) for x in ref[:3]])
