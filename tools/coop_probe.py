"""Run one aligned batch through the library (coop on unless SALOBA_COOP_PAIRS=0) and report timing:
python tools/coop_probe.py <config> <pairs> <seed> <mode> [repeats]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2301_09310_b200 as sb  # noqa: E402
import synth  # noqa: E402

cfg, n, seed, mode = (int(x) for x in sys.argv[1:5])
reps = int(sys.argv[5]) if len(sys.argv) > 5 else 3
b = synth.generate(cfg, n, seed=seed)
d = "cuda"
args = [torch.from_numpy(x).to(d) for x in (b.q_ascii, b.q_off, b.t_ascii, b.t_off, b.h0)]
lg = torch.zeros(1, dtype=torch.int32, device=d)
bins = torch.zeros(16, dtype=torch.int32, device=d)
for r in range(reps):
    t = time.time()
    s, qe, te, st, _, _ = sb.align(args[0], args[1], args[2], args[3], args[4] if mode else None, sb.BWA_MEM, mode,
                                   options=sb.Options(bin_counts=bins, long_group=lg))
    torch.cuda.synchronize()
    print(f"rep {r}: {1e3 * (time.time() - t):.1f} ms status {int(st.item())} long_group {int(lg.item())} "
          f"bins {bins.cpu().numpy().tolist()} checksum {int(s.sum().item())}", flush=True)
