"""Probe the banded routing: bins taken and time per call, per force_path (usage: cfg n [fp...])."""
import sys, torch
sys.path.insert(0, '.')
import synth, paper_2301_09310_b200 as sb
torch.cuda.set_device(0)
cfg, n = int(sys.argv[1]), int(sys.argv[2])
fps = [int(x) for x in sys.argv[3:]] or [0, 2]
b = synth.generate(cfg, n)
d = 'cuda'
qa, qo = torch.from_numpy(b.q_ascii).to(d), torch.from_numpy(b.q_off).to(d)
ta, to = torch.from_numpy(b.t_ascii).to(d), torch.from_numpy(b.t_off).to(d)
qw, qwo, ql, _ = sb.pack(qa, qo)
tw, two, tl, _ = sb.pack(ta, to)
w = torch.full((b.n,), 100, dtype=torch.int32, device=d)
for fp in fps:
    bins = torch.zeros(16, dtype=torch.int32, device=d)
    s, qe, te, st = sb.align_banded(qw, qwo[:-1], ql, tw, two[:-1], tl, w, None, sb.BWA_MEM, sb.LOCAL, options=sb.Options(force_path=fp, bin_counts=bins))
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        sb.align_banded(qw, qwo[:-1], ql, tw, two[:-1], tl, w, None, sb.BWA_MEM, sb.LOCAL, options=sb.Options(force_path=fp))
    e1.record(); torch.cuda.synchronize()
    print(cfg, n, 'force_path', fp, 'bins', bins.cpu().tolist(), 'ms', e0.elapsed_time(e1)/3, flush=True)
