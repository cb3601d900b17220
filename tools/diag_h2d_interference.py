"""Does a concurrent pinned H2D stream slow the DP step?  Times the bench step alone and with a
400 MB host->device copy looping on another stream."""
import sys, threading, time, torch
sys.path.insert(0, '.')
import synth, paper_2301_09310_b200 as sb
n = 1_000_000
b = synth.generate(2, n)
d = 'cuda'
qa, qo = torch.from_numpy(b.q_ascii).to(d), torch.from_numpy(b.q_off).to(d)
ta, to = torch.from_numpy(b.t_ascii).to(d), torch.from_numpy(b.t_off).to(d)
al = sb.Aligner(n, len(b.q_ascii), len(b.t_ascii), 150)
host = torch.empty(400_000_000, dtype=torch.uint8, pin_memory=True)
dev = torch.empty_like(host, device=d)
cs = torch.cuda.Stream()
def run(k, copy):
    for _ in range(2): al.run(qa, qo, ta, to)
    torch.cuda.synchronize()
    if copy:
        with torch.cuda.stream(cs):
            for _ in range(4): dev.copy_(host, non_blocking=True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(k): al.run(qa, qo, ta, to)
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / k
for copy in (False, True, False, True):
    print(f"copy={copy}: {run(3, copy):.3f} ms per step")
