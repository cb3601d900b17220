"""Diagnose the host-buffer path: raw pinned H2D bandwidth vs the e2e call."""
import sys, time, torch
sys.path.insert(0, '.')
import synth, paper_2301_09310_b200 as sb
n = 1_000_000
pinned = {}
def alloc(name, nb):
    t = torch.empty(max(nb, 1), dtype=torch.uint8, pin_memory=True); pinned[name] = t; return t.numpy()[:nb]
b = synth.generate(2, n, out=alloc)
def pc(a):
    t = torch.empty(len(a), dtype=torch.from_numpy(a[:0]).dtype, pin_memory=True); t.numpy()[:] = a; return t.numpy()
b = synth.Batch(b.q_ascii, pc(b.q_off), b.t_ascii, pc(b.t_off), pc(b.h0))
dq = torch.empty(len(b.q_ascii), dtype=torch.uint8, device='cuda')
dt = torch.empty(len(b.t_ascii), dtype=torch.uint8, device='cuda')
for _ in range(2):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    dq.copy_(pinned['q'][:len(b.q_ascii)], non_blocking=True); dt.copy_(pinned['t'][:len(b.t_ascii)], non_blocking=True)
    torch.cuda.synchronize(); t1 = time.perf_counter()
print(f"H2D {(len(b.q_ascii)+len(b.t_ascii))/1e6:.0f} MB in {1e3*(t1-t0):.2f} ms -> {(len(b.q_ascii)+len(b.t_ascii))/(t1-t0)/1e9:.1f} GB/s")
ctx = sb.HostContext(n, len(b.q_ascii), len(b.t_ascii), 150)
out = torch.empty((3, n), dtype=torch.int32, pin_memory=True).numpy()
for _ in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    sb.align_host(b, sb.BWA_MEM, sb.LOCAL, out=out, ctx=ctx)
    t1 = time.perf_counter()
    print(f"e2e {1e3*(t1-t0):.2f} ms -> {b.cells()/(t1-t0)/1e12:.2f} TCUPS")
