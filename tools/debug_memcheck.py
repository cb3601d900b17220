import sys, torch
sys.path.insert(0, '.')
import synth, paper_2301_09310_b200 as sb
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
n = int(sys.argv[2]) if len(sys.argv) > 2 else 20000
b = synth.generate(cfg, n, seed=9)
d = 'cuda'
args = [torch.from_numpy(x).to(d) for x in (b.q_ascii, b.q_off, b.t_ascii, b.t_off, b.h0)]
s, qe, te, st, qst, tst = sb.align(*args[:4], None, sb.BWA_MEM, 0)
torch.cuda.synchronize()
print('ok', int(st.item()), s[:5].tolist())
