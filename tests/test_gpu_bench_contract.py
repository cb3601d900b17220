"""bench.py's JSON line keeps the driver contract (keys, types, units) and the CUDA-graph replay of a
step reproduces the stream-launched results bit for bit."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_line_contract():
    cmd = [sys.executable, "bench.py", "--pairs", "50000", "--steps", "3", "--warmup", "3", "--cpu-seconds", "1",
           "--e2e-steps", "1", "--start-steps", "1"]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-2000:]
    d = json.loads([l for l in r.stdout.splitlines() if l.startswith("{")][-1])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e", "gpu_launches", "clocks"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] == 3 and d["higher_is_better"] is True
    assert d["unit"] == "GCUPS" and d["value"] > 0 and "workload" in d["config"]
    roof = d["roofline"]
    assert roof["bound"] == "alu" and 0 < roof["frac"] < 1 and roof["peak"] > roof["achieved"] > 0
    cpu = d["cpu_baseline"]
    assert cpu["kind"] == "oracle" and cpu["cores"] >= 1 and cpu["value"] > 0
    e2e = d["e2e"]
    assert e2e["value"] > 0 and e2e["h2d_bytes_per_step"] > 0 and e2e["d2h_bytes_per_step"] == 12 * 50000
    assert d["gpu_launches"] > 0 and "sm_mhz" in d["clocks"]
    assert d["cuda_graph"]["value"] > 0 and d["start_pass"]["gcups_prefix_cells"] > 0


def test_cuda_graph_replay_matches_stream_launch():
    import torch

    import paper_2301_09310_b200 as sb

    b = synth.generate(3, 20000, seed=17, p_n=0.002)
    d = "cuda"
    qa, qo = torch.from_numpy(b.q_ascii).to(d), torch.from_numpy(b.q_off).to(d)
    ta, to = torch.from_numpy(b.t_ascii).to(d), torch.from_numpy(b.t_off).to(d)
    h0 = torch.from_numpy(b.h0).to(d)
    for mode in (sb.LOCAL, sb.EXTEND):
        al = sb.Aligner(b.n, len(b.q_ascii), len(b.t_ascii), int(b.qlen.max()), sb.BWA_MEM, mode)
        ref = [x.clone() for x in al.run(qa, qo, ta, to, h0)]
        torch.cuda.synchronize()
        al.out.fill_(-7)
        g = al.capture(qa, qo, ta, to, h0)
        torch.cuda.synchronize()
        al.out.fill_(-7)
        for _ in range(2):
            g.replay()
        torch.cuda.synchronize()
        got = [al.out[i, :b.n] for i in range(3)]
        assert all(torch.equal(x, y) for x, y in zip(ref, got)), mode
        assert al.status.cpu().tolist()[:3] == [-1, -1, -1]
