#!/usr/bin/env python
"""bench.py — GCUPS of the batched affine-gap seed-extension hot path on 1..8 B200s.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 2] [--mode local|extend]
    torchrun --nproc-per-node N bench.py --gpus N ...        (one process per GPU, NCCL)
    python bench.py --impl reference ...                      (the CPU oracle arm)

One step = one pass of the whole hot path (pack A1 -> schedule A2 -> DP A3 ->
write-back A4, + results gather to rank 0 when N > 1, A5) over one batch of synthetic input that
is already resident in HBM.  Weak scaling: every rank owns a disjoint slice of a global batch of
N x (config pairs) pairs (per-pair seeded generator, so slices are independent).  Inputs (ASCII,
~400 MB for config 2) are larger than L2, so no flush is needed between steps.

Prints ONE JSON line on rank 0 (see the keys below).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "GCUPS (cell updates/s) at 1/2/4/8 B200; fraction of int-pipe peak"
WORKLOADS = {
    1: "config1: 1k pairs, 150 bp query vs 150-250 bp target, ~5% mutations",
    2: "config2: 1M Illumina-like pairs, 150 bp reads vs 250 bp windows, 2% sub + small indels",
    3: "config3: 500k pairs, query 100-1000 bp log-uniform (load-imbalance stress)",
    4: "config4: 100k long-read pairs, 1-10 kbp, ~15% errors",
    5: "config5: 10M length-skewed pairs (Fig. 3 histograms + long tails)",
}
# Minimal ALU-pipe instructions per cell.  Per register the update needs 3 max-type
# ops (E, F, H), the substitution lookup (PRMT) and half a running-max op: 4.5 ALU-only
# instructions (max/min/PRMT have no FMA-pipe form on sm_100a; the two adds go to the FMA pipe).
# int16x2 registers carry 2 cells -> 2.25 ALU ops per cell; int32 -> 4.5.  EXTEND adds the
# dead-zero rule of its definition (D = H(i-1,j-1) + S only if H(i-1,j-1) > 0): one
# more min-type op per register, D = min(hdiag + s, lambda*hdiag) -> 5.5 per register, 2.75 per cell.
OPS_PER_CELL = {("int32", "local"): 4.5, ("int16x2", "local"): 2.25,
                ("int32", "extend"): 5.5, ("int16x2", "extend"): 2.75}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="saloba", choices=["saloba", "reference"])
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--pairs", type=int, default=None, help="pairs per GPU (default: the config's count)")
    ap.add_argument("--mode", default="local", choices=["local", "extend"])
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--start-steps", type=int, default=3, help="LOCAL: time saloba_locate_start (0: skip)")
    ap.add_argument("--no-graph", dest="graph", action="store_false",
                    help="skip timing the step replayed from a CUDA graph (N=1 extra key cuda_graph)")
    ap.add_argument("--band", type=int, default=-1, help="NEXT-2: also time saloba_align_banded with this w")
    ap.add_argument("--band-steps", type=int, default=3)
    ap.add_argument("--ksw-steps", type=int, default=3,
                    help="NEXT-1: time saloba_ksw_extend (BWA-MEM defaults) on the same packed batch (0: skip)")
    ap.add_argument("--partition", default="balanced", choices=["balanced", "equal"],
                    help="N>1: length-balanced (saloba_partition) or the paper's equal contiguous split")
    ap.add_argument("--force-group", type=int, default=0)
    ap.add_argument("--force-path", type=int, default=0)
    ap.add_argument("--keep-order", type=int, default=0)
    ap.add_argument("--i16-rows", type=int, default=0)
    ap.add_argument("--p-n", type=float, default=0.0, help="probability of N per base (real reads carry a few)")
    ap.add_argument("--grouped", action="store_true", help="config 5: components contiguous")
    ap.add_argument("--strong", action="store_true",
                    help="strong scaling: the global batch is --pairs (default: the config's count) pairs "
                         "whatever N; default is weak scaling (N x pairs)")
    ap.add_argument("--dump-results", default=None,
                    help="rank 0 saves the (3, n_total) results of the last timed step, input order (.npy)")
    ap.add_argument("--dist-backend", default="nccl", help="test hook: gloo lets several ranks share one GPU")
    return ap.parse_args()


# ---- clocks sampled during the timed region ----------------------------------------------------
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows: list[list[str]] = []
        self.proc = None
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            if self.thread:
                self.thread.join(timeout=2)

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            try:
                sm.append(float(r[0]))
                mx.append(float(r[1]))
            except (ValueError, IndexError):
                continue
            for nm, v in zip(names, r[4:8]):
                if v.strip().lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


def dist_setup(args):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        if args.impl == "saloba":
            torch.cuda.set_device(local % torch.cuda.device_count())
        dist.init_process_group(args.dist_backend if args.impl == "saloba" else "gloo")
    elif args.impl == "saloba":
        torch.cuda.set_device(0)
    return world, rank, local


def load_intpipe():
    """Measured int-pipe lane-ops/clk/SM (tools/intpipe.cu, profiles/intpipe_b200.json)."""
    path = os.path.join(ROOT, "profiles", "intpipe_b200.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return float(d["alu_lane_ops_per_clk_per_sm"]), "measured ALU pipe rate (profiles/intpipe_b200.json)"
    except Exception:
        return 64.0, "guide: alu pipe rt_SMSP=2 -> 16 lanes/clk/SMSP x 4 (B300_MICROARCH.md)"


def cpu_baseline(batch, mode, seconds):
    import oracle  # the oracle, as it stands (cpu_baseline leg)

    r = oracle.timed_sample(batch, seconds=seconds, mode=mode)
    r1 = oracle.timed_sample(batch, seconds=min(4.0, seconds / 3), mode=mode, threads=1)
    model = ""
    try:
        model = next(l.split(":", 1)[1].strip() for l in open("/proc/cpuinfo") if l.startswith("model name"))
    except Exception:  # noqa: BLE001
        pass
    return {"value": round(r["gcups"], 4), "unit": "GCUPS", "cores": r["threads"], "kind": "oracle",
            "single_core_gcups": round(r1["gcups"], 4), "cpu_model": model, "nproc": os.cpu_count(),
            "sample": f"first {r['pairs']} pairs of the same workload ({r['cells']:.3e} cells, "
                      f"{r['seconds']:.1f} s, full-matrix C oracle, {r['threads']} threads; single core "
                      f"{r1['seconds']:.1f} s)"}


def run_reference(args, world, rank):
    """--impl reference: the CPU oracle on the host cores, as it stands, on a bounded sample."""
    import synth

    if rank != 0:
        return
    mode = 0 if args.mode == "local" else 1
    n_sample = 20_000 if args.config in (1, 2, 3, 5) else 200
    b = synth.generate(args.config, min(n_sample, args.pairs or synth.CONFIG_PAIRS[args.config]), seed=args.config)
    per_step = max(2.0, min(8.0, 150.0 / max(1, args.steps + args.warmup)))
    import oracle

    for _ in range(args.warmup):
        oracle.timed_sample(b, seconds=per_step / 4, mode=mode)
    vals, cells, secs, thr, pairs = [], 0, 0.0, 0, 0
    for _ in range(args.steps):
        r = oracle.timed_sample(b, seconds=per_step, mode=mode)
        vals.append(r["gcups"])
        cells += r["cells"]
        secs += r["seconds"]
        thr = r["threads"]
        pairs += r["pairs"]
    value = cells / secs / 1e9
    line = {"metric": METRIC, "impl": "reference", "value": round(value, 4), "unit": "GCUPS", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(1e3 * secs / args.steps, 2),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int32",
            "data": "synthetic", "config": {"workload": WORKLOADS[args.config], "mode": args.mode,
                                            "sample": f"bounded prefix of the workload per step (~{per_step:.0f} s)"},
            "cpu_baseline": {"value": round(value, 4), "unit": "GCUPS", "cores": thr, "kind": "oracle",
                             "sample": f"{pairs} pairs over {args.steps} steps"},
            "e2e": {"value": round(value, 4), "unit": "GCUPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    world, rank, local = dist_setup(args)
    if args.impl == "reference":
        run_reference(args, world, rank)
        return
    import numpy as np
    import torch
    import torch.distributed as dist

    import build_native

    if rank == 0 or world == 1:
        build_native.build_all()
    if world > 1:
        dist.barrier()
    import paper_2301_09310_b200 as sb
    import synth

    cfg = args.config
    n = args.pairs or synth.CONFIG_PAIRS[cfg]
    mode = sb.LOCAL if args.mode == "local" else sb.EXTEND
    dev = torch.device("cuda", torch.cuda.current_device())

    # this rank's slice of the global batch, generated straight into pinned host memory
    pinned = {}

    def alloc(name, nbytes):
        t = torch.empty(max(nbytes, 1), dtype=torch.uint8, pin_memory=True)
        pinned[name] = t
        return t.numpy()[:nbytes]

    t0 = time.time()
    # weak scaling (default): every rank owns `n` pairs of a world*n-pair global batch; strong
    # scaling (--strong): the global batch is `n` pairs whatever the world size
    n_total = n if args.strong else world * n
    partition_desc = "single GPU"
    from paper_2301_09310_b200 import dist as sd

    if world > 1 and args.partition == "balanced":
        # A5: every rank computes the same length-balanced partition of the global
        # batch on its own GPU (saloba_partition: cost sort + snake deal; deterministic, so no
        # collective) and generates only the pairs it owns.
        gql, gtl, _ = synth.shapes(cfg, n_total, seed=cfg, grouped=args.grouped)
        owner = sd.balanced_partition(gql, gtl, world)
        index_of_rank = [np.nonzero(owner == r)[0] for r in range(world)]
        cost = sd.pair_cost(gql, gtl)
        partition_desc = f"length-balanced snake over {world} ranks (saloba_partition), modelled max/mean {sd.imbalance(cost, owner, world):.4f}"
        batch = synth.generate_idx(cfg, index_of_rank[rank], n_total, seed=cfg, grouped=args.grouped, p_n=args.p_n,
                                   out=alloc)
        del gql, gtl, owner, cost
    else:
        if world > 1:
            partition_desc = f"equal contiguous split over {world} ranks"
        ranges = [sd.shard_range(n_total, world, r) for r in range(world)]
        index_of_rank = [np.arange(a_, b_) for a_, b_ in ranges]
        a_, b_ = ranges[rank]
        batch = synth.generate(cfg, b_ - a_, seed=cfg, first=a_, n_total=n_total, grouped=args.grouped, p_n=args.p_n,
                               out=alloc)
    counts = [len(ix) for ix in index_of_rank]
    n = batch.n  # pairs on this rank
    gen_s = time.time() - t0
    cells_rank = batch.cells()
    total_cells = cells_rank
    if world > 1:
        tc = torch.tensor([cells_rank], dtype=torch.int64, device=dev if args.dist_backend == "nccl" else "cpu")
        dist.all_reduce(tc)
        total_cells = int(tc[0])
    max_q = int(batch.qlen.max())
    qa = torch.from_numpy(batch.q_ascii).to(dev)
    ta = torch.from_numpy(batch.t_ascii).to(dev)
    qo = torch.from_numpy(batch.q_off).to(dev)
    to = torch.from_numpy(batch.t_off).to(dev)
    h0 = torch.from_numpy(batch.h0).to(dev)
    opts = sb.Options(args.force_group, args.force_path, args.keep_order, i16_rows=args.i16_rows)
    al = sb.Aligner(n, int(batch.q_off[-1]), int(batch.t_off[-1]), max_q, sb.BWA_MEM, mode, sb.PACK4, opts)
    stream = torch.cuda.current_stream()
    gather_buf = None
    nmax = max(counts)
    send_buf = torch.full((3, nmax), -9, dtype=torch.int32, device=dev) if world > 1 else None
    full_out = full_status = index_dev = None
    if world > 1 and rank == 0:
        # A5 reassembly on rank 0: the gathered shards (world, 3, nmax) go back to input order by
        # saloba_scatter_results, with each column's global index (-1 = padding)
        gathered = torch.empty((world, 3, nmax), dtype=torch.int32, device=dev)
        gather_buf = list(gathered.unbind(0))
        idx_host = np.full((world, nmax), -1, np.int32)
        for r, ix in enumerate(index_of_rank):
            idx_host[r, :len(ix)] = ix
        index_dev = torch.from_numpy(idx_host).to(dev)
        full_out = torch.full((3, n_total), -9, dtype=torch.int32, device=dev)

    bins = torch.zeros(16, dtype=torch.int32, device=dev)
    long_group = torch.zeros(1, dtype=torch.int32, device=dev)

    gather_events = []

    full_status = None

    def step(dp_ev=None):
        o = sb.Options(args.force_group, args.force_path, args.keep_order, dp_ev, bins, args.i16_rows,
                       long_group) if dp_ev else None
        s, qe, te = al.run(qa, qo, ta, to, h0, options=o)
        if world > 1:  # A5: results gathered to rank 0 (the only collective; none inside the DP)
            if dp_ev:
                ge = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                ge[0].record(stream)
                gather_events.append(ge)
            send_buf[:, :n].copy_(al.out[:, :n])  # ranks own different counts: padded to the max
            if args.dist_backend == "nccl":
                dist.gather(send_buf, gather_buf if rank == 0 else None, dst=0)
            else:  # gloo test hook: host copies
                host = [torch.empty((3, nmax), dtype=torch.int32) for _ in range(world)] if rank == 0 else None
                dist.gather(send_buf.cpu(), host, dst=0)
                if rank == 0:
                    gathered.copy_(torch.stack(host))
            if rank == 0:
                nonlocal full_status
                _, full_status = sb.scatter_results(gathered, index_dev, n_total, out=full_out)
            if dp_ev:
                gather_events[-1][1].record(stream)
        return s

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    st = al.status.cpu().tolist()
    assert st[0] == -1 and st[1] == -1 and st[2] == -1, f"bad status {st}"
    if full_status is not None:
        assert int(full_status.item()) == -1 and int((full_out == -9).sum().item()) == 0, "reassembly incomplete"

    dp_events = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                 for _ in range(args.steps)]
    for e_a, e_b in dp_events:  # torch creates the CUDA events lazily: record once so they exist
        e_a.record(stream)
        e_b.record(stream)
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    launches0 = sb.kernel_launches()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ev0.record(stream)
    step_ev = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    for k in range(args.steps):
        step(dp_events[k])
        step_ev[k].record(stream)
    ev1.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    launches = sb.kernel_launches() - launches0
    clocks.stop()
    ms = ev0.elapsed_time(ev1)
    dp_ms = [a.elapsed_time(b) for a, b in dp_events]
    step_ms = [ev0.elapsed_time(step_ev[0])] + [step_ev[k - 1].elapsed_time(step_ev[k]) for k in range(1, args.steps)]
    gather_ms = sum(a.elapsed_time(b) for a, b in gather_events) / max(1, len(gather_events)) if gather_events else None
    if args.dump_results and rank == 0:  # the reassembled results of the last timed step, input order
        res = full_out if world > 1 else al.out[:, :n]
        np.save(args.dump_results, res.cpu().numpy())
    t = torch.tensor([ms, sum(dp_ms) / len(dp_ms)], dtype=torch.float64, device=dev)
    if world > 1:
        if args.dist_backend != "nccl":
            t = t.cpu()
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max, dp_ms_avg = float(t[0]), float(t[1])
    ms_per_step = ms_max / args.steps
    # per-rank balance of the measured step time (max/mean over ranks)
    balance = None
    if world > 1:
        tt = torch.tensor([ms], dtype=torch.float64, device=dev)
        if args.dist_backend != "nccl":
            tt = tt.cpu()
        allt = [torch.zeros_like(tt) for _ in range(world)]
        dist.all_gather(allt, tt)
        per = [float(x[0]) for x in allt]
        balance = round(max(per) / (sum(per) / len(per)), 4)
    value = total_cells * args.steps / (ms_max * 1e-3) / 1e9

    # ---- end-to-end through the host-buffer C-ABI entry point (H2D + pack + align + D2H) ----
    e2e = None
    if args.e2e_steps > 0:
        # every host buffer of the call pinned (include/saloba.h): ASCII (generated into pinned
        # memory above), offsets and h0 copied once into pinned arrays (outside the timed region)
        def pinned_copy(a):
            t = torch.empty(len(a), dtype=torch.from_numpy(a[:0]).dtype, pin_memory=True)
            t.numpy()[:] = a
            return t.numpy()

        hb = synth.Batch(batch.q_ascii, pinned_copy(batch.q_off), batch.t_ascii, pinned_copy(batch.t_off),
                         pinned_copy(batch.h0))
        import ctypes

        def timed(fn):
            if world > 1:
                dist.barrier()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            fn()
            e1.record(stream)
            torch.cuda.synchronize()
            te2 = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
            if world > 1:
                if args.dist_backend != "nccl":
                    te2 = te2.cpu()
                dist.all_reduce(te2, op=dist.ReduceOp.MAX)
            return total_cells * args.e2e_steps / (float(te2[0]) * 1e-3) / 1e9

        # (a) the streaming API (saloba_stream_*): two host contexts in flight, batch k+1's upload and
        # packing overlap batch k's alignment; every batch still uploads its ASCII and reads back its
        # results inside the timed region
        outs = [torch.empty((3, n), dtype=torch.int32, pin_memory=True).numpy() for _ in range(2)]
        sts = [ctypes.c_int64(0), ctypes.c_int64(0)]
        hs = sb.HostStream(n, len(batch.q_ascii), len(batch.t_ascii), max_q)
        hs.submit(hb, outs[0], sts[0], sb.BWA_MEM, mode, opts)  # warm
        hs.wait()

        def stream_steps():
            for k in range(args.e2e_steps):
                hs.submit(hb, outs[k & 1], sts[k & 1], sb.BWA_MEM, mode, opts)
            hs.wait()

        e2e_val = timed(stream_steps)
        assert all(sts[k].value == -1 for k in range(min(2, args.e2e_steps))), [x.value for x in sts]
        hs.close()
        # (b) one synchronous call per batch (saloba_align_host_ctx, 4 pipelined slices inside a batch)
        out = outs[0]
        hctx = sb.HostContext(n, len(batch.q_ascii), len(batch.t_ascii), max_q)
        sb.align_host(hb, sb.BWA_MEM, mode, opts, out=out, ctx=hctx)  # warm
        e2e_sync = timed(lambda: [sb.align_host(hb, sb.BWA_MEM, mode, opts, out=out, ctx=hctx)
                                  for _ in range(args.e2e_steps)])
        hctx.close()
        h2d = int(len(batch.q_ascii) + len(batch.t_ascii) + 16 * (n + 1) + (4 * n if mode == sb.EXTEND else 0))
        e2e = {"value": round(e2e_val, 2), "unit": "GCUPS", "h2d_bytes_per_step": h2d * world,
               "d2h_bytes_per_step": 12 * n * world,
               "api": "saloba_stream_submit/_wait (pinned host ASCII in, host results out; two batches in flight)",
               "sync_call_value": round(e2e_sync, 2),
               "sync_call_api": "saloba_align_host_ctx (one blocking call per batch, 4 pipelined slices)"}

    # ---- optional: the same step captured once into a CUDA graph and replayed (launch-bound batches) ----
    graph = None
    if args.graph and world == 1:
        g = al.capture(qa, qo, ta, to, h0)
        torch.cuda.synchronize()
        g.replay()
        torch.cuda.synchronize()
        assert al.status.cpu().tolist()[:3] == [-1, -1, -1]
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        g0.record(stream)
        for _ in range(args.steps):
            g.replay()
        g1.record(stream)
        torch.cuda.synchronize()
        gms = g0.elapsed_time(g1) / args.steps
        graph = {"ms_per_step": round(gms, 4), "value": round(cells_rank / (gms * 1e-3) / 1e9, 2),
                 "what": "pack + schedule + DP of one step captured once as a CUDA graph, replayed"}

    # ---- NEXT-3: start coordinates of the same LOCAL results (saloba_locate_start), timed alone ----
    start_pass = None
    if mode == sb.LOCAL and args.start_steps > 0:
        n_ = al.n
        s_, qe_, te_ = al.out[0, :n_], al.out[1, :n_], al.out[2, :n_]
        sws = torch.empty(sb.start_workspace_bytes(n_, al.q_words.numel(), al.t_words.numel(), max_q, dev.index),
                          dtype=torch.uint8, device=dev)
        sout = torch.empty((2, n_), dtype=torch.int32, device=dev)
        args_s = (al.q_words, al.q_word_off[:-1], al.t_words, al.t_word_off[:-1], s_, qe_, te_, sb.BWA_MEM, sb.PACK4)
        _, _, sst = sb.locate_start(*args_s, out=sout, workspace=sws)  # warm
        torch.cuda.synchronize()
        assert int(sst.item()) == -1
        pc = int(((qe_.long() + 1) * (te_.long() + 1) * (s_ > 0).long()).sum().item())
        l0 = sb.kernel_launches()
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s0.record(stream)
        for _ in range(args.start_steps):
            sb.locate_start(*args_s, out=sout, workspace=sws)
        s1.record(stream)
        torch.cuda.synchronize()
        sms_ = s0.elapsed_time(s1) / args.start_steps
        start_pass = {"ms_per_call": round(sms_, 3), "prefix_cells": pc,
                      "gcups_prefix_cells": round(pc / (sms_ * 1e-3) / 1e9, 2),
                      "forward_plus_start_gcups": round(cells_rank / ((ms_per_step + sms_) * 1e-3) / 1e9, 2),
                      "launches_per_call": (sb.kernel_launches() - l0) // args.start_steps,
                      "api": "saloba_locate_start (reversed prefixes through the same DP kernels)"}

    # ---- NEXT-2: banded DP over the same packed batch (saloba_align_banded), timed alone ----
    banded = None
    if args.band >= 0:
        n_ = al.n
        wd = torch.full((n_,), args.band, dtype=torch.int32, device=dev)
        bout = torch.empty((3, n_), dtype=torch.int32, device=dev)
        bargs = (al.q_words, al.q_word_off[:-1], al.q_len[:n_], al.t_words, al.t_word_off[:-1], al.t_len[:n_], wd,
                 h0 if mode == sb.EXTEND else None, sb.BWA_MEM, mode, sb.PACK4)
        _, _, _, bst = sb.align_banded(*bargs, out=bout, workspace=al.ws)  # warm
        torch.cuda.synchronize()
        assert int(bst.item()) == -1
        ql_, tl_ = batch.qlen.astype(np.int64), batch.tlen.astype(np.int64)
        band_cells = 0
        for d in range(-args.band, args.band + 1):  # cells on diagonal j - i = d inside the table
            band_cells += int(np.maximum(0, np.minimum(tl_, ql_ - d) - max(0, -d)).sum())
        l0 = sb.kernel_launches()
        b0, b1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        b0.record(stream)
        for _ in range(args.band_steps):
            sb.align_banded(*bargs, out=bout, workspace=al.ws)
        b1.record(stream)
        torch.cuda.synchronize()
        bms = b0.elapsed_time(b1) / args.band_steps
        banded = {"band_w": args.band, "ms_per_call": round(bms, 3), "band_cells": band_cells,
                  "gcups_band_cells": round(band_cells / (bms * 1e-3) / 1e9, 2),
                  "full_table_cells": cells_rank,
                  "speedup_vs_unbanded_step": round(ms_per_step / bms, 3),
                  "launches_per_call": (sb.kernel_launches() - l0) // args.band_steps,
                  "api": "saloba_align_banded (int16x2 G = 1 kernel with per-strip band step ranges for short reads, exact int32 kernel for long or wide-band ones)"}

    # ---- NEXT-1: BWA-MEM-compatible extension over the same packed batch (saloba_ksw_extend) ----
    ksw = None
    if args.ksw_steps > 0:
        n_ = al.n
        kout = torch.empty((7, n_), dtype=torch.int32, device=dev)
        kws = torch.empty(int(sb.lib().saloba_ksw_workspace_bytes(n_, max_q, dev.index)), dtype=torch.uint8,
                          device=dev)
        kargs = (al.q_words, al.q_word_off[:-1], al.q_len[:n_], al.t_words, al.t_word_off[:-1], al.t_len[:n_], h0,
                 sb.BWA_KSW, sb.PACK4)
        _, kst = sb.ksw_extend(*kargs, max_qlen=max_q, out=kout, workspace=kws)  # warm
        torch.cuda.synchronize()
        assert int(kst.item()) == -1
        l0 = sb.kernel_launches()
        k0, k1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        k0.record(stream)
        for _ in range(args.ksw_steps):
            sb.ksw_extend(*kargs, max_qlen=max_q, out=kout, workspace=kws)
        k1.record(stream)
        torch.cuda.synchronize()
        kms = k0.elapsed_time(k1) / args.ksw_steps
        ksw = {"ms_per_call": round(kms, 3), "gcups_full_table": round(cells_rank / (kms * 1e-3) / 1e9, 2),
               "launches_per_call": (sb.kernel_launches() - l0) // args.ksw_steps,
               "params": "BWA-MEM defaults a1 b4 o6 e1 w100 end_bonus5 zdrop100, h0 = the batch's seed scores",
               "api": "saloba_ksw_extend (ksw_extend2 semantics: band, row trimming, z-drop, gscore; warp-per-pair row sweep)"}

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    csum = clocks.summary()
    p_int, p_src = load_intpipe()
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    f_mhz = csum["sm_mhz"] or 1965.0
    bc = bins.cpu().tolist()
    lg = int(long_group.item())
    n16, n32 = sum(bc[8:15]) + bc[6], sum(bc[0:6]) + bc[7]  # bins 14 / 6: int16x2 G=1 / G=2 with N in the query
    path = "int16x2" if n16 >= n32 else "int32"
    opc = OPS_PER_CELL[(path, args.mode)]
    peak = sms * f_mhz * 1e6 * p_int / opc / 1e9
    achieved = cells_rank / (dp_ms_avg * 1e-3) / 1e9
    traffic = None
    try:  # DRAM bytes per launch of the dominant kernel from the committed ncu capture of this command
        tpath = os.path.join(ROOT, "profiles", "r02_dp_traffic.json")
        if not os.path.exists(tpath):
            tpath = os.path.join(ROOT, "profiles", "r01_dp_traffic.json")
        tj = json.load(open(tpath))
        if tj.get("workload") == f"config{cfg}" and tj.get("pairs") == n and args.mode == "local":
            traffic = tj["traffic_bytes_per_launch"]
    except Exception:
        pass
    roof = {"bound": "alu", "achieved": round(achieved, 2), "peak": round(peak, 2), "unit": "GCUPS",
            "frac": round(achieved / peak, 4), "traffic": traffic,
            "kernel": (("dp_g1_kernel" if bc[8] + bc[14] >= n16 / 2 else
                        "dp_coop_kernel" if lg == 6 and bc[13] else "dp_i16_kernel") if path == "int16x2"
                       else "dp_i32_kernel") + " (runs most pairs; achieved = all DP kernels of one call, CUDA events on the launching stream)",
            # bin 13 = the int16x2 long bin, run at G = 2^long_group (16 or 32) this call, or (6) on the
            # cooperative kernel (several warps per duo)
            "bins": {("i16_G1_queryN" if b == 14 else "i16_G2_queryN" if b == 6 else
                      (f"{'i16' if b >= 8 else 'i32'}_G{1 << (lg if b == 13 else b % 8)}{'_long' if b == 13 else ''}" if not (b == 13 and lg == 6) else "i16_long_coop")): c
                     for b, c in enumerate(bc) if c and b != 15},
            "dp_share_of_step": round(dp_ms_avg / ms_per_step, 3),
            "peak_derivation": f"{sms} SMs x {f_mhz:.0f} MHz (median under load) x {p_int:.0f} int lane-ops/clk/SM "
                               f"[{p_src}] / {opc} ALU ops per cell ({path} path, {args.mode} mode)"}
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(batch, mode, args.cpu_seconds)
    line = {
        "metric": METRIC, "value": round(value, 2), "unit": "GCUPS", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms_per_step, 3), "higher_is_better": True,
        "scaling": "strong" if args.strong else "weak", "vs_baseline": None, "dtype": path, "data": "synthetic",
        "step_ms": {"min": round(min(step_ms), 3), "median": round(float(np.median(step_ms)), 3),
                    "max": round(max(step_ms), 3), "rank": 0},
        "comms": None if gather_ms is None else {"gather_ms_per_step": round(gather_ms, 3),
                                                  "share_of_step": round(gather_ms / ms_per_step, 4),
                                                  "what": "NCCL gather of 12 B per pair to rank 0 + saloba_scatter_results back to input order (rank-0 stream)"},
        "config": {"workload": WORKLOADS[cfg], "mode": args.mode, "pairs_per_gpu": n,
                   "cells_per_step": total_cells, "scoring": "match 1, mismatch -4, alpha 7, beta 1 (BWA-MEM-style)",
                   "l2": "inputs larger than L2 (ASCII %.0f MB per GPU per step)" % ((len(batch.q_ascii) + len(batch.t_ascii)) / 1e6),
                   "parallelism": f"pairs sharded over {world} GPU(s), results gathered to rank 0 and put back in input order",
                   "pairs_total": n_total,
                   "partition": partition_desc, "measured_rank_balance_max_over_mean": balance,
                   "gen_seconds": round(gen_s, 1)},
        "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": int(launches),
        "start_pass": start_pass, "banded": banded, "ksw_extend": ksw, "cuda_graph": graph,
        "clocks": {"sm_mhz": csum["sm_mhz"], "sm_max_mhz": csum["sm_max_mhz"], "reasons": csum["reasons"]},
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
