#!/usr/bin/env python
"""bench.py — SparseDrop fwd+bwd on B200 (BASELINE.json metric, configs[1]).

One step = one SparseDrop linear layer training step on the hot path:
  K1+K2 mask generation + compaction (fresh draw, seed varies per step)
  K4 forward  Y  = s (X (.) m) W         (dsd, dropped K-blocks never read)
  K6 backward dW = s (X (.) m)^T dY       (dsd over mask columns)
  [N > 1: NCCL all-reduce of dW on a side stream, overlapped with dX]
  K5 backward dX = s (dY W^T) (.) m       (sdd, dropped output tiles = +0.0)
at M=N=K=4096 per GPU (configs[1]), 128x128 blocks, headline p = 0.5, with the
p = 0.0..0.9 sweep and our own dense tcgen05 fwd+bwd (same kernel, no mask) as
the speed-up denominator. Row-sharded data parallel for N > 1 (weak scaling:
each rank owns 4096 rows of M; masks are generated shard-locally from the
global block-row index, bit-identical with the global mask; W is replicated).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

--impl reference times the reference's own CPU implementation (oracle/_ref,
compiled from /root/reference, else the oracle port) on the host cores.
Prints ONE JSON line (rank 0).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "SparseDrop fwd+bwd TFLOP/s (dense-equiv) & speedup vs dense GEMM vs p"
UNIT = "TFLOP/s"
SWEEP_P = [0.0, 0.1, 0.2, 0.3, 0.4, 0.5, 0.6, 0.7, 0.8, 0.9]


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--size", type=int, default=4096, help="M (per GPU) = N = K")
    ap.add_argument("--p", type=float, default=0.5, help="headline drop rate")
    ap.add_argument("--no-sweep", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--profile", action="store_true", help="minimal run for ncu (headline loop only)")
    ap.add_argument("--preroll", type=float, default=0.3, help="seconds of sustained load before each timing")
    ap.add_argument("--rotate", type=int, default=3,
                    help="input sets cycled step to step (their combined size exceeds L2, so steps run "
                         "back-to-back without an L2 flush)")
    ap.add_argument("--dw-parts", type=int, default=None,
                    help="N>1: dW computed in this many row slabs, each all-reduced while the next slab and dX run "
                         "(default: 1 for configs[4] — one all-reduce, hidden behind dX; slabbing costs ~4%% of "
                         "compute there, profiles/r02_split_backward_ab.txt — and 2 for the weak-scaled configs[1])")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="gloo lets several ranks share one GPU (CI check of the data-parallel path)")
    ap.add_argument("--config", choices=["cfg2", "cfg5"], default=None,
                    help="cfg2 = configs[1] (4096^3 per GPU, the N=1 default); cfg5 = configs[4] (M=524288, "
                         "K=N=8192 row-sharded over the ranks, strong scaling; the N>1 default)")
    ap.add_argument("--m-global", type=int, default=524288, help="cfg5: global M (reduced only for CI tests)")
    ap.add_argument("--kn", type=int, default=8192, help="cfg5: K = N (reduced only for CI tests)")
    return ap.parse_args()


def workload_config(size, p, world, dw_parts=2):
    return {
        "workload": f"configs[1]: SparseDrop linear fwd+bwd (mask gen + dsd fwd + dsd dW + sdd dX), "
                    f"M={size}/GPU, N=K={size}, 128x128 blocks, p={p} (sweep p=0..0.9 in 'sweep')",
        "M_per_gpu": size, "N": size, "K": size, "M_global": size * world,
        "m_blk": 128, "k_blk": 128, "p": p, "seed": 0,
        "dtypes": {"x/w/dy/y/dx": "bf16", "dw": "fp32", "accumulate": "fp32"},
        "l2": "inputs larger than L2: steps rotate over several input sets whose combined footprint exceeds "
              "the 126 MB L2 (see 'timing')",
        "parallelism": (f"dp{world} row-sharded (shard-local masks, dW all-reduced in {max(1, dw_parts)} row "
                        "slabs overlapping the next slab and dX)") if world > 1 else "single GPU",
    }


# ------------------------------------------------------------------ CPU legs (reference / oracle)

def _cpu_layer_runner():
    """-> (kind, fn(x, w, dy, p, threads)) timing the reference's layer fwd+bwd."""
    import numpy as np

    from oracle.oracle import ORACLE_LIB, REF_LIB, Oracle, Reference

    if REF_LIB.exists():
        ref = Reference()

        def run(x, w, dy, p, threads):
            ref.layer_fwd_bwd(x, w, dy, p, 128, 128, 128, seed=0, step_seed=0, layer_index=0, threads=threads,
                              dtype=np.float32)

        return "reference", run
    if not ORACLE_LIB.exists():
        subprocess.run(["make", "-C", str(ROOT / "oracle"), "all"], check=True, stdout=subprocess.DEVNULL)
    o = Oracle()

    def run(x, w, dy, p, threads):
        eff = o.effective_seed(0, 0, 0)
        words, _ = o.sample_mask(p, 128, 128, eff, x.shape[0], x.shape[1])
        s = 1.0 / (1.0 - p)
        o.dsd_matmul(x, words, w, 128, 128, 128, s, threads=threads)
        o.layer_dw(x, dy, words, 128, 128, s, threads=threads)
        o.layer_dx(dy, w, words, 128, 128, s, threads=threads)

    return "port", run


def cpu_sample_inputs(size, n_slab):
    """The configs[1] problem restricted to an N-column slab: M=K=size, N=n_slab.
    Work is linear in N, and the reference's tile-row parallelism (M/128 rows for
    fwd/dX, K/128 for dW) is unchanged by the slab."""
    from oracle.oracle import Oracle

    o = Oracle()
    bf = lambda r, c, s: o.bf16_bits_to_f64(o.to_bf16_bits(o.random_matrix(r, c, s))).astype("float32")
    return bf(size, size, 1), bf(size, n_slab, 2), bf(size, n_slab, 3)


def cpu_baseline(size, p, budget_s=12.0):
    threads = os.cpu_count() or 1
    kind, run = _cpu_layer_runner()
    n_slab = max(128, min(size, 512))
    x, w, dy = cpu_sample_inputs(size, n_slab)
    times = []
    t_start = time.perf_counter()
    while len(times) < 3 or (time.perf_counter() - t_start < budget_s and len(times) < 20):
        t0 = time.perf_counter()
        run(x, w, dy, p, threads)
        times.append(time.perf_counter() - t0)
        if time.perf_counter() - t_start > 4 * budget_s:
            break
    t = sorted(times)[len(times) // 2]
    flops = 3 * 2 * size * n_slab * size
    return {
        "value": flops / t / 1e12, "unit": UNIT, "cores": threads, "kind": kind,
        "sample": f"layer fwd+bwd (sample_mask+dsd fwd+sdd dX+dsd dW, float) at M=K={size}, N-column slab "
                  f"{n_slab} of {size} (work linear in N), p={p}, median of {len(times)} runs, "
                  f"{threads} threads; dense-equivalent FLOP/s",
        "seconds_per_sample": t,
    }


def run_reference_arm(args, rank, world):
    """The reference's own CPU layer fwd+bwd (oracle/_ref, else the oracle port)
    on the box's host cores, on the GPU arm's config/metric: a bounded slab of
    the same problem per step (work is linear in the slab), rank 0 only."""
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    kind, run = _cpu_layer_runner()
    if args.config == "cfg5":
        # a 2048-row slab of M (16 tile rows: the reference parallelises over them)
        from oracle.oracle import Oracle

        o = Oracle()
        bf = lambda r, c, sd_: o.bf16_bits_to_f64(o.to_bf16_bits(o.random_matrix(r, c, sd_))).astype("float32")  # noqa: E731
        rows = min(2048, args.m_global)
        x, w, dy = bf(rows, args.kn, 1), bf(args.kn, args.kn, 2), bf(rows, args.kn, 3)
        flops = 3 * 2 * rows * args.kn * args.kn
        config = cfg5_config(args.m_global, args.kn, args.p, world, max(1, args.dw_parts), args.dist_backend)
        scaling = "strong"
        sample = (f"per step: the reference layer fwd+bwd on a {rows}-row slab of M (K=N={args.kn}; every GEMM of "
                  f"the layer is linear in M), {threads} host threads; value = slab FLOPs / slab time")
    else:
        n_slab = max(128, min(args.size, 512))
        x, w, dy = cpu_sample_inputs(args.size, n_slab)
        flops = 3 * 2 * args.size * n_slab * args.size
        config = workload_config(args.size, args.p, world, args.dw_parts)
        scaling = "weak"
        sample = (f"per step: the reference layer fwd+bwd at M=K={args.size}, N-column slab {n_slab} (work linear "
                  f"in N), {threads} host threads")
    for _ in range(args.warmup):
        run(x, w, dy, args.p, threads)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        run(x, w, dy, args.p, threads)
    dt = (time.perf_counter() - t0) / args.steps
    value = flops / dt / 1e12
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True,
        "scaling": scaling, "vs_baseline": None, "dtype": "f32", "data": "synthetic (reference random_matrix)",
        "config": config,
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": kind, "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ clocks

class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"error": "no nvidia-smi samples parsed", "raw": self.lines[:3]}
        s = sorted(sm)
        return {"sm_mhz": s[len(s) // 2], "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------------ GPU arm

def small_config_point(S, p, dev, flush_buf):
    """configs[0]: an S^3 layer step (mask + forward + backward, SD_PLAN_DY_READY),
    our dense step and cuBLAS, each spin-gated so the numbers are device time:
    the median of 20 isolated steps (L2 flushed before each) and the mean of 50
    back-to-back steps."""
    import torch

    import paper_2411_01238_b200 as sd

    g = torch.Generator(device=dev)
    g.manual_seed(4321)

    def synth(r, c):
        u = torch.rand(r, c, generator=g, device=dev)
        return ((0.25 + u) * torch.where(torch.rand(r, c, generator=g, device=dev) < 0.5, -1.0, 1.0)).to(torch.bfloat16)

    sets = [(synth(S, S), synth(S, S), synth(S, S)) for _ in range(3)]
    plans = [sd.LayerPlan(x, w, dy, p, dy_ready=True) for x, w, dy in sets]

    def sparse(i):
        plans[i % 3].forward(i)
        plans[i % 3].backward()

    def dense(i):
        plans[i % 3].dense_forward()
        plans[i % 3].dense_backward()

    def cublas(i):
        x, w, dy = sets[i % 3]
        return x @ w, x.t() @ dy, dy @ w.t()

    out = {"shape": [S, S, S], "p": p}
    for name, fn in (("sparse", sparse), ("dense", dense), ("cublas", cublas)):
        for i in range(300):
            fn(i)
        torch.cuda.synchronize()
        iso = []
        for i in range(20):
            flush_buf.fill_(1.0)
            torch.cuda._sleep(200000)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn(1000 + i)
            b.record()
            b.synchronize()
            iso.append(a.elapsed_time(b))
        torch.cuda._sleep(2000000)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for i in range(50):
            fn(2000 + i)
        b.record()
        torch.cuda.synchronize()
        out[f"{name}_isolated_ms"] = sorted(iso)[len(iso) // 2]
        out[f"{name}_back_to_back_ms"] = a.elapsed_time(b) / 50
    out["speedup_vs_dense_isolated"] = out["dense_isolated_ms"] / out["sparse_isolated_ms"]
    out["speedup_vs_dense_back_to_back"] = out["dense_back_to_back_ms"] / out["sparse_back_to_back_ms"]
    out["speedup_vs_cublas_back_to_back"] = out["cublas_back_to_back_ms"] / out["sparse_back_to_back_ms"]
    out["timing"] = ("spin-gated (every launch queued before the first runs): device time; isolated = median of 20 "
                     "single steps after a 512 MiB L2 flush; back to back = 50 steps over 3 L2-resident input sets")
    return out


def main():
    args = parse_args()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.config is None:
        args.config = "cfg2" if world == 1 else "cfg5"
    if args.dw_parts is None:
        args.dw_parts = 1 if args.config == "cfg5" else 2

    if args.impl == "reference":
        run_reference_arm(args, rank, world)
        return
    if world > 1:
        # NCCL communicator lines (rank count, transport) on stderr, for the record
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")

    import torch
    import torch.distributed as dist

    import paper_2411_01238_b200 as sd

    ndev = max(torch.cuda.device_count(), 1)
    dev_index = local_rank % ndev
    torch.cuda.set_device(dev_index)
    dev = torch.device("cuda", dev_index)
    if world > 1:
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group("gloo")
    if args.config == "cfg5":
        run_cfg5(args, rank, world, dev_index, dev)
        if world > 1:
            dist.destroy_process_group()
        return

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(v):
        if world == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    S = args.size
    M, N, K = S, S, S
    gen = torch.Generator(device=dev)
    gen.manual_seed(1234 + rank)

    def synth(r, c):
        # random_matrix's distribution (oracles.hpp:31-41): |v| in [0.25, 1.25), random sign
        u = torch.rand(r, c, generator=gen, device=dev)
        sign = torch.where(torch.rand(r, c, generator=gen, device=dev) < 0.5, -1.0, 1.0)
        return ((0.25 + u) * sign).to(torch.bfloat16)

    gen_w = torch.Generator(device=dev)
    gen_w.manual_seed(99)  # W replicated: same on every rank
    n_sets = max(1, args.rotate)
    sets = []
    for _ in range(n_sets):
        w_ = ((0.25 + torch.rand(K, N, generator=gen_w, device=dev)) *
              torch.where(torch.rand(K, N, generator=gen_w, device=dev) < 0.5, -1.0, 1.0)).to(torch.bfloat16)
        sets.append((synth(M, K), w_, synth(M, N)))
    x, w, dy = sets[0]
    set_bytes = (M * K + K * N + M * N) * 2
    flush_buf = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    comm = torch.cuda.Stream(device=dev) if world > 1 else None
    row_off = rank * (M // 128)

    def flush():
        flush_buf.fill_(float(len(str(flush_buf.numel()))))

    def time_steps(step, steps, warmup, preroll_s=None, rotate=None, windows=1):
        preroll_s = args.preroll if preroll_s is None else preroll_s
        rotate = (n_sets > 1) if rotate is None else rotate
        """Device time per step (CUDA events on the launching stream, max over
        ranks). rotate: steps run back-to-back, each on the next of `n_sets`
        input sets whose combined footprint exceeds L2; else: L2 flushed before
        every step outside the per-step events. A short sustained pre-roll of
        the same step first, so every configuration is timed in the same
        (power-capped) steady state rather than a cold burst. windows > 1
        (legs other than the headline): that many consecutive windows of
        `steps` steps, the median window is returned (one host hiccup while
        enqueueing once doubled a sweep point)."""
        if preroll_s > 0:
            # estimate the step time, then run the same number of pre-roll steps
            # on every rank (each step may contain a collective)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for j in range(3):
                step(j)
            torch.cuda.synchronize()
            est = max((time.perf_counter() - t0) / 3, 1e-5)
            n_pre = int(max_over_ranks(float(min(max(preroll_s / est, 1), 20000))))
            for j in range(n_pre):
                step(j)
                if j % 64 == 63:
                    torch.cuda.synchronize()
        for i in range(warmup):
            if not rotate:
                flush()
            step(i)
        torch.cuda.synchronize()
        barrier()
        torch.cuda.synchronize()
        l0 = sd.launch_count()
        if rotate:
            # back-to-back steps over rotating input sets (combined > L2): one
            # event pair around exactly `steps` steps. One untimed step is
            # enqueued first, so the GPU is busy (and the host ahead of it) when
            # the start event is reached: no launch-latency gap inside the window
            step(warmup + steps)
            l0 = sd.launch_count()
            evs = []
            for wi in range(windows):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                for i in range(steps):
                    step(warmup + i)
                b.record()
                evs.append((a, b))
            torch.cuda.synchronize()
            win = sorted(a_.elapsed_time(b_) for a_, b_ in evs)
            total_ms = win[len(win) // 2]
            launches = (sd.launch_count() - l0) // windows
        else:
            evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                   for _ in range(steps)]
            for i in range(steps):
                flush()
                evs[i][0].record()
                step(warmup + i)
                evs[i][1].record()
            torch.cuda.synchronize()
            total_ms = sum(a_.elapsed_time(b_) for a_, b_ in evs)
            launches = sd.launch_count() - l0
        barrier()
        torch.cuda.synchronize()
        launch_box[0] = launches
        return max_over_ranks(total_ms) / steps

    plans = {}
    launch_box = [0]

    def plan_for(p, j=0):
        if (p, j) not in plans:
            xs, ws, dys = sets[j]
            plans[(p, j)] = sd.LayerPlan(xs, ws, dys, p, row_block_offset=row_off, dy_ready=True)
        return plans[(p, j)]

    def drop_plans(p):
        for j in range(n_sets):
            plans.pop((p, j), None)

    def sparse_step_fn(p):
        pls = [plan_for(p, j) for j in range(n_sets)]

        def step(i):
            plan = pls[i % n_sets]
            plan.forward(seed=sd.effective_seed(0, i, 0))
            if world > 1:
                # dW slab by slab: each slab's all-reduce (comm stream) overlaps
                # the next slab and dX on the compute stream
                nparts = max(1, args.dw_parts)
                for part in range(nparts):
                    slab = plan.backward_dw_part(part, nparts) if nparts > 1 else plan.backward_dw()
                    comm.wait_stream(torch.cuda.current_stream())
                    with torch.cuda.stream(comm):
                        dist.all_reduce(slab)
                plan.backward_dx()
                torch.cuda.current_stream().wait_stream(comm)
            else:
                plan.backward()

        return step

    def dense_step_fn():
        pls = [plan_for(args.p, j) for j in range(n_sets)]

        def step(i):
            plan = pls[i % n_sets]
            plan.dense_forward()
            if world > 1:
                plan.dense_backward()  # dw then dx on the compute stream
                comm.wait_stream(torch.cuda.current_stream())
                with torch.cuda.stream(comm):
                    dist.all_reduce(plan.dw)
                torch.cuda.current_stream().wait_stream(comm)
            else:
                plan.dense_backward()

        return step

    def torch_step(i):
        xs, ws, dys = sets[i % n_sets]
        y = xs @ ws
        dw = xs.t() @ dys
        dx = dys @ ws.t()
        return y, dw, dx

    flops_dense_step = 3 * 2 * M * N * K  # per GPU

    # ---- headline: sparse fwd+bwd at args.p
    head_step = sparse_step_fn(args.p)
    with ClockSampler(dev_index) as clk:
        # sustained load first (~1.5 s of the same step) so the 100 ms nvidia-smi
        # samples see the clocks the timed steps run at
        ms = time_steps(head_step, args.steps, args.warmup,
                        preroll_s=0.2 if args.profile else max(args.preroll, 1.5 if args.preroll > 0 else 0.0))
    gpu_launches = launch_box[0]  # our kernels enqueued inside the timed region (3 per step)
    ms_isolated = time_steps(head_step, args.steps, args.warmup, rotate=False) if not args.profile else None
    plan = plan_for(args.p)
    keep = plan.mask.keep_count() / plan.mask.total_blocks()
    value = world * flops_dense_step / (ms * 1e-3) / 1e12

    if args.profile:
        if rank == 0:
            print(json.dumps({"metric": METRIC, "value": value, "unit": UNIT, "ms_per_step": ms, "profile": True}),
                  flush=True)
        return

    # ---- dense baseline (same kernel, no mask) and cuBLAS for context. Each
    # configuration is timed in its own steady state: under the power cap the
    # SM clock settles over ~1 s and differs by workload (a 0.3 s pre-roll left
    # the denominator and the sweep points up to ~10% apart in clock state)
    settle = max(args.preroll, 1.5 if args.preroll > 0 else 0.0)
    _lib_t = sd.load_library()

    def dense_1cta_step():
        # the same dense step on the 1-CTA tile machinery the masked GEMMs use
        # (tuning 16: no 2-CTA kernel) — the like-for-like (1-p) reference
        _lib_t.sd_set_tuning(16)
        try:
            return time_steps(dense_step_fn(), args.steps, args.warmup, preroll_s=settle, windows=3)
        finally:
            _lib_t.sd_set_tuning(0)

    # our dense step and cuBLAS alternate over three rounds, each leg after its
    # own settle; the median round of each is reported. Under the power cap a
    # cuBLAS leg is bimodal (0.276 or 0.323 ms at 4096^3 in consecutive rounds of
    # one run; ours 0.313-0.320): profiles/r02_dense_vs_cublas_ab.txt
    rounds = {"dense": [], "torch": []}
    for _ in range(3):
        rounds["dense"].append(time_steps(dense_step_fn(), args.steps, args.warmup, preroll_s=settle, windows=3))
        rounds["torch"].append(time_steps(torch_step, args.steps, args.warmup, preroll_s=settle, windows=3))
    ms_dense, ms_torch = sorted(rounds["dense"])[1], sorted(rounds["torch"])[1]
    ms_dense_1cta = dense_1cta_step()

    # ---- per-kernel durations at the headline p (roofline): each kernel run
    # back-to-back over the rotating input sets, one event pair around them
    lib = sd.load_library()
    import ctypes as _ct

    def rot_ms(fns, steps, settle_s=1.0):
        # each kernel in its own settled power-capped state, like every other leg
        # (without it the kernel times depended on which leg ran before: a fused
        # backward read 133 us in one run and 156 us in the next)
        t_end = time.perf_counter() + (settle_s if args.preroll > 0 else 0.0)
        j = 0
        while j < 3 * n_sets or time.perf_counter() < t_end:
            fns[j % n_sets]()
            j += 1
            if j % 64 == 0:
                torch.cuda.synchronize()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for i in range(steps):
            fns[i % n_sets]()
        b.record()
        torch.cuda.synchronize()
        return a.elapsed_time(b) / steps

    pls = [plan_for(args.p, j) for j in range(n_sets)]
    st_ = lambda: _ct.c_void_p(torch.cuda.current_stream().cuda_stream)  # noqa: E731

    def fwd_only(pl):
        return lambda: sd.api.check(lib.sd_linear_forward(pl.x.data_ptr(), pl.mask.cptr(), pl.w.data_ptr(), pl.scale,
                                                          pl.y.data_ptr(), 1, M, N, K, st_()))

    for pl in pls:
        pl.forward(seed=7)
    keep_blocks = plan.mask.keep_count()
    exec_flops = 2 * N * 128 * 128 * keep_blocks  # flops_effective (gemm.hpp:222-228), per GEMM
    ksteps = max(args.steps, 10)
    kms = {
        "mask_gen+compact": rot_ms([lambda pl=pl: sd.sample_mask(sd.DropoutSpec(args.p, 128, 128, 7), M, K,
                                                                 row_block_offset=row_off, out=pl.mask)
                                    for pl in pls], ksteps),
        "dsd_fwd": rot_ms([fwd_only(pl) for pl in pls], ksteps),
        "bwd_fused(dsd_dw+sdd_dx)": rot_ms([pl.backward for pl in pls], ksteps),
        "dsd_dw(standalone)": rot_ms([pl.backward_dw for pl in pls], ksteps),
        "sdd_dx(standalone)": rot_ms([pl.backward_dx for pl in pls], ksteps),
    }
    kflops = {"dsd_fwd": exec_flops, "bwd_fused(dsd_dw+sdd_dx)": 2 * exec_flops, "dsd_dw(standalone)": exec_flops,
              "sdd_dx(standalone)": exec_flops}
    # the dominant kernel of the step as it runs: the longest of forward / fused backward
    dom = max(("dsd_fwd", "bwd_fused(dsd_dw+sdd_dx)"), key=kms.get)
    achieved = kflops[dom] / (kms[dom] * 1e-3) / 1e12
    exec_flops_dom = kflops[dom]
    peaks = {}
    try:
        peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
    except Exception:
        pass
    # the kernels are timed after 1 s of their own sustained load (rot_ms): the
    # denominator is the sustained cuBLAS figure (B200_PROFILING.md: "the
    # sustained one for a kernel timed inside a long step"); the burst fraction
    # is reported beside it
    peak_burst = float(peaks.get("bf16_tflops", 1590.0))
    peak = float(peaks.get("bf16_tflops_sustained", 1400.0))
    traffic = None
    tfile = ROOT / "profiles" / "ncu_traffic.json"
    if tfile.exists():
        try:
            traffic = json.loads(tfile.read_text()).get(dom)
        except Exception:
            traffic = None
    roofline = {
        "bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
        "traffic": traffic, "kernel": dom,
        "algorithmic_per_launch": {"flops": exec_flops_dom,
                                   "note": "keep_count*2*N*128*128 per GEMM (flops_effective, gemm.hpp:222-228); "
                                           "the fused backward launch carries dW + dX"},
        "per_kernel_tflops": {k: kflops[k] / (kms[k] * 1e-3) / 1e12 for k in kflops},
        "peak_source": ("MEASURED_PEAKS.json bf16_tflops_sustained (the kernel is timed after 1 s of its own "
                        "sustained load)") if peaks else "fallback 1400 sustained (B200_PROFILING.md)",
        "peak_burst": peak_burst,
        "frac_of_burst": achieved / peak_burst,
        "kernel_ms": kms,
        "kernel_timing": "each kernel back-to-back over the rotating input sets after 1 s of its own sustained "
                         "load (mask_gen is host-launch-bound here; ncu: ~5-7 us)",
    }

    # ---- sweep
    sweep = []
    if not args.no_sweep:
        for p in SWEEP_P:
            msp = time_steps(sparse_step_fn(p), max(5, args.steps // 2), 3, preroll_s=settle, windows=3)
            pl = plan_for(p)
            kp = pl.mask.keep_count() / pl.mask.total_blocks()
            sweep.append({
                "p": p, "keep": kp, "ms_per_step": msp,
                "dense_equiv_tflops": world * flops_dense_step / (msp * 1e-3) / 1e12,
                "executed_tflops": world * kp * flops_dense_step / (msp * 1e-3) / 1e12,
                "speedup_vs_dense": ms_dense / msp,
                "speedup_vs_dense_1cta": ms_dense_1cta / msp,
                "speedup_vs_cublas": ms_torch / msp,
                "time_vs_dense_over_keep": (msp / ms_dense) / max(kp, 1e-9),
            })
            if p != args.p:
                drop_plans(p)

    # ---- T8: the north-star 8192^3 target (sparse p=0.1/0.5 vs our dense), single GPU only
    t8 = None
    if world == 1 and not args.no_sweep and S != 8192:
        S8 = 8192
        x8, w8, dy8 = synth(S8, S8), synth(S8, S8), synth(S8, S8)
        t8 = {"shape": [S8, S8, S8]}
        for p8 in (0.0, 0.1, 0.5):
            pl8 = sd.LayerPlan(x8, w8, dy8, p8, dy_ready=True)

            def st8(i, pl8=pl8):
                pl8.forward(seed=sd.effective_seed(0, i, 0))
                pl8.backward()

            ms8 = time_steps(st8, max(5, args.steps // 2), 3, preroll_s=settle, windows=3)
            k8 = pl8.mask.keep_count() / pl8.mask.total_blocks()
            ex8 = k8 * 3 * 2 * S8 ** 3 / (ms8 * 1e-3) / 1e12
            t8[f"p{p8}"] = {"ms_per_step": ms8, "keep": k8,
                            "dense_equiv_tflops": 3 * 2 * S8 ** 3 / (ms8 * 1e-3) / 1e12,
                            "executed_tflops": ex8,
                            "executed_frac_of_burst_peak": ex8 / float(peaks.get("bf16_tflops", 1590.0)),
                            "executed_frac_of_sustained_peak": ex8 / float(peaks.get("bf16_tflops_sustained", 1400.0))}
            if p8 == 0.5:
                def dn8(i, pl8=pl8):
                    pl8.dense_forward()
                    pl8.dense_backward()

                msd8 = time_steps(dn8, max(5, args.steps // 2), 3, preroll_s=settle, windows=3)
                t8["dense_ms_per_step"] = msd8
                t8["dense_tflops"] = 3 * 2 * S8 ** 3 / (msd8 * 1e-3) / 1e12
                t8["speedup_vs_dense_p0.5"] = msd8 / ms8
            del pl8
        mst = time_steps(lambda i: (x8 @ w8, x8.t() @ dy8, dy8 @ w8.t()), max(5, args.steps // 2), 3,
                         preroll_s=settle, windows=3)
        t8["torch_cublas_dense_tflops"] = 3 * 2 * S8 ** 3 / (mst * 1e-3) / 1e12
        del x8, w8, dy8
        torch.cuda.empty_cache()

    # ---- e2e through the public API with pinned host buffers: every step copies
    # its inputs host->device and its outputs device->host; steps are double-
    # buffered so H2D(i+1), compute(i) and D2H(i-1) overlap (HostLayerPipeline)
    e2e = None
    if not args.no_e2e:
        from paper_2411_01238_b200.pipeline import HostLayerPipeline

        xh = x.cpu().pin_memory(); wh = w.cpu().pin_memory(); dyh = dy.cpu().pin_memory()
        pipe = HostLayerPipeline(xh, wh, dyh, args.p, row_block_offset=row_off, device=dev)
        ar = (lambda t: dist.all_reduce(t)) if world > 1 else None
        n_e2e = max(40, args.steps)  # steady state: the fill and drain amortised (10 steps: +4%)
        for i in range(3):
            pipe.step(i, ar)
        pipe.synchronize()
        barrier()
        torch.cuda.synchronize()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record(pipe.s_h2d)
        pipe.s_cmp.wait_stream(pipe.s_h2d)
        for i in range(n_e2e):
            pipe.step(3 + i, ar)
        pipe.s_d2h.wait_stream(pipe.s_cmp)
        pipe.s_d2h.wait_stream(pipe.s_h2d)
        ev1.record(pipe.s_d2h)
        pipe.synchronize()
        ms_e2e = max_over_ranks(ev0.elapsed_time(ev1)) / n_e2e
        e2e = {"value": world * flops_dense_step / (ms_e2e * 1e-3) / 1e12, "unit": UNIT, "ms_per_step": ms_e2e,
               "h2d_bytes_per_step": pipe.h2d_bytes, "d2h_bytes_per_step": pipe.d2h_bytes,
               "path": "HostLayerPipeline -> LayerPlan (C-ABI sd_layer_plan_*): pinned host X/W/dY in, "
                       "Y/dX/dW out every step; H2D(i+1) | compute(i) | D2H(i-1) double-buffered, 40 steps; "
                       "per-step footprint 224 MiB > L2",
               "pcie_gbps": (pipe.h2d_bytes + pipe.d2h_bytes) / (ms_e2e * 1e-3) / 1e9}
        del pipe

    # configs[4] on this one GPU (the G = 1 point of its strong-scaling curve: the
    # N > 1 runs of this script measure configs[4] by default)
    cfg5_g1 = None
    if world == 1 and not args.no_sweep:
        import copy

        a5 = copy.copy(args)
        a5.steps, a5.warmup, a5.no_e2e, a5.config = max(5, args.steps // 2), 3, True, "cfg5"
        l5 = run_cfg5(a5, rank, world, dev_index, dev, emit=False)
        cfg5_g1 = {k: l5[k] for k in ("value", "unit", "ms_per_step", "executed_tflops", "keep_fraction", "config",
                                      "roofline", "clocks", "gpu_launches")}
        cfg5_g1["note"] = ("configs[4] (M=524288, K=N=8192, p=%g) on one B200: the strong-scaling baseline for the "
                           "N > 1 runs (torchrun ... bench.py --gpus N, default --config cfg5)" % args.p)

    # configs[0] (1024^3) beside the headline: latency-bound, so it is reported
    # spin-gated (device time only): isolated steps after a 512 MiB L2 flush, and
    # back-to-back steps (its 6 MiB operands stay L2-resident there)
    cfg1 = None
    if world == 1 and not args.no_sweep:
        cfg1 = small_config_point(1024, args.p, dev, flush_buf)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        try:
            cpu = cpu_baseline(S, args.p)
        except Exception as exc:  # reported, never fatal for the GPU line
            cpu = {"error": repr(exc)}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "bf16", "data": "synthetic (random_matrix distribution, on device)",
            "config": workload_config(S, args.p, world, args.dw_parts),
            "keep_fraction": keep, "executed_tflops": value * keep,
            "dense_ms_per_step": ms_dense, "speedup_vs_dense": ms_dense / ms,
            "dense_1cta_ms_per_step": ms_dense_1cta, "speedup_vs_dense_1cta": ms_dense_1cta / ms,
            "speedup_vs_cublas": ms_torch / ms,
            "dense_note": ("dense_ms_per_step: our 2-CTA (cta_group::2) dense kernel, the speed-up denominator; "
                           "dense_1cta_ms_per_step: the same dense step on the 1-CTA tiles the masked GEMMs use"),
            "isolated_ms_per_step": ms_isolated,
            "timing": (f"{n_sets} rotating input sets ({n_sets * set_bytes / 2**20:.0f} MiB > L2), steps back-to-back, "
                       "one CUDA-event pair around the K timed steps, entered with one untimed step already queued "
                       "(no launch-latency gap in the window); every leg (headline, dense, sweep points, t8) after "
                       "1.5 s of its own sustained load (power-capped steady state); legs other than the headline: "
                       "median of three consecutive K-step windows; isolated_ms_per_step: one step at a time with a "
                       "512 MiB L2 flush before each, per-step events (includes launch latency)"),
            "cfg1": cfg1,
            "torch_cublas_dense_ms_per_step": ms_torch,
            "dense_rounds_ms": rounds["dense"], "torch_cublas_rounds_ms": rounds["torch"],
            "gpu_launches": gpu_launches,
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "clocks": clk.summary(),
            "sweep": sweep,
            "t8": t8,
            "cfg5_g1": cfg5_g1,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


# ------------------------------------------------------------------ configs[4]: row-sharded data parallel

def cfg5_config(m_global, kn, p, world, nparts, backend):
    return {
        "workload": f"configs[4]: row-sharded data-parallel SparseDrop linear fwd+bwd, M={m_global} (global, "
                    f"M/{world} rows per GPU), K=N={kn}, 128x128 blocks, p={p}, one dW all-reduce per step",
        "M_global": m_global, "M_per_gpu": m_global // world, "N": kn, "K": kn, "m_blk": 128, "k_blk": 128,
        "p": p, "seed": 0,
        "dtypes": {"x/w/dy/y/dx": "bf16", "dw": "fp32 (all-reduced)", "accumulate": "fp32"},
        "l2": "inputs larger than L2 (each rank's X and dY exceed the 126 MB L2 at every N <= 8)",
        "parallelism": (f"dp{world}: rank g owns global rows [g*M/{world}, (g+1)*M/{world}), shard-local masks "
                        f"(bit-identical to the global mask rows), W replicated; "
                        + ("dW computed, then ONE sum all-reduce of it on a comm stream while dX computes"
                           if nparts == 1 else f"dW in {nparts} row slabs, each all-reduced while the next slab and "
                                               "dX compute")
                        + (" (the library's NCCL communicator, C-ABI sd_layer_plan_backward_allreduce)"
                           if backend == "nccl" else " (torch.distributed gloo: CI path, several ranks on one GPU)"))
        if world > 1 else "single GPU (the strong-scaling baseline: the whole M on one B200)",
    }


def run_cfg5(args, rank, world, dev_index, dev, emit=True):
    """configs[4]: M=524288, K=N=8192 strong-scaled over the ranks.
    value = 3*2*M*N*K (dense-equivalent, whole job) / max-over-ranks step time.
    Returns the line (rank 0); prints it when `emit`."""
    import torch
    import torch.distributed as dist

    import paper_2411_01238_b200 as sd
    from paper_2411_01238_b200.sharding import shard_rows

    KN, MG, p = args.kn, args.m_global, args.p
    shard = shard_rows(MG, 128, world, rank)
    M = shard.rows
    nparts = max(1, args.dw_parts)
    use_lib_comm = world > 1 and args.dist_backend == "nccl"

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(v):
        if world == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64, device=dev if args.dist_backend == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    gen = torch.Generator(device=dev)
    gen.manual_seed(1234 + rank)

    def synth(r, c, g):
        out = torch.empty(r, c, dtype=torch.bfloat16, device=dev)
        step = max(1, (1 << 28) // c)  # chunks of <= 256 M elements (bounded fp32 temporaries)
        for r0 in range(0, r, step):
            r1 = min(r, r0 + step)
            u = torch.rand(r1 - r0, c, generator=g, device=dev)
            sign = torch.where(torch.rand(r1 - r0, c, generator=g, device=dev) < 0.5, -1.0, 1.0)
            out[r0:r1] = ((0.25 + u) * sign).to(torch.bfloat16)
            del u, sign
        return out

    gen_w = torch.Generator(device=dev)
    gen_w.manual_seed(99)  # W replicated: the same on every rank
    x, w, dy = synth(M, KN, gen), synth(KN, KN, gen_w), synth(M, KN, gen)
    plan = sd.LayerPlan(x, w, dy, p, row_block_offset=shard.row_block_offset, dy_ready=True)
    comm = None
    if use_lib_comm:
        obj = [sd.Communicator.new_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        comm = sd.Communicator(world, rank, obj[0])
    comm_stream = torch.cuda.Stream(device=dev)
    cur = torch.cuda.current_stream()

    def step(i):
        plan.forward(seed=sd.effective_seed(0, i, 0))
        if world == 1:
            plan.backward()
        elif comm is not None:
            plan.backward_allreduce(comm, nparts, stream=cur, comm_stream=comm_stream)
        else:
            for part in range(nparts):
                slab = plan.backward_dw_part(part, nparts)
                comm_stream.wait_stream(cur)
                with torch.cuda.stream(comm_stream):
                    dist.all_reduce(slab)
            plan.backward_dx()
            cur.wait_stream(comm_stream)

    def compute_only(i):
        plan.forward(seed=sd.effective_seed(0, i, 0))
        if world == 1:
            plan.backward()
        else:
            for part in range(nparts):
                plan.backward_dw_part(part, nparts)
            plan.backward_dx()

    def allreduce_only(i):
        if comm is not None:
            comm.allreduce_sum(plan.dw, stream=cur)
        elif world > 1:
            dist.all_reduce(plan.dw)

    def timed(fn, steps, warmup, preroll_s):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn(0)
        torch.cuda.synchronize()
        est = max(time.perf_counter() - t0, 1e-5)
        n_pre = int(max_over_ranks(float(min(max(preroll_s / est, 0), 200))))
        for j in range(n_pre + warmup):
            fn(j)
        torch.cuda.synchronize()
        barrier()
        torch.cuda.synchronize()
        l0 = sd.launch_count()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for i in range(steps):
            fn(warmup + i)
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / steps
        barrier()
        return max_over_ranks(ms), sd.launch_count() - l0

    with ClockSampler(dev_index) as clk:
        ms, launches = timed(step, args.steps, args.warmup, args.preroll if args.preroll > 0 else 0.0)
    ms_compute, _ = timed(compute_only, max(3, args.steps // 2), 2, 0.0)
    ms_ar = timed(allreduce_only, max(3, args.steps // 2), 2, 0.0)[0] if world > 1 else 0.0
    keep_local = plan.mask.keep_count()
    keep_t = torch.tensor([float(keep_local)], dtype=torch.float64,
                          device=dev if args.dist_backend == "nccl" else "cpu")
    if world > 1:
        dist.all_reduce(keep_t)
    keep = float(keep_t.item()) / ((MG // 128) * (KN // 128))
    flops = 3 * 2 * MG * KN * KN
    value = flops / (ms * 1e-3) / 1e12
    exposed = max(0.0, ms - ms_compute)
    comm_info = {
        "allreduce_ms": ms_ar, "allreduce_bytes": KN * KN * 4, "compute_only_ms_per_step": ms_compute,
        "exposed_comm_ms": exposed,
        "overlap_fraction": (min(1.0, max(0.0, 1.0 - exposed / ms_ar)) if ms_ar > 0 else None),
        "busbw_gbps": (KN * KN * 4 * 2 * (world - 1) / world / (ms_ar * 1e-3) / 1e9) if ms_ar > 0 else None,
        "path": ("C-ABI sd_layer_plan_backward_allreduce (library-owned NCCL communicator, NCCL "
                 f"{sd.Communicator.nccl_version()})" if comm is not None else
                 ("torch.distributed gloo (CI)" if world > 1 else "none (single GPU)")),
        "note": "device-timed, max over ranks: allreduce_ms = the dW all-reduce alone; compute_only = the "
                "same step without it; overlap_fraction = 1 - (step - compute_only) / allreduce",
    }
    # roofline of the per-GPU step's GEMM work (the step's kernels overlap under
    # PDL, so the whole compute-only step is the timed unit here)
    peaks = {}
    try:
        peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
    except Exception:
        pass
    peak = float(peaks.get("bf16_tflops_sustained", 1400.0))
    achieved = keep * 3 * 2 * M * KN * KN / (ms_compute * 1e-3) / 1e12
    roof = {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
            "traffic": None, "kernel": "the per-GPU step without the all-reduce (mask + forward + backward GEMMs)",
            "peak_source": "MEASURED_PEAKS.json bf16_tflops_sustained (steps timed after a sustained pre-roll)",
            "algorithmic_per_launch": {"flops": keep * 3 * 2 * M * KN * KN,
                                       "note": "executed: keep x 3 GEMMs x 2 M_local N K per step"}}
    # e2e through the public API with host buffers (pinned), every step
    e2e = None
    if not args.no_e2e:
        from paper_2411_01238_b200.pipeline import HostLayerPipeline

        xh, wh, dyh = x.cpu().pin_memory(), w.cpu().pin_memory(), dy.cpu().pin_memory()
        del plan
        torch.cuda.empty_cache()
        pipe = HostLayerPipeline(xh, wh, dyh, p, row_block_offset=shard.row_block_offset, device=dev,
                                 nslots=2)  # configs[4] shards: GBs per buffer set
        ar = None
        if world > 1:
            ar = ((lambda t: comm.allreduce_sum(t)) if comm is not None else (lambda t: dist.all_reduce(t)))
        n_e2e = 3
        for i in range(2):
            pipe.step(i, ar)
        pipe.synchronize()
        barrier()
        torch.cuda.synchronize()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record(pipe.s_h2d)
        pipe.s_cmp.wait_stream(pipe.s_h2d)
        for i in range(n_e2e):
            pipe.step(2 + i, ar)
        pipe.s_d2h.wait_stream(pipe.s_cmp)
        pipe.s_d2h.wait_stream(pipe.s_h2d)
        ev1.record(pipe.s_d2h)
        pipe.synchronize()
        ms_e2e = max_over_ranks(ev0.elapsed_time(ev1)) / n_e2e
        e2e = {"value": flops / (ms_e2e * 1e-3) / 1e12, "unit": UNIT, "ms_per_step": ms_e2e,
               "h2d_bytes_per_step": pipe.h2d_bytes, "d2h_bytes_per_step": pipe.d2h_bytes,
               "path": "HostLayerPipeline -> LayerPlan (C-ABI), pinned host X/W/dY in and Y/dX/dW out every "
                       "step on every rank (per-rank bytes above)" + (", dW all-reduced" if world > 1 else "")}
        del pipe
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "bf16", "data": "synthetic (random_matrix distribution, on device)",
            "config": cfg5_config(MG, KN, p, world, nparts, args.dist_backend),
            "keep_fraction": keep, "executed_tflops": value * keep,
            "comm": comm_info, "gpu_launches": launches,
            "roofline": roof,
            "gpu_launches_note": "per step: mask, forward, " + (f"{nparts} dW slabs, dX" if world > 1 else
                                                               "fused dW+dX (or dW + masked dX at low p)"),
            "cpu_baseline": None,
            "cpu_baseline_note": "the reference CPU path is timed in the configs[1] line (N=1 default run)",
            "e2e": e2e, "clocks": clk.summary(),
        }
        if emit:
            print(json.dumps(line), flush=True)
    if comm is not None:
        torch.cuda.synchronize()
        comm.close()
    del x, w, dy
    torch.cuda.empty_cache()
    return line if rank == 0 else None


if __name__ == "__main__":
    main()
