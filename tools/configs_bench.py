"""Every BASELINE.json configuration on one B200 (bench.py measures configs[1]).

  python tools/configs_bench.py [--out gpurun_out/configs.json] [--quick]

cfg1  SparseDrop layer fwd+bwd 1024^3, p=0.5
cfg3  ViT-B MLP training step, 65536 tokens, 768 -> 3072 -> 768, SparseDrop
      before each Linear (GELU between), p=0.1/0.5, vs the same step dense
cfg4  LLM projection M=65536, K=N=8192, p=0.1/0.3/0.5, vs dense
cfg5  one GPU's row shard of M=524288, K=N=8192 (the G=1 point), p=0.1/0.5
Timing: CUDA events per step, L2 flushed between steps, each step queued behind
a short spin kernel (torch.cuda._sleep) so its launches are all enqueued before
the GPU reaches the first event (device time, not host launch latency), 0.3 s sustained
pre-roll per configuration (steady power-capped state); dense-equivalent and
executed TFLOP/s, speed-up vs our dense tcgen05 path on the same buffers.
Beside each: the reference CPU layer fwd+bwd (oracle/_ref, all host threads,
float) on a row slab of the same problem, extrapolated linearly in M (every
GEMM of the layer, dW included, is linear in M) — SURVEY §8(d).
"""
import argparse
import json
import sys
import time
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_2411_01238_b200 as sd  # noqa: E402
from paper_2411_01238_b200.mlp import SparseDropMLP  # noqa: E402

dev = torch.device("cuda", 0)
gen = torch.Generator(device=dev)
gen.manual_seed(7)
flush_buf = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)


def synth(r, c):
    u = torch.rand(r, c, generator=gen, device=dev)
    sign = torch.where(torch.rand(r, c, generator=gen, device=dev) < 0.5, -1.0, 1.0)
    return ((0.25 + u) * sign).to(torch.bfloat16)


def timed(step, steps, preroll_s=0.3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for j in range(2):
        step(j)
    torch.cuda.synchronize()
    est = max((time.perf_counter() - t0) / 2, 1e-5)
    for j in range(int(min(max(preroll_s / est, 1), 5000))):
        step(j)
    torch.cuda.synchronize()
    tot = 0.0
    for i in range(steps):
        flush_buf.fill_(1.0)
        torch.cuda._sleep(200000)  # ~100 us: the step's launches are queued before it starts
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        step(100 + i)
        b.record()
        b.synchronize()
        tot += a.elapsed_time(b)
    return tot / steps


def back_to_back(step, steps=20):
    """Steps enqueued back to back behind a spin kernel (device time, the
    regime bench.py measures): ms per step."""
    for j in range(3):
        step(j)
    torch.cuda.synchronize()
    torch.cuda._sleep(400000)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for i in range(steps):
        step(200 + i)
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / steps


def cpu_reference(M, N, K, p, slab_rows):
    """The reference's layer fwd+bwd (mask generation included) on the first
    `slab_rows` rows, timed with all host threads; ms extrapolated to M rows."""
    import os

    import numpy as np

    from oracle.oracle import REF_LIB, Oracle, Reference

    if not REF_LIB.exists():
        return None
    o, ref = Oracle(), Reference()
    # the reference parallelises the forward and dX over 128-row tile rows:
    # give every host thread one (16 M-blocks on a 16-core host)
    threads = os.cpu_count() or 1
    rows = min(M, max(slab_rows, 128 * threads))
    x = o.random_matrix(rows, K, 1).astype(np.float32)
    w = o.random_matrix(K, N, 2).astype(np.float32)
    dy = o.random_matrix(rows, N, 3).astype(np.float32)
    t0 = time.perf_counter()
    ref.layer_fwd_bwd(x, w, dy, p, 128, 128, 128, seed=0, step_seed=0, layer_index=0, threads=threads,
                      dtype=np.float32)
    t = time.perf_counter() - t0
    return {"slab_rows": rows, "slab_seconds": t, "threads": threads, "kind": "reference",
            "ms_per_step_extrapolated": t * 1e3 * M / rows}


def layer_cfg(name, M, N, K, ps, steps, slab_rows=512):
    x, w, dy = synth(M, K), synth(K, N), synth(M, N)
    out = []
    dense_ms = None
    flops = 3 * 2 * M * N * K
    for p in ps:
        plan = sd.LayerPlan(x, w, dy, p, dy_ready=True)
        ms = timed(lambda i: (plan.forward(sd.effective_seed(0, i, 0)), plan.backward()), steps)
        keep = plan.mask.keep_count() / plan.mask.total_blocks()
        if dense_ms is None:
            dense_ms = timed(lambda i: (plan.dense_forward(), plan.dense_backward()), steps)
        small = M * N * K <= (1 << 33)
        b2b = back_to_back(lambda i: (plan.forward(sd.effective_seed(0, i, 0)), plan.backward())) if small else None
        b2b_dense = back_to_back(lambda i: (plan.dense_forward(), plan.dense_backward())) if small else None
        cpu = cpu_reference(M, N, K, p, slab_rows)
        if cpu:
            cpu["dense_equiv_tflops"] = flops / (cpu["ms_per_step_extrapolated"] * 1e-3) / 1e12
            cpu["gpu_speedup"] = cpu["ms_per_step_extrapolated"] / ms
        out.append({"config": name, "M": M, "N": N, "K": K, "p": p, "keep": keep, "ms_per_step": ms,
                    "dense_ms_per_step": dense_ms, "speedup_vs_dense": dense_ms / ms,
                    "dense_equiv_tflops": flops / (ms * 1e-3) / 1e12,
                    "executed_tflops": keep * flops / (ms * 1e-3) / 1e12,
                    "dense_tflops": flops / (dense_ms * 1e-3) / 1e12, "cpu_reference": cpu})
        if b2b is not None:
            out[-1].update({"back_to_back_ms_per_step": b2b, "dense_back_to_back_ms_per_step": b2b_dense,
                            "speedup_vs_dense_back_to_back": b2b_dense / b2b})
        print(json.dumps(out[-1]), flush=True)
        del plan
    del x, w, dy
    torch.cuda.empty_cache()
    return out


def mlp_cfg(ps, steps):
    M, D, H = 65536, 768, 3072
    x, w1, w2, dy = synth(M, D), synth(D, H), synth(H, D), synth(M, D)
    flops = 2 * (3 * 2 * M * D * H)  # two Linears, fwd + bwd (GELU not counted)
    dense = SparseDropMLP(x, w1, w2, dy, 0.0, dense=True)
    dense_ms = timed(lambda i: dense.step(i), steps)
    del dense
    out = []
    for p in ps:
        mlp = SparseDropMLP(x, w1, w2, dy, p)
        ms = timed(lambda i: mlp.step(i), steps)
        k1 = mlp.fc1.mask.keep_count() / mlp.fc1.mask.total_blocks()
        k2 = mlp.fc2.mask.keep_count() / mlp.fc2.mask.total_blocks()
        keep = (k1 + k2) / 2
        c1, c2 = cpu_reference(M, H, D, p, 1024), cpu_reference(M, D, H, p, 1024)
        cpu = None
        if c1 and c2:
            cms = c1["ms_per_step_extrapolated"] + c2["ms_per_step_extrapolated"]
            cpu = {"kind": "reference", "threads": c1["threads"], "slab_rows": c1["slab_rows"],
                   "ms_per_step_extrapolated": cms, "dense_equiv_tflops": flops / (cms * 1e-3) / 1e12,
                   "gpu_speedup": cms / ms, "note": "fc1 + fc2 layer fwd+bwd (the reference has no GELU)"}
        out.append({"config": "cfg3_vit_b_mlp", "tokens": M, "dims": [D, H, D], "p": p, "keep_fc1": k1,
                    "keep_fc2": k2, "ms_per_step": ms, "dense_ms_per_step": dense_ms,
                    "speedup_vs_dense": dense_ms / ms, "dense_equiv_tflops": flops / (ms * 1e-3) / 1e12,
                    "executed_tflops": keep * flops / (ms * 1e-3) / 1e12,
                    "note": "GELU / GELU' are this library's single-pass bf16 kernels inside the timed step",
                    "cpu_reference": cpu})
        print(json.dumps(out[-1]), flush=True)
        del mlp
    del x, w1, w2, dy
    torch.cuda.empty_cache()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=str(ROOT / "gpurun_out" / "configs.json"))
    ap.add_argument("--quick", action="store_true")
    args = ap.parse_args()
    res = []
    res += layer_cfg("cfg1", 1024, 1024, 1024, [0.5], 20, slab_rows=1024)
    res += mlp_cfg([0.1, 0.5], 5 if args.quick else 10)
    res += layer_cfg("cfg4", 65536, 8192, 8192, [0.1, 0.3, 0.5], 3 if args.quick else 5)
    if not args.quick:
        res += layer_cfg("cfg5_G1_shard", 524288, 8192, 8192, [0.1, 0.5], 3)
    Path(args.out).parent.mkdir(parents=True, exist_ok=True)
    Path(args.out).write_text(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
