"""Fig. 4a-style sweep on B200 (SPEC.md:444-451 bench_sweep, CSV per :453-459).

  python tools/fig4_bench.py [--sizes 1024,4096] [--sparsity 0,0.1,...] [--repeats 20] [--out f.csv]

Methods: dense, dropout_dense, block_dropout_dense, sparsedrop — all on the
same tcgen05 kernels. Per (method, size, sparsity): warm-up runs, then timed
repeats of forward, backward and total with FRESH masks (mask generation inside
the timed region), L2 flushed between repeats;
median / p10 / p90 in nanoseconds. effective_gflops = executed FLOPs / median
(sparsedrop: flops_effective on the realised keep; the others: dense FLOPs).
Each timed repeat is queued behind a short spin kernel (torch.cuda._sleep, after
the flush) so the forward and backward launches are all enqueued before the GPU
reaches the first event: the numbers are device time, not Python/driver launch
latency (--no-gate restores host-in-the-loop timing; at 1024^3 that measured
~46 us for every method, i.e. the host).
Honesty check: sparsedrop's device work counter must equal the
keep-count prediction for every configuration.
"""
import argparse
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_2411_01238_b200 as sd  # noqa: E402
from paper_2411_01238_b200.baselines import BaselineLayer  # noqa: E402
from paper_2411_01238_b200.benchrec import emit_csv, percentile_record  # noqa: E402

dev = torch.device("cuda", 0)
flush_buf = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)


def synth(r, c, g):
    u = torch.rand(r, c, generator=g, device=dev)
    s = torch.where(torch.rand(r, c, generator=g, device=dev) < 0.5, -1.0, 1.0)
    return ((0.25 + u) * s).to(torch.bfloat16)


def time_pass(fn, i):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    fn(i)
    b.record()
    return a, b


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", default="1024,4096")
    ap.add_argument("--sparsity", default="0,0.1,0.2,0.3,0.4,0.5,0.6,0.7,0.8,0.9")
    ap.add_argument("--repeats", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--out", default=str(ROOT / "gpurun_out" / "fig4.csv"))
    ap.add_argument("--no-gate", action="store_true", help="time with the host enqueue in the loop")
    args = ap.parse_args()
    if args.repeats < 3:
        raise SystemExit("repeats must be >= 3 (SPEC.md:445)")
    records = []
    g = torch.Generator(device=dev)
    g.manual_seed(3)
    for S in [int(v) for v in args.sizes.split(",")]:
        M = N = K = S
        x, w, dy = synth(M, K, g), synth(K, N, g), synth(M, N, g)
        dense_flops = 2 * M * N * K
        for p in [float(v) for v in args.sparsity.split(",")]:
            for method in ("dense", "dropout_dense", "block_dropout_dense", "sparsedrop"):
                if method == "sparsedrop":
                    lay = sd.LayerPlan(x, w, dy, p, dy_ready=True)
                    fwd = lambda i, lay=lay: lay.forward(sd.effective_seed(0, i, 0))  # noqa: E731
                    bwd = lambda i, lay=lay: lay.backward()  # noqa: E731
                else:
                    lay = BaselineLayer(method, x, w, dy, p)
                    fwd = lambda i, lay=lay: lay.forward(i)  # noqa: E731
                    bwd = lambda i, lay=lay: lay.backward()  # noqa: E731
                for i in range(args.warmup):
                    fwd(i), bwd(i)
                torch.cuda.synchronize()
                tf, tb, tt = [], [], []
                for i in range(args.repeats):
                    flush_buf.fill_(1.0)
                    if not args.no_gate:
                        torch.cuda._sleep(200000)  # ~100 us: covers the host enqueue of the pass
                    e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
                    e0.record()
                    fwd(1000 + i)
                    e1.record()
                    bwd(1000 + i)
                    e2.record()
                    e2.synchronize()
                    tf.append(e0.elapsed_time(e1) * 1e6)
                    tb.append(e1.elapsed_time(e2) * 1e6)
                    tt.append(e0.elapsed_time(e2) * 1e6)
                if method == "sparsedrop":
                    keep = lay.mask.keep_count()
                    realized = 1.0 - keep / lay.mask.total_blocks()
                    fl = 2 * N * 128 * 128 * keep  # flops_effective (gemm.hpp:222-228), per GEMM
                    # honesty: device work counter == keep-count prediction
                    cnt = sd.KernelCounters()
                    sd.dsd_matmul(x, lay.mask, w, 1.0, counters=cnt)
                    assert cnt.kblock_iterations == keep * (N // 128), (cnt.kblock_iterations, keep)
                elif method == "block_dropout_dense":
                    realized = 1.0 - lay.mask.keep_count() / lay.mask.total_blocks()
                    fl = dense_flops
                else:
                    realized = p if method == "dropout_dense" else 0.0
                    fl = dense_flops
                for pass_, ts, mult in (("forward", tf, 1), ("backward", tb, 2), ("total", tt, 3)):
                    records.append(percentile_record(method, M, N, K, p, realized, pass_, ts, fl * mult))
                r = records[-1]
                print(f"{S} p={p:.1f} {method:20s} total median {r.nanos_median / 1e3:9.1f} us  "
                      f"{r.effective_gflops / 1e3:7.1f} TFLOP/s eff", flush=True)
                del lay
        del x, w, dy
        torch.cuda.empty_cache()
    Path(args.out).parent.mkdir(parents=True, exist_ok=True)
    emit_csv(records, args.out)
    print("wrote", args.out)


if __name__ == "__main__":
    main()
