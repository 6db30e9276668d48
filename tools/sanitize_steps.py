"""Plan steps for compute-sanitizer (memcheck / racecheck / synccheck).

Runs `--steps` back-to-back SparseDrop layer steps (mask generation + forward +
fused backward, a fresh seed per step) on a few shapes that reach every launch
path of the library: the narrow and wide 1-CTA kernels, split-K dW, the masked
2-CTA dense dX (p <= 0.2), the 2-CTA dense step (p = 0), long kept lists
(> 64 entries per unit) and the cross-step launch overlap (mask generation
waiting on the reader release counter). SD_TUNING=384 in the environment turns
both overlaps off (every launch waits for the whole preceding grid).

  compute-sanitizer --tool memcheck python tools/sanitize_steps.py --steps 512
"""
import argparse
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

import paper_2411_01238_b200 as sd  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=512)
    ap.add_argument("--cases", default="all")
    args = ap.parse_args()
    torch.cuda.set_device(0)
    g = torch.Generator(device="cuda")
    g.manual_seed(5)

    def rnd(r, c):
        return (torch.rand(r, c, generator=g, device="cuda") - 0.5).to(torch.bfloat16)

    # (M, N, K, p): 1024^3 fused narrow backward; wide forward + split-K dW
    # (MLP-like dW); masked 2-CTA dense dX; dense p = 0; p = 0.9; dW lists of ~90
    # entries (> the 64-entry smem staging: per-CTA release)
    cases = [(1024, 1024, 1024, 0.5), (16384, 512, 256, 0.5), (2048, 1024, 2048, 0.1), (1024, 1024, 1024, 0.0),
             (1024, 1536, 1024, 0.9), (16384, 4096, 4096, 0.3)]
    if args.cases != "all":
        cases = [cases[int(i)] for i in args.cases.split(",")]
    per_case = max(1, args.steps // len(cases))
    n0 = sd.launch_count()
    for i_case, (M, N, K, p) in enumerate(cases):
        x, w, dy = rnd(M, K), rnd(K, N), rnd(M, N)
        plan = sd.LayerPlan(x, w, dy, p, dy_ready=(i_case % 2 == 0))
        for i in range(per_case):
            plan.forward(seed=sd.effective_seed(0, i, 0))
            plan.backward()
        torch.cuda.synchronize()
        del plan
    torch.cuda.synchronize()
    print(f"sanitize_steps ok: {per_case * len(cases)} steps, {sd.launch_count() - n0} launches")


if __name__ == "__main__":
    main()
