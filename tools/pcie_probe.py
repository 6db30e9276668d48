"""PCIe copy rates on the GPU box: pinned H2D, D2H, and both at once (dev tool)."""
import torch

n_in, n_out = 96 * 2**20, 128 * 2**20
hi = torch.empty(n_in, dtype=torch.uint8).pin_memory()
ho = torch.empty(n_out, dtype=torch.uint8).pin_memory()
di = torch.empty(n_in, dtype=torch.uint8, device="cuda")
do = torch.empty(n_out, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def t(fn, reps=5):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best


def both():
    cur = torch.cuda.current_stream()
    s1.wait_stream(cur)
    s2.wait_stream(cur)
    with torch.cuda.stream(s1):
        di.copy_(hi, non_blocking=True)
    with torch.cuda.stream(s2):
        ho.copy_(do, non_blocking=True)
    cur.wait_stream(s1)
    cur.wait_stream(s2)


h2d = t(lambda: di.copy_(hi, non_blocking=True))
d2h = t(lambda: ho.copy_(do, non_blocking=True))
bt = t(both)
print(f"H2D 96 MiB: {h2d:.3f} ms ({n_in / h2d / 1e6:.1f} GB/s); D2H 128 MiB: {d2h:.3f} ms ({n_out / d2h / 1e6:.1f} GB/s); "
      f"both at once: {bt:.3f} ms ({(n_in + n_out) / bt / 1e6:.1f} GB/s combined)")
