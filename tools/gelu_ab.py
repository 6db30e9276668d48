import ctypes, sys, torch
libs = [ctypes.CDLL(p, mode=ctypes.RTLD_LOCAL) for p in sys.argv[1:3]]
n = 65536 * 3072
h = torch.randn(n, device="cuda").to(torch.bfloat16)
g = torch.randn(n, device="cuda").to(torch.bfloat16)
outs = [torch.empty_like(h) for _ in range(4)]
st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
for lib in libs:
    lib.sd_gelu_forward.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p]
    lib.sd_gelu_backward.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p]
res = {}
for r in range(6):
    for li, lib in enumerate(libs):
        for kind in ("fwd", "bwd"):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            if kind == "fwd":
                lib.sd_gelu_forward(h.data_ptr(), outs[2 * li].data_ptr(), n, st)
            else:
                lib.sd_gelu_backward(h.data_ptr(), g.data_ptr(), outs[2 * li + 1].data_ptr(), n, st)
            e1.record()
            torch.cuda.synchronize()
            res.setdefault((li, kind), []).append(e0.elapsed_time(e1) * 1e3)
for (li, kind), v in sorted(res.items()):
    t = sorted(v)[len(v) // 2]
    gb = (2 if kind == "fwd" else 3) * n * 2 / 1e9
    print(f"lib{li} {kind}: {t:.1f} us  {gb / (t * 1e-6):.0f} GB/s")
print("fwd equal", torch.equal(outs[0], outs[2]), "bwd equal", torch.equal(outs[1], outs[3]))
