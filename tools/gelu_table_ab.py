import ctypes, sys, torch
sys.path.insert(0, "/root/repo")
import paper_2411_01238_b200 as sd
lib = sd.load_library()
n = 65536 * 3072
h = (torch.randn(n, device="cuda") * 2).to(torch.bfloat16)
g = torch.randn(n, device="cuda").to(torch.bfloat16)
o = [torch.empty_like(h) for _ in range(2)]
st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
res = {0: [], 512: []}
for r in range(8):
    for i, t in enumerate((0, 512)):
        lib.sd_set_tuning(t)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); lib.sd_gelu_backward(ctypes.c_void_p(h.data_ptr()), ctypes.c_void_p(g.data_ptr()), ctypes.c_void_p(o[i].data_ptr()), ctypes.c_int64(n), st); e1.record()
        torch.cuda.synchronize(); res[t].append(e0.elapsed_time(e1) * 1e3)
lib.sd_set_tuning(0)
for t, v in res.items():
    m = sorted(v)[len(v) // 2]; print(f"tuning {t}: gelu bwd {m:.1f} us  {3 * n * 2 / (m * 1e-6) / 1e9:.0f} GB/s")
print("equal", torch.equal(o[0], o[1]))
