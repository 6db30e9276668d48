"""Randomised stress of the launch-overlap protocol (GPU).

Random sequences of layer-plan operations (forward with a fresh seed, fused
backward, split backward, dX-only, dense forward/backward), standalone mask
generations and generic C-ABI readers of the shared workspace, over three plans:
two of them share ONE bound mask workspace, plans run at p = 0.1 (dX on the
masked 2-CTA dense kernel), 0.5 and 0.9. Every sequence is enqueued twice:
back to back with no synchronisation (mask generations overlap GEMM tails,
backwards skip the wait for their forward), then with a device sync after
every operation. The final contents of every output buffer must be
bit-identical between the two runs."""
import ctypes
import random

import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def sd():
    assert torch.cuda.is_available(), "GPU tests need a B200"
    import paper_2411_01238_b200 as sd

    sd.load_library()
    return sd


def _mask(lib, SdBlockMask, R, C):
    nbytes = lib.sd_mask_workspace_bytes(R, C)
    ws = torch.zeros(nbytes + 256, dtype=torch.uint8, device="cuda")
    m = SdBlockMask()
    assert lib.sd_mask_bind(ctypes.byref(m), ctypes.c_void_p((ws.data_ptr() + 255) & ~255), R, C, 128, 128, 0) == 0
    return ws, m


def test_random_operation_sequences(sd):
    from paper_2411_01238_b200._capi import SdBlockMask

    lib = sd.load_library()
    S = 4096
    g = torch.Generator(device="cuda").manual_seed(5)
    shared_ws, shared_mask = _mask(lib, SdBlockMask, S // 128, S // 128)
    own_ws, own_mask = _mask(lib, SdBlockMask, S // 128, S // 128)
    plans = []
    for p, mask in ((0.1, shared_mask), (0.5, shared_mask), (0.9, own_mask)):
        x, w, dy = (torch.randn(S, S, device="cuda", generator=g).to(torch.bfloat16) for _ in range(3))
        y = torch.empty(S, S, dtype=torch.bfloat16, device="cuda")
        dx = torch.empty(S, S, dtype=torch.bfloat16, device="cuda")
        dw = torch.empty(S, S, dtype=torch.float32, device="cuda")
        h = ctypes.c_void_p()
        assert lib.sd_layer_plan_create(ctypes.byref(h), ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(w.data_ptr()),
                                        ctypes.c_void_p(dy.data_ptr()), ctypes.c_void_p(y.data_ptr()), 1,
                                        ctypes.c_void_p(dx.data_ptr()), 1, ctypes.c_void_p(dw.data_ptr()), 0, S, S, S,
                                        ctypes.c_double(p), ctypes.byref(mask)) == 0
        plans.append({"h": h, "keep": (x, w, dy), "out": (y, dx, dw)})
    st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    ops = ["fwd", "fwd", "bwd", "bwd", "dw_dx", "dx", "dense_fwd", "dense_bwd", "sample", "generic_fwd"]
    scratch = torch.empty(S, S, dtype=torch.bfloat16, device="cuda")
    xs, ws_ = plans[0]["keep"][0], plans[0]["keep"][1]

    def run(seq, sync):
        for pi, op, seed in seq:
            h = plans[pi]["h"]
            if op == "fwd":
                rc = lib.sd_layer_plan_forward(h, ctypes.c_uint64(seed), st)
            elif op == "bwd":
                rc = lib.sd_layer_plan_backward(h, st)
            elif op == "dw_dx":
                rc = lib.sd_layer_plan_backward_dw(h, st) or lib.sd_layer_plan_backward_dx(h, st)
            elif op == "dx":
                rc = lib.sd_layer_plan_backward_dx(h, st)
            elif op == "dense_fwd":
                rc = lib.sd_layer_plan_dense_forward(h, st)
            elif op == "sample":
                # a standalone generation into the shared workspace (tracked readers
                # of its previous lists may still be running)
                rc = lib.sd_mask_sample(ctypes.byref(shared_mask), ctypes.c_uint64(seed), ctypes.c_double(0.3), S, S,
                                        st)
            elif op == "generic_fwd":
                # a generic C-ABI reader of the shared workspace's lists
                rc = lib.sd_linear_forward(ctypes.c_void_p(xs.data_ptr()), ctypes.byref(shared_mask),
                                           ctypes.c_void_p(ws_.data_ptr()), ctypes.c_float(1.25),
                                           ctypes.c_void_p(scratch.data_ptr()), 1, S, S, S, st)
            else:
                rc = lib.sd_layer_plan_dense_backward(h, st)
            assert rc == 0, lib.sd_last_error()
            if sync:
                torch.cuda.synchronize()
        torch.cuda.synchronize()
        return [t.clone() for pl in plans for t in pl["out"]] + [scratch.clone()]

    try:
        rng = random.Random(1234)
        for trial in range(12):
            # a shared-workspace plan's backward reads the mask of the LAST
            # generation into that workspace: keep forward/backward pairs per
            # workspace so both runs agree on which mask a backward sees
            seq = []
            for _ in range(24):
                pi = rng.randrange(3)
                seq.append((pi, "fwd", rng.randrange(1 << 30)))
                for _ in range(rng.randrange(3)):
                    seq.append((pi, rng.choice(ops[2:]), rng.randrange(1 << 30)))
            for t in [t for pl in plans for t in pl["out"]] + [scratch]:
                t.fill_(0)
            a = run(seq, sync=False)
            for t in [t for pl in plans for t in pl["out"]] + [scratch]:
                t.fill_(0)
            b = run(seq, sync=True)
            for i, (u, v) in enumerate(zip(a, b)):
                assert torch.equal(u, v), f"trial {trial}: buffer {i} differs between overlapped and serialized runs"
    finally:
        for pl in plans:
            lib.sd_layer_plan_destroy(pl["h"])


def test_concurrent_streams_keep_their_own_scheduler_slots(sd):
    """Persistent GEMM launches on several streams at once: each stream's
    launches take scheduler-counter slots from that stream's own ring
    (sd_capi.cu sched_slot), so a long launch on one stream never shares its
    work-stealing counters with launches on another, however many are issued
    meanwhile. Every output must equal the same GEMM run alone."""
    torch.manual_seed(11)
    streams = [torch.cuda.Stream() for _ in range(3)]
    # one long launch (70 units over a 65536-long reduction) and many short ones
    big_a = torch.randn(70 * 128, 16384, device="cuda").to(torch.bfloat16)
    big_b = torch.randn(16384, 256, device="cuda").to(torch.bfloat16)
    big_m = sd.sample_mask(sd.DropoutSpec(0.5, 128, 128, 3), 70 * 128, 16384)
    small = []
    for i in range(40):
        a = torch.randn(256, 512, device="cuda").to(torch.bfloat16)
        b = torch.randn(512, 256, device="cuda").to(torch.bfloat16)
        m = sd.sample_mask(sd.DropoutSpec(0.5, 128, 128, 100 + i), 256, 512)
        small.append((a, b, m))
    torch.cuda.synchronize()
    ref_big = sd.dsd_matmul(big_a, big_m, big_b, 2.0)
    ref_small = [sd.dsd_matmul(a, m, b, 2.0) for a, b, m in small]
    torch.cuda.synchronize()
    for rep in range(3):
        outs = [None] * len(small)
        with torch.cuda.stream(streams[0]):
            out_big = sd.dsd_matmul(big_a, big_m, big_b, 2.0, stream=streams[0])
        for j in range(8):  # > 64 launches per stream ring while the long launch runs
            for i, (a, b, m) in enumerate(small):
                st = streams[1 + (i + j) % 2]
                with torch.cuda.stream(st):
                    o = sd.dsd_matmul(a, m, b, 2.0, stream=st)
                if j == 7:
                    outs[i] = o
        torch.cuda.synchronize()
        assert torch.equal(out_big, ref_big), rep
        for i in range(len(small)):
            assert torch.equal(outs[i], ref_small[i]), (rep, i)
