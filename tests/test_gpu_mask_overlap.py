"""Mask regeneration and the backward overlapping their predecessors (GPU).

A layer plan's next sample_mask (layer.hpp:94, one mask per fwd/bwd pair)
writes into the same workspace the previous backward is still reading. The
library lets that generation start during the backward's tail: each GEMM CTA
releases the workspace once its list reads are done, and the generation waits
for the count of reader CTAs instead of for the whole preceding grid
(sd_internal.h, reader tracking). A plan's backward right after its forward
skips the wait for the forward grid (it needs nothing the forward writes) and
fills the SMs the forward's last wave leaves idle. These tests enqueue many steps back to back
— several plans sharing ONE bound mask workspace, no host sync and no other
kernel in between — and require every step's outputs to be bit-identical to
the same steps run one at a time with a device sync after each."""
import ctypes

import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def sd():
    assert torch.cuda.is_available(), "GPU tests need a B200"
    import paper_2411_01238_b200 as sd

    sd.load_library()
    return sd


def _bound_mask(lib, SdBlockMask, R, C):
    nbytes = lib.sd_mask_workspace_bytes(R, C)
    ws = torch.zeros(nbytes + 256, dtype=torch.uint8, device="cuda")
    m = SdBlockMask()
    assert lib.sd_mask_bind(ctypes.byref(m), ctypes.c_void_p((ws.data_ptr() + 255) & ~255), R, C, 128, 128, 0) == 0
    return ws, m


class _Plans:
    """`nplans` C-ABI layer plans over the same operands and ONE mask workspace,
    each with its own outputs (so every step's results survive)."""

    def __init__(self, sd, M, N, K, p, nplans):
        from paper_2411_01238_b200._capi import SdBlockMask

        self.lib = lib = sd.load_library()
        g = torch.Generator(device="cuda").manual_seed(7)
        self.x = torch.randn(M, K, device="cuda", generator=g).to(torch.bfloat16)
        self.w = torch.randn(K, N, device="cuda", generator=g).to(torch.bfloat16)
        self.dy = torch.randn(M, N, device="cuda", generator=g).to(torch.bfloat16)
        self.ws, self.mask = _bound_mask(lib, SdBlockMask, M // 128, K // 128)
        self.plans, self.outs = [], []
        for _ in range(nplans):
            y = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
            dx = torch.empty(M, K, dtype=torch.bfloat16, device="cuda")
            dw = torch.empty(K, N, dtype=torch.float32, device="cuda")
            plan = ctypes.c_void_p()
            rc = lib.sd_layer_plan_create(ctypes.byref(plan), ctypes.c_void_p(self.x.data_ptr()),
                                          ctypes.c_void_p(self.w.data_ptr()), ctypes.c_void_p(self.dy.data_ptr()),
                                          ctypes.c_void_p(y.data_ptr()), 1, ctypes.c_void_p(dx.data_ptr()), 1,
                                          ctypes.c_void_p(dw.data_ptr()), 0, M, N, K, ctypes.c_double(p),
                                          ctypes.byref(self.mask))
            assert rc == 0, lib.sd_last_error()
            self.plans.append(plan)
            self.outs.append((y, dx, dw))

    def step(self, i, seed, fused, sync=False):
        st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
        pl = self.plans[i]
        assert self.lib.sd_layer_plan_forward(pl, ctypes.c_uint64(seed), st) == 0
        if sync:  # the backward then waits for the forward grid like any launch
            torch.cuda.synchronize()
        if fused:
            assert self.lib.sd_layer_plan_backward(pl, st) == 0
        else:
            assert self.lib.sd_layer_plan_backward_dw(pl, st) == 0
            assert self.lib.sd_layer_plan_backward_dx(pl, st) == 0

    def snapshot(self):
        return [[t.clone() for t in o] for o in self.outs]

    def close(self):
        for pl in self.plans:
            self.lib.sd_layer_plan_destroy(pl)


@pytest.mark.parametrize("M,N,K,p", [(2048, 2048, 2048, 0.5), (4096, 4096, 4096, 0.5), (1024, 3072, 768, 0.1),
                                     (2048, 1024, 2048, 0.9)])
@pytest.mark.parametrize("fused", [True, False])
def test_back_to_back_steps_equal_serialized_steps(sd, M, N, K, p, fused):
    steps = 8
    P = _Plans(sd, M, N, K, p, steps)
    try:
        seeds = [1000 + 17 * i for i in range(steps)]
        waits0 = P.lib.sd_dev_mask_counter_waits()
        # back to back: mask(i+1) may run while backward(i) finishes
        for rep in range(2):  # second pass: every generation has pending readers
            for i in range(steps):
                P.step(i, seeds[i], fused)
        torch.cuda.synchronize()
        overlapped = P.snapshot()
        waits = P.lib.sd_dev_mask_counter_waits() - waits0
        # the counter protocol must actually have been used (all but the very
        # first generation into the fresh workspace)
        assert waits >= 2 * steps - 1, waits
        for o in P.outs:
            for t in o:
                t.fill_(float("nan"))
        for i in range(steps):
            P.step(i, seeds[i], fused, sync=True)
            torch.cuda.synchronize()
        serial = P.snapshot()
        for i in range(steps):
            for name, a, b in zip(("y", "dx", "dw"), overlapped[i], serial[i]):
                assert torch.equal(a, b), f"step {i} {name} differs when steps overlap"
    finally:
        P.close()


def test_two_layers_interleaved(sd):
    """fc1/fc2-like pattern: two workspaces, forward 0, forward 1, backward 1,
    backward 0, repeated without sync; equals the serialized run."""
    A = _Plans(sd, 2048, 1536, 1024, 0.5, 4)
    B = _Plans(sd, 2048, 1024, 1536, 0.3, 4)
    try:
        st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)

        def run(sync):
            for i in range(4):
                assert A.lib.sd_layer_plan_forward(A.plans[i], ctypes.c_uint64(11 + i), st) == 0
                assert B.lib.sd_layer_plan_forward(B.plans[i], ctypes.c_uint64(91 + i), st) == 0
                assert B.lib.sd_layer_plan_backward(B.plans[i], st) == 0
                assert A.lib.sd_layer_plan_backward(A.plans[i], st) == 0
                if sync:
                    torch.cuda.synchronize()
            torch.cuda.synchronize()
            return A.snapshot(), B.snapshot()

        run(False)
        o = run(False)
        s = run(True)
        for got, ref in zip(o, s):
            for i in range(4):
                for a, b in zip(got[i], ref[i]):
                    assert torch.equal(a, b)
    finally:
        A.close()
        B.close()


def test_untracked_reader_forces_full_wait(sd):
    """A 2-CTA union-mode launch over the workspace's lists does not release:
    the next generation into that workspace must not use the counter."""
    P = _Plans(sd, 1024, 1024, 1024, 0.5, 1)
    P.lib.sd_set_tuning(2097152)  # kTuneNoSmallHash: this plan's GEMMs read the lists (counter protocol)
    try:
        P.step(0, 5, True)
        torch.cuda.synchronize()
        lib = P.lib
        m = P.mask
        # a union-mode dsd call whose pair lists live inside the bound workspace
        # (contents irrelevant: counts forced to 0 so the GEMM writes zeros)
        cnt_ptr = ctypes.cast(m.row_cnt, ctypes.c_void_p).value
        zeros = torch.zeros(1024 * 1024, dtype=torch.float32, device="cuda")
        torch.cuda.synchronize()
        w0 = lib.sd_dev_mask_counter_waits()
        st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
        pair_cnt = torch.zeros(4, dtype=torch.int32, device="cuda")
        rc = lib.sd_dev_dsd_pairs(ctypes.c_void_p(P.x.data_ptr()), ctypes.c_void_p(P.w.data_ptr()),
                                  ctypes.c_void_p(zeros.data_ptr()), 0, 1024, 1024, 1024, 0, 128,
                                  ctypes.c_void_p(pair_cnt.data_ptr()), ctypes.c_void_p(cnt_ptr), 8,
                                  ctypes.c_float(1.0), st)
        assert rc == 0, lib.sd_last_error()
        P.step(0, 6, True)  # generation after an untracked reader: full wait
        assert lib.sd_dev_mask_counter_waits() == w0
        P.step(0, 7, True)  # tracked readers only again: counter mode
        assert lib.sd_dev_mask_counter_waits() == w0 + 1
        torch.cuda.synchronize()
    finally:
        P.lib.sd_set_tuning(0)
        P.close()


@pytest.mark.parametrize("M,N,K,p", [(1024, 1024, 1024, 0.5), (512, 768, 1536, 0.1), (1024, 512, 1024, 0.9)])
@pytest.mark.parametrize("fused", [True, False])
def test_small_plans_back_to_back_equal_serialized(sd, M, N, K, p, fused):
    """Small plans (hash-mode GEMMs, the mask generation after the forward and
    off the critical path, generations into the shared workspace chained through
    ticket word 2): several plans sharing ONE workspace, steps back to back,
    bit-identical to the same steps one at a time."""
    steps = 6
    P = _Plans(sd, M, N, K, p, steps)
    try:
        seeds = [2000 + 31 * i for i in range(steps)]
        for rep in range(2):
            for i in range(steps):
                P.step(i, seeds[i], fused)
        torch.cuda.synchronize()
        overlapped = P.snapshot()
        for o in P.outs:
            for t in o:
                t.fill_(float("nan"))
        for i in range(steps):
            P.step(i, seeds[i], fused, sync=True)
            torch.cuda.synchronize()
        serial = P.snapshot()
        for i in range(steps):
            for name, a, b in zip(("y", "dx", "dw"), overlapped[i], serial[i]):
                assert torch.equal(a, b), f"step {i} {name} differs when small steps overlap"
    finally:
        P.close()


def test_overlap_switches_do_not_change_results(sd):
    """Tuning bits 128 (backward waits for the forward) and 256 (generation
    waits for the whole preceding grid) give the same bits as the default."""
    P = _Plans(sd, 2048, 2048, 2048, 0.5, 3)
    try:
        outs = []
        for bits in (0, 128 | 256, 0):
            P.lib.sd_set_tuning(bits)
            for i in range(3):
                P.step(i, 40 + i, True)
            torch.cuda.synchronize()
            outs.append(P.snapshot())
        for o in outs[1:]:
            for i in range(3):
                for a, b in zip(o[i], outs[0][i]):
                    assert torch.equal(a, b)
    finally:
        P.lib.sd_set_tuning(0)
        P.close()


def test_aliased_buffers_keep_the_backward_waiting(sd):
    """dY aliasing Y (the forward's output is the backward's input): the plan
    must not start its backward before the forward grid completes."""
    from paper_2411_01238_b200._capi import SdBlockMask

    lib = sd.load_library()
    M = N = K = 2048
    g = torch.Generator(device="cuda").manual_seed(3)
    x = torch.randn(M, K, device="cuda", generator=g).to(torch.bfloat16)
    w = (torch.randn(K, N, device="cuda", generator=g) * 0.05).to(torch.bfloat16)
    ydy = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
    dx = torch.empty(M, K, dtype=torch.bfloat16, device="cuda")
    dw = torch.empty(K, N, dtype=torch.float32, device="cuda")
    ws, mask = _bound_mask(lib, SdBlockMask, M // 128, K // 128)
    plan = ctypes.c_void_p()
    assert lib.sd_layer_plan_create(ctypes.byref(plan), ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(w.data_ptr()),
                                    ctypes.c_void_p(ydy.data_ptr()), ctypes.c_void_p(ydy.data_ptr()), 1,
                                    ctypes.c_void_p(dx.data_ptr()), 1, ctypes.c_void_p(dw.data_ptr()), 0, M, N, K,
                                    ctypes.c_double(0.5), ctypes.byref(mask)) == 0
    st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    try:
        res = []
        for sync in (False, True):
            for rep in range(3):
                ydy.zero_()
                assert lib.sd_layer_plan_forward(plan, ctypes.c_uint64(77), st) == 0
                if sync:
                    torch.cuda.synchronize()
                assert lib.sd_layer_plan_backward(plan, st) == 0
                torch.cuda.synchronize()
                res.append((dx.clone(), dw.clone()))
        for a, b in res[1:]:
            assert torch.equal(a, res[0][0]) and torch.equal(b, res[0][1])
        assert res[0][1].abs().sum() > 0
    finally:
        lib.sd_layer_plan_destroy(plan)
