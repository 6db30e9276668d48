"""Host-buffer SparseDrop layer steps with copy/compute overlap.

A caller whose X, W, dY live in (pinned) host memory and who wants Y, dX, dW
back in host memory every step — the reference-facing contract, where
`forward`/`backward` take and return host matrices (layer.hpp:85-162). On B200
the step is PCIe-bound (at 4096^3: 96 MiB in, 128 MiB out vs ~0.25 ms of GPU
work), so steps rotate over `nslots` buffer sets (default 2; 3 measured no faster) across three streams:

    h2d stream : inputs of step i+1      ─┐ overlap
    compute    : mask + fwd + bwd of i    ├─ (PCIe is full duplex)
    d2h stream : outputs of step i-1     ─┘

Every step still moves all of its inputs in and all of its outputs out.
"""
from __future__ import annotations

import torch

from .api import LayerPlan, effective_seed


class HostLayerPipeline:
    def __init__(self, x_host: torch.Tensor, w_host: torch.Tensor, dy_host: torch.Tensor, p: float,
                 row_block_offset: int = 0, device=None, dw_dtype=torch.float32, seed: int = 0,
                 layer_index: int = 0, nslots: int = 2):
        for name, t in (("x", x_host), ("w", w_host), ("dy", dy_host)):
            if t.is_cuda or t.dtype != torch.bfloat16 or not t.is_contiguous():
                raise ValueError(f"{name} must be a contiguous bf16 host tensor")
        dev = device if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.host_in = (x_host, w_host, dy_host)
        self.seed, self.layer_index = seed, layer_index
        self.slots = []
        if nslots < 2:
            raise ValueError("nslots must be >= 2")
        for _ in range(nslots):
            xd = torch.empty_like(x_host, device=dev)
            wd = torch.empty_like(w_host, device=dev)
            dyd = torch.empty_like(dy_host, device=dev)
            plan = LayerPlan(xd, wd, dyd, p, row_block_offset=row_block_offset, dw_dtype=dw_dtype,
                             dy_ready=True)  # dY is uploaded (h2d stream) before the forward
            self.slots.append({
                "in": (xd, wd, dyd), "plan": plan,
                "h2d": torch.cuda.Event(), "cmp": torch.cuda.Event(), "d2h": torch.cuda.Event(),
                "out": tuple(torch.empty(t.shape, dtype=t.dtype).pin_memory() for t in (plan.y, plan.dx, plan.dw)),
                "used": False,
            })
        self.s_h2d = torch.cuda.Stream(device=dev)
        self.s_cmp = torch.cuda.Stream(device=dev)
        self.s_d2h = torch.cuda.Stream(device=dev)
        self.h2d_bytes = sum(t.numel() * t.element_size() for t in self.host_in)
        p0 = self.slots[0]["plan"]
        self.d2h_bytes = sum(t.numel() * t.element_size() for t in (p0.y, p0.dx, p0.dw))

    def step(self, i: int, allreduce_dw=None):
        """Enqueue step i (asynchronous). Returns the host output tensors of this
        step (valid once `outputs_ready(i)` / synchronize)."""
        sl = self.slots[i % len(self.slots)]
        plan = sl["plan"]
        if sl["used"]:
            self.s_h2d.wait_event(sl["cmp"])   # step i - nslots finished reading this slot's inputs
        with torch.cuda.stream(self.s_h2d):
            for d, h in zip(sl["in"], self.host_in):
                d.copy_(h, non_blocking=True)
            sl["h2d"].record(self.s_h2d)
        self.s_cmp.wait_event(sl["h2d"])
        if sl["used"]:
            self.s_cmp.wait_event(sl["d2h"])   # step i - nslots's outputs of this slot are on the host
        with torch.cuda.stream(self.s_cmp):
            plan.forward(effective_seed(self.seed, i, self.layer_index), stream=self.s_cmp)
            if allreduce_dw is None:
                plan.backward(stream=self.s_cmp)
            else:
                plan.backward_dw(stream=self.s_cmp)
                allreduce_dw(plan.dw)
                plan.backward_dx(stream=self.s_cmp)
            sl["cmp"].record(self.s_cmp)
        self.s_d2h.wait_event(sl["cmp"])
        with torch.cuda.stream(self.s_d2h):
            for h, d in zip(sl["out"], (plan.y, plan.dx, plan.dw)):
                h.copy_(d, non_blocking=True)
            sl["d2h"].record(self.s_d2h)
        sl["used"] = True
        return sl["out"]

    def synchronize(self):
        for s in (self.s_h2d, self.s_cmp, self.s_d2h):
            s.synchronize()
