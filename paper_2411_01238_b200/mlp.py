"""The SparseDrop MLP block (BASELINE configs[2]): the direct
caller of the hot path in the paper's ViT-B experiments (§4).

  forward : h = SparseDrop_L0(x) W1 ; a = GELU(h) ; y = SparseDrop_L1(a) W2
  backward: dW2, da  <- layer backward of fc2 (mask L1)
            dh = da * GELU'(h)
            dW1, dx  <- layer backward of fc1 (mask L0)

One block mask per (layer, step): seed_l = counter_hash(spec.seed, step, l)
(layer.hpp:64-67). Both Linears run on the B200 SparseDrop kernels (LayerPlan);
GELU and its derivative are single-pass bf16 kernels of the same library
(sd_gelu_forward / sd_gelu_backward; fusing them into the GEMM epilogues is
listed as future work in DESIGN.md).
"""
from __future__ import annotations

import math

import torch

from . import _capi
from .api import LayerPlan, _stream, check, effective_seed


def gelu(h: torch.Tensor, out: torch.Tensor = None, stream=None) -> torch.Tensor:
    """Exact GELU, bf16 in/out, one pass (sd_gelu_forward; large inputs read a
    64 K-entry table of every bf16 pattern, built with the same math)."""
    out = torch.empty_like(h) if out is None else out
    check(_capi.load().sd_gelu_forward(h.data_ptr(), out.data_ptr(), h.numel(), _stream(stream)))
    return out


def gelu_grad(h: torch.Tensor, g: torch.Tensor, out: torch.Tensor = None, stream=None) -> torch.Tensor:
    """dL/dh = g * GELU'(h), bf16, one pass (sd_gelu_backward)."""
    out = torch.empty_like(h) if out is None else out
    check(_capi.load().sd_gelu_backward(h.data_ptr(), g.data_ptr(), out.data_ptr(), h.numel(), _stream(stream)))
    return out


def gelu_reference(h: torch.Tensor) -> torch.Tensor:
    """torch fp32 reference of gelu() (tests)."""
    return torch.nn.functional.gelu(h.float()).to(torch.bfloat16)


def gelu_grad_reference(h: torch.Tensor, g: torch.Tensor) -> torch.Tensor:
    """torch fp32 reference of gelu_grad() (tests)."""
    hf = h.float()
    cdf = 0.5 * (1.0 + torch.erf(hf * (1.0 / math.sqrt(2.0))))
    pdf = torch.exp(-0.5 * hf * hf) * (1.0 / math.sqrt(2.0 * math.pi))
    return (g.float() * (cdf + hf * pdf)).to(torch.bfloat16)


class SparseDropMLP:
    """Two SparseDrop Linears with GELU between, bf16 activations, fp32 weight
    gradients. Buffers are bound once (two LayerPlans)."""

    def __init__(self, x: torch.Tensor, w1: torch.Tensor, w2: torch.Tensor, dy: torch.Tensor, p: float,
                 seed: int = 0, dense: bool = False):
        m, d = x.shape
        hdim = w1.shape[1]
        if w1.shape[0] != d or w2.shape != (hdim, d) or dy.shape != (m, d):
            raise ValueError("SparseDropMLP shapes: x (m,d), w1 (d,h), w2 (h,d), dy (m,d)")
        self.p, self.seed, self.dense = p, seed, dense
        dev = x.device
        self.x, self.dy = x, dy
        self.act = torch.empty(m, hdim, dtype=torch.bfloat16, device=dev)   # GELU(h), fc2's input
        self.dact = torch.empty(m, hdim, dtype=torch.bfloat16, device=dev)  # dL/dh, fc1's output grad
        # fc1: x -> h (plan writes y = h); fc2: act -> y
        self.fc1 = LayerPlan(x, w1, self.dact, p)
        self.fc2 = LayerPlan(self.act, w2, dy, p, dy_ready=True)  # dy is the caller's, ready before the step

    def step(self, step_seed: int, stream=None):
        f1, f2 = self.fc1, self.fc2
        if self.dense:
            f1.dense_forward(stream)
        else:
            f1.forward(effective_seed(self.seed, step_seed, 0), stream)
        h = f1.y
        gelu(h, out=self.act, stream=stream)
        if self.dense:
            f2.dense_forward(stream)
            f2.dense_backward(stream)
        else:
            f2.forward(effective_seed(self.seed, step_seed, 1), stream)
            f2.backward(stream)
        # fc2.dx = dL/d(act); dL/dh = that * GELU'(h)
        gelu_grad(h, f2.dx, out=self.dact, stream=stream)
        if self.dense:
            f1.dense_backward(stream)
        else:
            f1.backward(stream)
        return f2.y, f1.dx, f1.dw, f2.dw
