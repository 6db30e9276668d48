"""The paper's comparison methods on the same B200 kernels (
PAPER.md:161 "Dense … Dropout + Dense … Block dropout + Dense", Fig. 4a).

  dense                : y = x W ; dx = dy W^T ; dw = x^T dy
  dropout_dense        : element mask m = sample_element_mask(seed', p)
                         (layer.hpp:69-76, bit-exact counter hash per element)
                         y  = s (x (.) m) W                (layer.hpp:105-111)
                         dx = s (dy W^T) (.) m ; dw = s (x (.) m)^T dy  (layer.hpp:148-156)
  block_dropout_dense  : the SparseDrop block mask, but applied elementwise to a
                         copy of x and followed by DENSE GEMMs (the naive way
                         the paper compares against)
  sparsedrop           : LayerPlan (the hot path)

All GEMMs are the same tcgen05 kernel (sd_gemm_ex); masking is one bf16 pass
(sd_dropout_apply). seed' = effective_seed(spec.seed, step, layer_index).
"""
from __future__ import annotations

import ctypes

import torch

from . import _capi
from .api import BlockMask, _dtype_code, _stream, check, dropout_scale, effective_seed, sample_mask, DropoutSpec

METHODS = ("dense", "dropout_dense", "block_dropout_dense", "sparsedrop")


class BaselineLayer:
    """Dense / dropout_dense / block_dropout_dense layer step on bound buffers."""

    def __init__(self, method: str, x: torch.Tensor, w: torch.Tensor, dy: torch.Tensor, p: float,
                 seed: int = 0, layer_index: int = 0, m_blk: int = 128, k_blk: int = 128,
                 dw_dtype=torch.float32):
        if method not in METHODS[:3]:
            raise ValueError(f"unknown baseline method {method!r}")
        self.method, self.p, self.seed, self.layer_index = method, p, seed, layer_index
        self.x, self.w, self.dy = x, w, dy
        m, k = x.shape
        n = w.shape[1]
        self.m, self.n, self.k = m, n, k
        self.scale = dropout_scale(p) if method != "dense" else 1.0
        self.xm = torch.empty_like(x) if method != "dense" else x
        self.y = torch.empty(m, n, dtype=torch.bfloat16, device=x.device)
        self.dx = torch.empty(m, k, dtype=torch.bfloat16, device=x.device)
        self.dw = torch.empty(k, n, dtype=dw_dtype, device=x.device)
        self.mask = BlockMask(m // m_blk, k // k_blk, m_blk, k_blk, device=x.device) if method == "block_dropout_dense" else None
        self.m_blk, self.k_blk = m_blk, k_blk
        self._seed_eff = 0

    def _apply(self, src, dst, scale, stream):
        lib = _capi.load()
        mask_ptr = self.mask.cptr() if self.mask is not None else None
        check(lib.sd_dropout_apply(src.data_ptr(), dst.data_ptr(), src.shape[0], src.shape[1], self._seed_eff,
                                   float(self.p), float(scale), mask_ptr, ctypes.c_void_p(_stream(stream))))

    def forward(self, step_seed: int, stream=None):
        lib = _capi.load()
        st = ctypes.c_void_p(_stream(stream))
        if self.method != "dense":
            self._seed_eff = effective_seed(self.seed, step_seed, self.layer_index)
            if self.mask is not None:
                sample_mask(DropoutSpec(self.p, self.m_blk, self.k_blk, self._seed_eff), self.m, self.k,
                            stream=stream, out=self.mask)
            self._apply(self.x, self.xm, 1.0, stream)
        check(lib.sd_gemm_ex(self.xm.data_ptr(), 0, self.w.data_ptr(), 1, self.y.data_ptr(),
                             _dtype_code(self.y.dtype), self.m, self.n, self.k, self.scale, st))
        return self.y

    def backward(self, stream=None):
        lib = _capi.load()
        st = ctypes.c_void_p(_stream(stream))
        # dw = s (x (.) m)^T dy ; dx = s (dy W^T) (.) m
        check(lib.sd_gemm_ex(self.xm.data_ptr(), 1, self.dy.data_ptr(), 1, self.dw.data_ptr(),
                             _dtype_code(self.dw.dtype), self.k, self.n, self.m, self.scale, st))
        check(lib.sd_gemm_ex(self.dy.data_ptr(), 0, self.w.data_ptr(), 0, self.dx.data_ptr(),
                             _dtype_code(self.dx.dtype), self.m, self.k, self.n, self.scale, st))
        if self.method != "dense":
            self._apply(self.dx, self.dx, 1.0, stream)
        return self.dx, self.dw
