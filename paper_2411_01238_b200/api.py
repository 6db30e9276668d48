"""Host-side mirror of the reference's C++ operator API on B200 device memory.

Names, argument meaning and error behaviour follow namespace ``sparsedrop`` of
the reference (/root/reference/proj/include/sparsedrop/): ``TileConfig``,
``DropoutSpec``, ``BlockMask``, ``sample_mask``, ``kept_blocks_in_row``,
``transpose_mask``, ``retile``, ``dense_gemm``, ``dsd_matmul``, ``sdd_matmul``,
``LinearLayer``, ``forward``, ``backward``, ``flops_dense``, ``flops_effective``.
Differences, all forced by the device:
  * matrices are CUDA ``torch.Tensor`` s (bf16 inputs, row-major contiguous) —
    torch is only the allocator / stream plumbing; every op is one call into
    libsparsedrop_b200.so through the C-ABI;
  * ``threads=`` is replaced by the current CUDA stream;
  * exceptions: std::invalid_argument -> ValueError, std::out_of_range ->
    IndexError, std::runtime_error -> RuntimeError.
"""
from __future__ import annotations

import ctypes
import dataclasses
import enum
from typing import Optional

import torch

from . import _capi
from ._capi import SD_DTYPE_BF16, SD_DTYPE_F32, SdBlockMask, check


def _lib():
    return _capi.load()


_get_raw_stream = getattr(torch._C, "_cuda_getCurrentRawStream", None)


def _cur_raw_stream(device: int) -> int:
    """The current stream of `device` as a raw handle (cheap: no Stream object)."""
    if _get_raw_stream is not None:
        return _get_raw_stream(device)
    return torch.cuda.current_stream(device).cuda_stream


def _stream(stream=None) -> int:
    if stream is not None:
        return stream.cuda_stream
    return _cur_raw_stream(torch.cuda.current_device())


def _ptr(t: Optional[torch.Tensor]) -> Optional[int]:
    return None if t is None else t.data_ptr()


def _dtype_code(dtype: torch.dtype) -> int:
    if dtype == torch.bfloat16:
        return SD_DTYPE_BF16
    if dtype == torch.float32:
        return SD_DTYPE_F32
    raise ValueError(f"unsupported output dtype {dtype} (bf16 or fp32)")


def _require_bf16(name: str, t: torch.Tensor) -> None:
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor (the B200 path has no CPU fallback)")
    if t.dtype != torch.bfloat16 or t.dim() != 2 or not t.is_contiguous():
        raise ValueError(f"{name} must be a contiguous 2-D bf16 tensor, got {t.dtype} {tuple(t.shape)}")


# --------------------------------------------------------------------------- rng.hpp

SD_PLAN_DY_READY = 1  # include/sparsedrop_b200.h
MASK64 = (1 << 64) - 1


def mix64(z: int) -> int:
    """rng.hpp:11-16 (host helper for seeds; the device kernel hashes the blocks)."""
    z = (z + 0x9E3779B97F4A7C15) & MASK64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
    return z ^ (z >> 31)


def counter_hash(seed: int, a: int, b: int) -> int:
    """rng.hpp:18-20."""
    return mix64(mix64(mix64(seed & MASK64) ^ (a & MASK64)) ^ (b & MASK64))


def effective_seed(spec_seed: int, step_seed: int, layer_index: int) -> int:
    """layer.hpp:64-67: one seed per (layer instance, step)."""
    return counter_hash(spec_seed, step_seed, layer_index & MASK64)


def dropout_scale(p: float) -> float:
    """layer.hpp:78-81 dropout_scale<float>: float(1.0 / (1.0 - p))."""
    import numpy as np

    return float(np.float32(1.0 / (1.0 - p)))


# --------------------------------------------------------------------------- block_mask.hpp


@dataclasses.dataclass
class TileConfig:
    """block_mask.hpp:14-18. On B200 the kernel tile is fixed (128 x 256 x 64);
    TileConfig here only carries the mask block sizes used for validation."""

    m_blk: int = 128
    n_blk: int = 128
    k_blk: int = 128


@dataclasses.dataclass
class DropoutSpec:
    """block_mask.hpp:21-26."""

    p: float = 0.0
    m_blk: int = 128
    k_blk: int = 128
    seed: int = 0


class BlockMask:
    """Device-resident sparsedrop::BlockMask (block_mask.hpp:31-76) plus the
    compaction lists the GEMMs consume (row lists = kept_blocks_in_row, column
    lists = kept_blocks_in_row of transpose_mask)."""

    def __init__(self, block_rows: int, block_cols: int, m_blk: int, k_blk: int,
                 row_block_offset: int = 0, device=None):
        if block_rows <= 0 or block_cols <= 0 or m_blk <= 0 or k_blk <= 0:
            raise ValueError(
                f"BlockMask geometry must be positive: grid {block_rows}x{block_cols}, "
                f"blocks {m_blk}x{k_blk}")
        lib = _lib()
        nbytes = lib.sd_mask_workspace_bytes(block_rows, block_cols)
        dev = device if device is not None else torch.device("cuda", torch.cuda.current_device())
        # zero-initialised once: all-clear mask, re-armed completion ticket
        self._ws = torch.zeros(nbytes + 256, dtype=torch.uint8, device=dev)
        base = self._ws.data_ptr()
        aligned = (base + 255) & ~255
        self._c = SdBlockMask()
        check(lib.sd_mask_bind(ctypes.byref(self._c), ctypes.c_void_p(aligned), block_rows, block_cols,
                               m_blk, k_blk, row_block_offset))
        self._base_off = aligned - base
        self.device = self._ws.device

    # geometry (block_mask.hpp:41-52)
    def block_rows(self) -> int: return self._c.block_rows
    def block_cols(self) -> int: return self._c.block_cols
    def m_blk(self) -> int: return self._c.m_blk
    def k_blk(self) -> int: return self._c.k_blk
    def rows(self) -> int: return self._c.block_rows * self._c.m_blk
    def cols(self) -> int: return self._c.block_cols * self._c.k_blk
    def row_block_offset(self) -> int: return self._c.row_block_offset
    def total_blocks(self) -> int: return self._c.block_rows * self._c.block_cols
    def n_words(self) -> int: return (self.total_blocks() + 63) // 64

    def _view(self, field: str, count: int, dtype: torch.dtype) -> torch.Tensor:
        off = getattr(self._c, field) - self._ws.data_ptr()
        nbytes = count * torch.tensor([], dtype=dtype).element_size()
        return self._ws[off:off + nbytes].view(dtype)

    # device views (no copies)
    def words_device(self) -> torch.Tensor: return self._view("words", self.n_words(), torch.int64)
    def keep_count_device(self) -> torch.Tensor: return self._view("keep_count", 1, torch.int64)
    def row_cnt_device(self) -> torch.Tensor: return self._view("row_cnt", self.block_rows(), torch.int32)
    def row_idx_device(self) -> torch.Tensor:
        return self._view("row_idx", self.total_blocks(), torch.int32).view(self.block_rows(), self.block_cols())
    def col_cnt_device(self) -> torch.Tensor: return self._view("col_cnt", self.block_cols(), torch.int32)
    def col_idx_device(self) -> torch.Tensor:
        return self._view("col_idx", self.total_blocks(), torch.int32).view(self.block_cols(), self.block_rows())
    def row_order_device(self) -> torch.Tensor: return self._view("row_order", self.block_rows(), torch.int32)
    def col_order_device(self) -> torch.Tensor: return self._view("col_order", self.block_cols(), torch.int32)

    # host reads (block_mask.hpp:46-62)
    def words(self) -> list:
        return [w & MASK64 for w in self.words_device().cpu().tolist()]

    def keep_count(self) -> int:
        return int(self.keep_count_device().item())

    def realized_sparsity(self) -> float:
        t = self.total_blocks()
        return 0.0 if t == 0 else 1.0 - self.keep_count() / t

    def kept(self, block_row: int, block_col: int) -> bool:
        b = block_row * self.block_cols() + block_col
        w = int(self.words_device()[b >> 6].item()) & MASK64
        return bool((w >> (b & 63)) & 1)

    @property
    def c_struct(self) -> SdBlockMask:
        return self._c

    def cptr(self):
        return ctypes.byref(self._c)


def sample_mask(spec: DropoutSpec, rows: int, cols: int, row_block_offset: int = 0,
                stream=None, out: Optional[BlockMask] = None) -> BlockMask:
    """block_mask.cpp:52-80 on the device (bit-exact splitmix64 draw), plus the
    compaction lists. `row_block_offset` selects the global block rows of a
    row shard. Raises ValueError like the reference's invalid_argument."""
    if not (0.0 <= spec.p < 1.0):
        raise ValueError(f"dropout rate must lie in [0, 1), got {spec.p:f}")
    if spec.m_blk <= 0 or rows % spec.m_blk != 0:
        raise ValueError(f"mask block size m_blk={spec.m_blk} does not divide rows={rows}")
    if spec.k_blk <= 0 or cols % spec.k_blk != 0:
        raise ValueError(f"mask block size k_blk={spec.k_blk} does not divide cols={cols}")
    m = out if out is not None else BlockMask(rows // spec.m_blk, cols // spec.k_blk, spec.m_blk,
                                              spec.k_blk, row_block_offset)
    check(_lib().sd_mask_sample(m.cptr(), spec.seed & MASK64, float(spec.p), rows, cols,
                                ctypes.c_void_p(_stream(stream))))
    return m


def mask_from_words(block_rows: int, block_cols: int, m_blk: int, k_blk: int, words,
                    stream=None) -> BlockMask:
    """block_mask.cpp:82-98: validates word count and zero padding, uploads, compacts."""
    words = [int(w) & MASK64 for w in words]
    bits = block_rows * block_cols
    if len(words) != (bits + 63) // 64:
        raise ValueError(f"BlockMask word count {len(words)} does not match grid of {bits} bits")
    if bits & 63 and words[-1] & (MASK64 ^ ((1 << (bits & 63)) - 1)):
        raise ValueError("BlockMask has nonzero bits past the block grid")
    m = BlockMask(block_rows, block_cols, m_blk, k_blk)
    signed = [w - (1 << 64) if w >= (1 << 63) else w for w in words]
    m.words_device().copy_(torch.tensor(signed, dtype=torch.int64))
    check(_lib().sd_mask_compact(m.cptr(), ctypes.c_void_p(_stream(stream))))
    return m


def transpose_mask(mask: BlockMask, stream=None) -> BlockMask:
    """block_mask.cpp:117-123."""
    out = BlockMask(mask.block_cols(), mask.block_rows(), mask.k_blk(), mask.m_blk())
    check(_lib().sd_mask_transpose(mask.cptr(), out.cptr(), ctypes.c_void_p(_stream(stream))))
    return out


def retile(mask: BlockMask, split_m: int, split_k: int, stream=None) -> BlockMask:
    """block_mask.cpp:100-115."""
    if split_m <= 0 or mask.m_blk() % split_m != 0:
        raise ValueError(f"split_m={split_m} does not divide m_blk={mask.m_blk()}")
    if split_k <= 0 or mask.k_blk() % split_k != 0:
        raise ValueError(f"split_k={split_k} does not divide k_blk={mask.k_blk()}")
    out = BlockMask(mask.block_rows() * split_m, mask.block_cols() * split_k,
                    mask.m_blk() // split_m, mask.k_blk() // split_k)
    check(_lib().sd_mask_retile(mask.cptr(), split_m, split_k, out.cptr(), ctypes.c_void_p(_stream(stream))))
    return out


def kept_blocks_in_row(mask: BlockMask, block_row: int) -> list:
    """block_mask.cpp:125-135, read from the device row lists."""
    if block_row < 0 or block_row >= mask.block_rows():
        raise IndexError(f"block row {block_row} outside grid with {mask.block_rows()} rows")
    n = int(mask.row_cnt_device()[block_row].item())
    return mask.row_idx_device()[block_row, :n].cpu().tolist()


# --------------------------------------------------------------------------- gemm.hpp

@dataclasses.dataclass
class KernelCounters:
    """gemm.hpp:31-37: executed 128x128x128 block products per 128-row tile row."""

    kblock_iterations: int = 0
    kblock_per_tile_row: list = dataclasses.field(default_factory=list)


def _out(m: int, n: int, dtype: torch.dtype, device) -> torch.Tensor:
    return torch.empty(m, n, dtype=dtype, device=device)


def dense_gemm(a: torch.Tensor, b: torch.Tensor, out_dtype=torch.bfloat16, stream=None,
               out: Optional[torch.Tensor] = None) -> torch.Tensor:
    """gemm.hpp:104-128: c = a * b on the tcgen05 tensor cores."""
    _require_bf16("a", a), _require_bf16("b", b)
    if a.shape[1] != b.shape[0]:
        raise ValueError(f"gemm shape mismatch: {a.shape[0]}x{a.shape[1]} * {b.shape[0]}x{b.shape[1]}")
    m, k = a.shape
    n = b.shape[1]
    c = out if out is not None else _out(m, n, out_dtype, a.device)
    check(_lib().sd_dense_gemm(a.data_ptr(), b.data_ptr(), c.data_ptr(), _dtype_code(c.dtype), m, n, k,
                               ctypes.c_void_p(_stream(stream))))
    return c


def _counters_buf(rows: int, device, counters: Optional[KernelCounters]):
    if counters is None:
        return None
    return torch.zeros(rows // 128, dtype=torch.int64, device=device)


def _fill_counters(counters: Optional[KernelCounters], buf: Optional[torch.Tensor]) -> None:
    if counters is None:
        return
    per = buf.cpu().tolist()
    counters.kblock_per_tile_row = per
    counters.kblock_iterations = sum(per)


def dsd_matmul(a: torch.Tensor, mask: BlockMask, b: torch.Tensor, scale_factor: float,
               tiles: Optional[TileConfig] = None, counters: Optional[KernelCounters] = None,
               out_dtype=torch.bfloat16, stream=None, out: Optional[torch.Tensor] = None) -> torch.Tensor:
    """gemm.hpp:133-170: scale * (a (.) expand(mask)) * b; dropped K-blocks never read."""
    _require_bf16("a", a), _require_bf16("b", b)
    if a.shape[1] != b.shape[0]:
        raise ValueError(f"gemm shape mismatch: {a.shape[0]}x{a.shape[1]} * {b.shape[0]}x{b.shape[1]}")
    if tiles is not None and (tiles.m_blk != mask.m_blk() or tiles.k_blk != mask.k_blk()):
        raise ValueError("dsd_matmul: mask geometry does not match problem (tile sizes)")
    m, k = a.shape
    n = b.shape[1]
    c = out if out is not None else _out(m, n, out_dtype, a.device)
    cb = _counters_buf(m, a.device, counters)
    check(_lib().sd_dsd_matmul(a.data_ptr(), mask.cptr(), b.data_ptr(), float(scale_factor), c.data_ptr(),
                               _dtype_code(c.dtype), m, n, k, _ptr(cb), ctypes.c_void_p(_stream(stream))))
    _fill_counters(counters, cb)
    return c


def sdd_matmul(a: torch.Tensor, b: torch.Tensor, mask: BlockMask, scale_factor: float,
               tiles: Optional[TileConfig] = None, counters: Optional[KernelCounters] = None,
               out_dtype=torch.bfloat16, stream=None, out: Optional[torch.Tensor] = None) -> torch.Tensor:
    """gemm.hpp:176-213: scale * (a * b) on kept OUTPUT blocks, exact +0.0 elsewhere."""
    _require_bf16("a", a), _require_bf16("b", b)
    if a.shape[1] != b.shape[0]:
        raise ValueError(f"gemm shape mismatch: {a.shape[0]}x{a.shape[1]} * {b.shape[0]}x{b.shape[1]}")
    m, k = a.shape
    n = b.shape[1]
    c = out if out is not None else _out(m, n, out_dtype, a.device)
    cb = _counters_buf(m, a.device, counters)
    check(_lib().sd_sdd_matmul(a.data_ptr(), b.data_ptr(), mask.cptr(), float(scale_factor), c.data_ptr(),
                               _dtype_code(c.dtype), m, n, k, _ptr(cb), ctypes.c_void_p(_stream(stream))))
    _fill_counters(counters, cb)
    return c


class SparseKind(enum.Enum):
    dsd = 0
    sdd = 1


def flops_dense(m: int, n: int, k: int) -> int:
    """gemm.hpp:217-219."""
    return 2 * m * n * k


def flops_effective(m: int, n: int, k: int, tiles: TileConfig, mask: BlockMask, kind: SparseKind) -> int:
    """gemm.hpp:222-228."""
    keep = mask.keep_count()
    if kind == SparseKind.dsd:
        return 2 * n * tiles.m_blk * tiles.k_blk * keep
    return 2 * k * tiles.m_blk * tiles.n_blk * keep


# --------------------------------------------------------------------------- layer.hpp

class LinearVariant(enum.Enum):
    dense = 0
    dropout_dense = 1
    sparsedrop = 2


@dataclasses.dataclass
class LinearLayer:
    """layer.hpp:29-47. weight is K x N bf16 on the device."""

    kind: LinearVariant
    weight: torch.Tensor
    spec: DropoutSpec
    tiles: TileConfig = dataclasses.field(default_factory=TileConfig)
    layer_index: int = 0

    def __post_init__(self):
        if self.kind == LinearVariant.dropout_dense:
            raise ValueError("dropout_dense is not implemented on the B200 path (out of scope, SURVEY §8f2)")
        if self.kind == LinearVariant.sparsedrop and (
                self.spec.m_blk != self.tiles.m_blk or self.spec.k_blk != self.tiles.k_blk):
            raise ValueError("sparsedrop mask block sizes must equal the GEMM tile sizes")


@dataclasses.dataclass
class LayerContext:
    """layer.hpp:51-58 (the input is referenced, not copied)."""

    input: torch.Tensor
    block_mask: Optional[BlockMask] = None
    training: bool = False
    step_seed: int = 0


@dataclasses.dataclass
class LayerGrads:
    dx: torch.Tensor
    dw: torch.Tensor


def forward(layer: LinearLayer, x: torch.Tensor, train: bool, step_seed: int, stream=None,
            out_dtype=torch.bfloat16, mask_out: Optional[BlockMask] = None):
    """layer.hpp:85-117: returns (y, ctx). Training + sparsedrop samples one block
    mask per (layer, step) and runs the dsd forward; otherwise dense."""
    _require_bf16("x", x)
    if x.shape[1] != layer.weight.shape[0]:
        raise ValueError(f"layer forward: input {x.shape[0]}x{x.shape[1]} does not match weight "
                         f"{layer.weight.shape[0]}x{layer.weight.shape[1]}")
    ctx = LayerContext(input=x, training=train, step_seed=step_seed)
    if not train or layer.kind == LinearVariant.dense:
        return dense_gemm(x, layer.weight, out_dtype=out_dtype, stream=stream), ctx
    seed = effective_seed(layer.spec.seed, step_seed, layer.layer_index)
    s = dropout_scale(layer.spec.p)
    spec = dataclasses.replace(layer.spec, seed=seed)
    ctx.block_mask = sample_mask(spec, x.shape[0], x.shape[1], stream=stream, out=mask_out)
    m, k = x.shape
    n = layer.weight.shape[1]
    y = torch.empty(m, n, dtype=out_dtype, device=x.device)
    check(_lib().sd_linear_forward(x.data_ptr(), ctx.block_mask.cptr(), layer.weight.data_ptr(), s, y.data_ptr(),
                                   _dtype_code(out_dtype), m, n, k, ctypes.c_void_p(_stream(stream))))
    return y, ctx


def backward(layer: LinearLayer, ctx: LayerContext, dy: torch.Tensor, stream=None,
             dx_dtype=torch.bfloat16, dw_dtype=torch.float32) -> LayerGrads:
    """layer.hpp:128-162: dx = s (dy W^T) (.) m (sdd), dw = s (x (.) m)^T dy (dsd on
    column lists) — W and x are read in place, no transposes are materialised.
    dW is computed first so a data-parallel caller can start its allreduce while
    dX runs."""
    _require_bf16("dy", dy)
    x = ctx.input
    if dy.shape[0] != x.shape[0] or dy.shape[1] != layer.weight.shape[1]:
        raise ValueError(f"layer backward: dy {dy.shape[0]}x{dy.shape[1]} does not match forward shapes "
                         f"{x.shape[0]}x{x.shape[1]} * {layer.weight.shape[0]}x{layer.weight.shape[1]}")
    m, k = x.shape
    n = dy.shape[1]
    st = ctypes.c_void_p(_stream(stream))
    dx = torch.empty(m, k, dtype=dx_dtype, device=dy.device)
    dw = torch.empty(k, n, dtype=dw_dtype, device=dy.device)
    if not ctx.training or layer.kind == LinearVariant.dense or ctx.block_mask is None:
        check(_lib().sd_dense_gemm_tn(x.data_ptr(), dy.data_ptr(), dw.data_ptr(), _dtype_code(dw_dtype),
                                      k, n, m, st))
        check(_lib().sd_dense_gemm_nt(dy.data_ptr(), layer.weight.data_ptr(), dx.data_ptr(),
                                      _dtype_code(dx_dtype), m, k, n, st))
        return LayerGrads(dx, dw)
    s = dropout_scale(layer.spec.p)
    mask = ctx.block_mask
    check(_lib().sd_linear_backward_dw(x.data_ptr(), mask.cptr(), dy.data_ptr(), s, dw.data_ptr(),
                                       _dtype_code(dw_dtype), m, n, k, st))
    check(_lib().sd_linear_backward_dx(dy.data_ptr(), layer.weight.data_ptr(), mask.cptr(), s, dx.data_ptr(),
                                       _dtype_code(dx_dtype), m, n, k, st))
    return LayerGrads(dx, dw)


class LayerPlan:
    """A bound sparsedrop layer (C-ABI sd_layer_plan): buffers and tensor maps are
    fixed at construction, each step is 2 (forward) + 1 (backward; 2 at p <= 0.2,
    where dX runs on the masked 2-CTA dense kernel) kernel launches with no
    host-side work — the runtime object a training loop keeps
    per layer. Row shards pass `row_block_offset` (global block row of local row 0).

    forward(seed)   : mask = sample_mask(seed) ; y = s (x (.) m) w
    backward()      : dw = s (x (.) m)^T dy ; dx = s (dy w^T) (.) m

    dy_ready=True (SD_PLAN_DY_READY) declares that dy is written before each
    forward and never between a forward and its backward (a fixed or uploaded
    dy): the backward may then start in the forward's tail. Leave it False when
    a kernel between forward and backward produces dy.
    """

    def __init__(self, x: torch.Tensor, w: torch.Tensor, dy: torch.Tensor, p: float, m_blk: int = 128,
                 k_blk: int = 128, row_block_offset: int = 0, y_dtype=torch.bfloat16,
                 dx_dtype=torch.bfloat16, dw_dtype=torch.float32, dy_ready: bool = False):
        _require_bf16("x", x), _require_bf16("w", w), _require_bf16("dy", dy)
        m, k = x.shape
        n = w.shape[1]
        if w.shape[0] != k or dy.shape != (m, n):
            raise ValueError(f"layer shapes: x {tuple(x.shape)} w {tuple(w.shape)} dy {tuple(dy.shape)}")
        if m_blk <= 0 or m % m_blk:
            raise ValueError(f"mask block size m_blk={m_blk} does not divide rows={m}")
        if k_blk <= 0 or k % k_blk:
            raise ValueError(f"mask block size k_blk={k_blk} does not divide cols={k}")
        self.x, self.w, self.dy = x, w, dy
        self.m, self.n, self.k, self.p = m, n, k, p
        self.mask = BlockMask(m // m_blk, k // k_blk, m_blk, k_blk, row_block_offset, device=x.device)
        self.y = torch.empty(m, n, dtype=y_dtype, device=x.device)
        self.dx = torch.empty(m, k, dtype=dx_dtype, device=x.device)
        self.dw = torch.empty(k, n, dtype=dw_dtype, device=x.device)
        self._plan = ctypes.c_void_p()
        check(_lib().sd_layer_plan_create(ctypes.byref(self._plan), x.data_ptr(), w.data_ptr(), dy.data_ptr(),
                                          self.y.data_ptr(), _dtype_code(y_dtype), self.dx.data_ptr(),
                                          _dtype_code(dx_dtype), self.dw.data_ptr(), _dtype_code(dw_dtype),
                                          m, n, k, float(p), self.mask.cptr()))
        if dy_ready:
            check(_lib().sd_layer_plan_set_options(self._plan, SD_PLAN_DY_READY))
        self.scale = dropout_scale(p)
        # the per-step calls, bound once: a small layer's step is ~16 us of
        # device time, so the Python side of forward()/backward() is kept to
        # one C call each (no Stream objects, no ctypes wrappers per call)
        self._dev = x.device.index if x.device.index is not None else torch.cuda.current_device()
        lib = _lib()
        self._h = self._plan.value
        self._c_forward = lib.sd_layer_plan_forward
        self._c_backward = lib.sd_layer_plan_backward

    def _s(self, stream) -> int:
        return stream.cuda_stream if stream is not None else _cur_raw_stream(self._dev)

    def forward(self, seed: int, stream=None):
        rc = self._c_forward(self._h, seed & MASK64,
                             stream.cuda_stream if stream is not None else _cur_raw_stream(self._dev))
        if rc:
            check(rc)
        return self.y

    def backward(self, stream=None):
        rc = self._c_backward(self._h, stream.cuda_stream if stream is not None else _cur_raw_stream(self._dev))
        if rc:
            check(rc)
        return self.dx, self.dw

    def graph_step(self, seed: int, backward: bool = True, stream=None):
        """forward(seed) [+ backward()] as ONE CUDA-graph launch
        (sd_layer_plan_graph_step): for host-bound callers; same results."""
        check(_lib().sd_layer_plan_graph_step(self._plan, seed & MASK64, 3 if backward else 1,
                                               self._s(stream)))
        return self.y

    def backward_dw(self, stream=None):
        check(_lib().sd_layer_plan_backward_dw(self._plan, self._s(stream)))
        return self.dw

    def backward_dw_part(self, part: int, nparts: int, stream=None):
        """dW rows of mask-column blocks [C*part/nparts, C*(part+1)/nparts): returns
        that row slab of self.dw (bit-identical to the same rows of backward_dw)."""
        check(_lib().sd_layer_plan_backward_dw_part(self._plan, part, nparts, self._s(stream)))
        C, kb = self.mask.block_cols(), self.mask.k_blk()
        return self.dw[(C * part // nparts) * kb:(C * (part + 1) // nparts) * kb]

    def backward_allreduce(self, comm: "Communicator", nparts: int = 2, stream=None, comm_stream=None):
        """Row-shard backward with the dW all-reduce behind the C-ABI
        (sd_layer_plan_backward_allreduce): dW in `nparts` row slabs, each
        summed over the ranks by NCCL on `comm_stream` while the next slab and
        dX compute on `stream`; `stream` then waits for the last all-reduce."""
        cs = ctypes.c_void_p(_stream(comm_stream)) if comm_stream is not None else None
        check(_lib().sd_layer_plan_backward_allreduce(self._plan, comm._c, nparts, self._s(stream),
                                                      cs))
        return self.dx, self.dw

    def backward_dx(self, stream=None):
        check(_lib().sd_layer_plan_backward_dx(self._plan, self._s(stream)))
        return self.dx

    def dense_forward(self, stream=None):
        check(_lib().sd_layer_plan_dense_forward(self._plan, self._s(stream)))
        return self.y

    def dense_backward(self, stream=None):
        check(_lib().sd_layer_plan_dense_backward(self._plan, self._s(stream)))
        return self.dx, self.dw

    def __del__(self):
        try:
            if self._plan:
                _lib().sd_layer_plan_destroy(self._plan)
                self._plan = ctypes.c_void_p()
        except Exception:
            pass


class Communicator:
    """The library's NCCL communicator (sd_comm_*) for the data-parallel
    backward. `unique_id` (128 bytes) comes from rank 0's
    Communicator.new_unique_id() and is broadcast by the caller (e.g. with
    torch.distributed.broadcast_object_list)."""

    ID_BYTES = 128

    @staticmethod
    def new_unique_id() -> bytes:
        buf = ctypes.create_string_buffer(Communicator.ID_BYTES)
        check(_lib().sd_comm_unique_id(buf))
        return buf.raw

    def __init__(self, nranks: int, rank: int, unique_id: bytes):
        if len(unique_id) != self.ID_BYTES:
            raise ValueError(f"unique_id must be {self.ID_BYTES} bytes")
        self._c = ctypes.c_void_p()
        self.nranks, self.rank = nranks, rank
        check(_lib().sd_comm_init(ctypes.byref(self._c), nranks, rank, ctypes.create_string_buffer(unique_id,
                                                                                                    self.ID_BYTES)))

    def allreduce_sum(self, t: torch.Tensor, stream=None) -> torch.Tensor:
        if t.dtype not in (torch.float32, torch.bfloat16) or not t.is_contiguous():
            raise ValueError("allreduce_sum: contiguous fp32 or bf16 tensor")
        check(_lib().sd_comm_allreduce_sum(self._c, t.data_ptr(), t.numel(), _dtype_code(t.dtype),
                                           ctypes.c_void_p(_stream(stream))))
        return t

    @staticmethod
    def nccl_version() -> int:
        v = ctypes.c_int32(0)
        check(_lib().sd_comm_nccl_version(ctypes.byref(v)))
        return int(v.value)

    def close(self):
        if self._c:
            check(_lib().sd_comm_destroy(self._c))
            self._c = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def launch_count() -> int:
    """Kernels enqueued by libsparsedrop_b200.so in this process."""
    return int(_lib().sd_launch_count())


def device_count() -> int:
    return int(_lib().sd_device_count())
