"""ctypes bindings for the oracle — TEST INFRASTRUCTURE ONLY.

  liboracle : oracle/libsdoracle.so, the C restatement (oracle/sd_oracle.c)
  libref    : oracle/_ref/libsdref.so, the UNMODIFIED reference compiled from
              /root/reference by oracle/Makefile (present only when built)

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs import
this module. The product package paper_2411_01238_b200 never does.
"""
from __future__ import annotations

import ctypes
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ORACLE_LIB = HERE / "libsdoracle.so"
REF_LIB = HERE / "_ref" / "libsdref.so"

_u64 = ctypes.c_uint64
_i32 = ctypes.c_int32
_i64 = ctypes.c_int64
_dbl = ctypes.c_double
_p = ctypes.c_void_p


def _np_ptr(a: np.ndarray | None):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


class Oracle:
    """The C restatement (sd_oracle.c)."""

    def __init__(self, path: Path = ORACLE_LIB):
        if not path.exists():
            raise FileNotFoundError(f"{path}: run `make -C oracle`")
        L = ctypes.CDLL(str(path))
        self.L = L
        L.sdo_mix64.restype = _u64
        L.sdo_mix64.argtypes = [_u64]
        L.sdo_counter_hash.restype = _u64
        L.sdo_counter_hash.argtypes = [_u64, _u64, _u64]
        L.sdo_effective_seed.restype = _u64
        L.sdo_effective_seed.argtypes = [_u64, _u64, ctypes.c_int]
        L.sdo_keep_threshold.restype = _u64
        L.sdo_keep_threshold.argtypes = [_dbl]
        L.sdo_last_error.restype = ctypes.c_char_p
        L.sdo_sample_mask.argtypes = [_dbl, ctypes.c_int, ctypes.c_int, _u64, ctypes.c_int, ctypes.c_int,
                                      ctypes.c_int, _p, _p]
        L.sdo_mask_from_words.argtypes = [ctypes.c_int, ctypes.c_int, _p, _i64, _p]
        L.sdo_kept_blocks_in_row.argtypes = [_p, ctypes.c_int, ctypes.c_int, ctypes.c_int, _p, _p]
        L.sdo_transpose_mask.argtypes = [_p, ctypes.c_int, ctypes.c_int, _p]
        L.sdo_retile.argtypes = [_p] + [ctypes.c_int] * 6 + [_p]
        L.sdo_random_matrix_f32.argtypes = [ctypes.c_int, ctypes.c_int, _u64, _p]
        L.sdo_f32_to_bf16.argtypes = [_p, _p, _i64]
        L.sdo_bf16_to_f64.argtypes = [_p, _p, _i64]
        L.sdo_dsd_matmul_f64.argtypes = [_p, _p, _p] + [ctypes.c_int] * 6 + [_dbl] + [ctypes.c_int] * 3 + [_p, _p]
        L.sdo_sdd_matmul_f64.argtypes = [_p, _p, _p] + [ctypes.c_int] * 5 + [_dbl] + [ctypes.c_int] * 3 + [_p]
        L.sdo_layer_dx_f64.argtypes = [_p, _p, _p] + [ctypes.c_int] * 5 + [_dbl] + [ctypes.c_int] * 3 + [_p]
        L.sdo_layer_dw_f64.argtypes = [_p, _p, _p] + [ctypes.c_int] * 5 + [_dbl] + [ctypes.c_int] * 3 + [_p]
        L.sdo_dense_gemm_f64.argtypes = [_p, _p] + [ctypes.c_int] * 6 + [_p]
        L.sdo_element_mask.argtypes = [_u64, _dbl, ctypes.c_int, ctypes.c_int, _p]
        L.sdo_write_mask.restype = _i64
        L.sdo_write_mask.argtypes = [_p] + [ctypes.c_int] * 4 + [_p]

    def _check(self, rc: int):
        if rc == 0:
            return
        msg = self.L.sdo_last_error().decode()
        raise (ValueError if rc == 1 else IndexError)(msg)

    def counter_hash(self, seed, a, b) -> int:
        return int(self.L.sdo_counter_hash(seed, a, b))

    def mix64(self, z) -> int:
        return int(self.L.sdo_mix64(z))

    def effective_seed(self, seed, step, layer) -> int:
        return int(self.L.sdo_effective_seed(seed, step, layer))

    def keep_threshold(self, p) -> int:
        return int(self.L.sdo_keep_threshold(p))

    def sample_mask(self, p, m_blk, k_blk, seed, rows, cols, row_block_offset=0):
        """-> (words uint64 array, keep_count)."""
        R, C = max(rows // max(m_blk, 1), 0), max(cols // max(k_blk, 1), 0)
        words = np.zeros(max((R * C + 63) // 64, 1), dtype=np.uint64)
        keep = ctypes.c_int64(0)
        self._check(self.L.sdo_sample_mask(p, m_blk, k_blk, seed & (2**64 - 1), rows, cols, row_block_offset,
                                           _np_ptr(words), ctypes.byref(keep)))
        return words[: (R * C + 63) // 64], keep.value

    def kept_blocks_in_row(self, words, R, C, row):
        idx = np.zeros(max(C, 1), dtype=np.int32)
        n = ctypes.c_int32(0)
        self._check(self.L.sdo_kept_blocks_in_row(_np_ptr(np.ascontiguousarray(words, dtype=np.uint64)), R, C,
                                                  row, _np_ptr(idx), ctypes.byref(n)))
        return idx[: n.value].tolist()

    def transpose_mask(self, words, R, C):
        out = np.zeros((R * C + 63) // 64, dtype=np.uint64)
        self.L.sdo_transpose_mask(_np_ptr(np.ascontiguousarray(words, dtype=np.uint64)), R, C, _np_ptr(out))
        return out

    def retile(self, words, R, C, m_blk, k_blk, sm, sk):
        out = np.zeros((R * sm * C * sk + 63) // 64, dtype=np.uint64)
        self._check(self.L.sdo_retile(_np_ptr(np.ascontiguousarray(words, dtype=np.uint64)), R, C, m_blk, k_blk,
                                      sm, sk, _np_ptr(out)))
        return out

    def random_matrix(self, rows, cols, seed) -> np.ndarray:
        out = np.empty((rows, cols), dtype=np.float32)
        self.L.sdo_random_matrix_f32(rows, cols, seed, _np_ptr(out))
        return out

    def element_mask(self, seed, p, rows, cols) -> np.ndarray:
        out = np.empty((rows, cols), dtype=np.uint8)
        self.L.sdo_element_mask(seed & (2**64 - 1), p, rows, cols, _np_ptr(out))
        return out

    def write_mask(self, words, R, C, m_blk, k_blk) -> bytes:
        buf = np.zeros(21 + 8 * ((R * C + 63) // 64), dtype=np.uint8)
        n = self.L.sdo_write_mask(_np_ptr(np.ascontiguousarray(words, dtype=np.uint64)), R, C, m_blk, k_blk,
                                  _np_ptr(buf))
        return bytes(buf[:n])

    def to_bf16_bits(self, a: np.ndarray) -> np.ndarray:
        a = np.ascontiguousarray(a, dtype=np.float32)
        out = np.empty(a.shape, dtype=np.uint16)
        self.L.sdo_f32_to_bf16(_np_ptr(a), _np_ptr(out), a.size)
        return out

    def bf16_bits_to_f64(self, b: np.ndarray) -> np.ndarray:
        b = np.ascontiguousarray(b, dtype=np.uint16)
        out = np.empty(b.shape, dtype=np.float64)
        self.L.sdo_bf16_to_f64(_np_ptr(b), _np_ptr(out), b.size)
        return out

    def dsd_matmul(self, a, words, b, m_blk, n_blk, k_blk, scale, row_lo=0, row_hi=None, threads=8):
        a = np.ascontiguousarray(a, dtype=np.float64)
        b = np.ascontiguousarray(b, dtype=np.float64)
        m, k = a.shape
        n = b.shape[1]
        row_hi = m if row_hi is None else row_hi
        c = np.empty((row_hi - row_lo, n), dtype=np.float64)
        self._check(self.L.sdo_dsd_matmul_f64(_np_ptr(a), _np_ptr(np.ascontiguousarray(words, dtype=np.uint64)),
                                              _np_ptr(b), m, n, k, m_blk, n_blk, k_blk, scale, row_lo, row_hi,
                                              threads, _np_ptr(c), None))
        return c

    def sdd_matmul(self, a, b, words, m_blk, n_blk, scale, row_lo=0, row_hi=None, threads=8):
        a = np.ascontiguousarray(a, dtype=np.float64)
        b = np.ascontiguousarray(b, dtype=np.float64)
        m, k = a.shape
        n = b.shape[1]
        row_hi = m if row_hi is None else row_hi
        c = np.empty((row_hi - row_lo, n), dtype=np.float64)
        self._check(self.L.sdo_sdd_matmul_f64(_np_ptr(a), _np_ptr(b), _np_ptr(np.ascontiguousarray(words, dtype=np.uint64)),
                                              m, n, k, m_blk, n_blk, scale, row_lo, row_hi, threads, _np_ptr(c)))
        return c

    def layer_dx(self, dy, w, words, m_blk, k_blk, scale, row_lo=0, row_hi=None, threads=8):
        dy = np.ascontiguousarray(dy, dtype=np.float64)
        w = np.ascontiguousarray(w, dtype=np.float64)
        m, n = dy.shape
        k = w.shape[0]
        row_hi = m if row_hi is None else row_hi
        dx = np.empty((row_hi - row_lo, k), dtype=np.float64)
        self._check(self.L.sdo_layer_dx_f64(_np_ptr(dy), _np_ptr(w), _np_ptr(np.ascontiguousarray(words, dtype=np.uint64)),
                                            m, n, k, m_blk, k_blk, scale, row_lo, row_hi, threads, _np_ptr(dx)))
        return dx

    def layer_dw(self, x, dy, words, m_blk, k_blk, scale, krow_lo=0, krow_hi=None, threads=8):
        x = np.ascontiguousarray(x, dtype=np.float64)
        dy = np.ascontiguousarray(dy, dtype=np.float64)
        m, k = x.shape
        n = dy.shape[1]
        krow_hi = k if krow_hi is None else krow_hi
        dw = np.empty((krow_hi - krow_lo, n), dtype=np.float64)
        self._check(self.L.sdo_layer_dw_f64(_np_ptr(x), _np_ptr(dy), _np_ptr(np.ascontiguousarray(words, dtype=np.uint64)),
                                            m, n, k, m_blk, k_blk, scale, krow_lo, krow_hi, threads, _np_ptr(dw)))
        return dw

    def dense_gemm(self, a, b, row_lo=0, row_hi=None, threads=8):
        a = np.ascontiguousarray(a, dtype=np.float64)
        b = np.ascontiguousarray(b, dtype=np.float64)
        m, k = a.shape
        n = b.shape[1]
        row_hi = m if row_hi is None else row_hi
        c = np.empty((row_hi - row_lo, n), dtype=np.float64)
        self._check(self.L.sdo_dense_gemm_f64(_np_ptr(a), _np_ptr(b), m, n, k, row_lo, row_hi, threads, _np_ptr(c)))
        return c


class Reference:
    """The unmodified reference (oracle/_ref/libsdref.so)."""

    def __init__(self, path: Path = REF_LIB):
        if not path.exists():
            raise FileNotFoundError(f"{path}: run `make -C oracle ref` (needs /root/reference)")
        L = ctypes.CDLL(str(path))
        self.L = L
        L.sdref_last_error.restype = ctypes.c_char_p
        L.sdref_mix64.restype = _u64
        L.sdref_mix64.argtypes = [_u64]
        L.sdref_counter_hash.restype = _u64
        L.sdref_counter_hash.argtypes = [_u64, _u64, _u64]
        L.sdref_effective_seed.restype = _u64
        L.sdref_effective_seed.argtypes = [_u64, _u64, ctypes.c_int]
        L.sdref_dropout_scale_f32.restype = ctypes.c_float
        L.sdref_dropout_scale_f32.argtypes = [_dbl]
        L.sdref_sample_mask.argtypes = [_dbl, ctypes.c_int, ctypes.c_int, _u64, ctypes.c_int, ctypes.c_int, _p,
                                        _i64, _p]
        L.sdref_kept_blocks_in_row.argtypes = [_p] + [ctypes.c_int] * 5 + [_p, _p]
        L.sdref_transpose_mask.argtypes = [_p] + [ctypes.c_int] * 4 + [_p]
        L.sdref_retile.argtypes = [_p] + [ctypes.c_int] * 6 + [_p]
        L.sdref_random_matrix_f32.argtypes = [ctypes.c_int, ctypes.c_int, _u64, _p]
        for t, ct in (("f32", ctypes.c_float), ("f64", ctypes.c_double)):
            getattr(L, f"sdref_dense_gemm_{t}").argtypes = [_p, _p] + [ctypes.c_int] * 7 + [_p]
            getattr(L, f"sdref_dsd_matmul_{t}").argtypes = [_p, _p, _p] + [ctypes.c_int] * 6 + [ct, ctypes.c_int, _p, _p]
            getattr(L, f"sdref_sdd_matmul_{t}").argtypes = [_p, _p, _p] + [ctypes.c_int] * 6 + [ct, ctypes.c_int, _p, _p]
            getattr(L, f"sdref_layer_fwd_bwd_{t}").argtypes = ([_p, _p, _p] + [ctypes.c_int] * 3 + [_dbl] +
                                                               [ctypes.c_int] * 3 + [_u64, _u64, ctypes.c_int,
                                                                                     ctypes.c_int, _p, _p, _p, _p])

    def _check(self, rc):
        if rc == 0:
            return
        msg = self.L.sdref_last_error().decode()
        raise {1: ValueError, 2: IndexError}.get(rc, RuntimeError)(msg)

    def counter_hash(self, seed, a, b):
        return int(self.L.sdref_counter_hash(seed, a, b))

    def write_mask(self, words, R, C, m_blk, k_blk) -> bytes:
        self.L.sdref_write_mask.argtypes = [_p] + [ctypes.c_int] * 4 + [_p, _i64, _p]
        buf = np.zeros(64 + 8 * ((R * C + 63) // 64), dtype=np.uint8)
        n = ctypes.c_int64(0)
        self._check(self.L.sdref_write_mask(_np_ptr(np.ascontiguousarray(words, dtype=np.uint64)), R, C, m_blk,
                                            k_blk, _np_ptr(buf), len(buf), ctypes.byref(n)))
        return bytes(buf[: n.value])

    def read_mask(self, data: bytes):
        self.L.sdref_read_mask.argtypes = [_p, _i64, _p, _p, _i64]
        arr = np.frombuffer(data, dtype=np.uint8).copy()
        geom = np.zeros(4, dtype=np.int32)
        words = np.zeros(max(len(data) // 8 + 1, 1), dtype=np.uint64)
        self._check(self.L.sdref_read_mask(_np_ptr(arr), len(arr), _np_ptr(geom), _np_ptr(words), len(words)))
        R, C = int(geom[0]), int(geom[1])
        return (R, C, int(geom[2]), int(geom[3])), words[: (R * C + 63) // 64].copy()

    def dropout_dense_fwd_bwd(self, x, w, dy, p, seed, step_seed, layer_index, threads=8):
        L = self.L
        L.sdref_dropout_dense_fwd_bwd_f64.argtypes = [_p, _p, _p] + [ctypes.c_int] * 3 + [_dbl, _u64, _u64,
                                                                                            ctypes.c_int, ctypes.c_int,
                                                                                            _p, _p, _p]
        x = np.ascontiguousarray(x, dtype=np.float64)
        w = np.ascontiguousarray(w, dtype=np.float64)
        dy = np.ascontiguousarray(dy, dtype=np.float64)
        m, k = x.shape
        n = w.shape[1]
        y, dx, dw = np.empty((m, n)), np.empty((m, k)), np.empty((k, n))
        self._check(L.sdref_dropout_dense_fwd_bwd_f64(_np_ptr(x), _np_ptr(w), _np_ptr(dy), m, n, k, p,
                                                      seed & (2**64 - 1), step_seed & (2**64 - 1), layer_index,
                                                      threads, _np_ptr(y), _np_ptr(dx), _np_ptr(dw)))
        return y, dx, dw

    def sample_mask(self, p, m_blk, k_blk, seed, rows, cols):
        cap = max(rows * cols, 64)
        words = np.zeros(cap // 64 + 1, dtype=np.uint64)
        keep = ctypes.c_int64(0)
        self._check(self.L.sdref_sample_mask(p, m_blk, k_blk, seed & (2**64 - 1), rows, cols, _np_ptr(words),
                                             len(words), ctypes.byref(keep)))
        R, C = rows // m_blk, cols // k_blk
        return words[: (R * C + 63) // 64].copy(), keep.value

    def kept_blocks_in_row(self, words, R, C, m_blk, k_blk, row):
        idx = np.zeros(max(C, 1), dtype=np.int32)
        n = ctypes.c_int32(0)
        self._check(self.L.sdref_kept_blocks_in_row(_np_ptr(np.ascontiguousarray(words, dtype=np.uint64)), R, C,
                                                    m_blk, k_blk, row, _np_ptr(idx), ctypes.byref(n)))
        return idx[: n.value].tolist()

    def transpose_mask(self, words, R, C, m_blk, k_blk):
        out = np.zeros((R * C + 63) // 64, dtype=np.uint64)
        self._check(self.L.sdref_transpose_mask(_np_ptr(np.ascontiguousarray(words, dtype=np.uint64)), R, C,
                                                m_blk, k_blk, _np_ptr(out)))
        return out

    def retile(self, words, R, C, m_blk, k_blk, sm, sk):
        out = np.zeros((R * sm * C * sk + 63) // 64, dtype=np.uint64)
        self._check(self.L.sdref_retile(_np_ptr(np.ascontiguousarray(words, dtype=np.uint64)), R, C, m_blk, k_blk,
                                        sm, sk, _np_ptr(out)))
        return out

    def random_matrix(self, rows, cols, seed):
        out = np.empty((rows, cols), dtype=np.float32)
        self.L.sdref_random_matrix_f32(rows, cols, seed, _np_ptr(out))
        return out

    def dsd_matmul(self, a, words, b, m_blk, n_blk, k_blk, scale, threads=8, dtype=np.float64):
        t = "f64" if dtype == np.float64 else "f32"
        a = np.ascontiguousarray(a, dtype=dtype)
        b = np.ascontiguousarray(b, dtype=dtype)
        m, k = a.shape
        n = b.shape[1]
        c = np.empty((m, n), dtype=dtype)
        cnt = np.zeros(m // m_blk, dtype=np.uint64)
        self._check(getattr(self.L, f"sdref_dsd_matmul_{t}")(
            _np_ptr(a), _np_ptr(np.ascontiguousarray(words, dtype=np.uint64)), _np_ptr(b), m, n, k, m_blk, n_blk,
            k_blk, scale, threads, _np_ptr(c), _np_ptr(cnt)))
        return c, cnt

    def sdd_matmul(self, a, b, words, m_blk, n_blk, k_blk, scale, threads=8, dtype=np.float64):
        t = "f64" if dtype == np.float64 else "f32"
        a = np.ascontiguousarray(a, dtype=dtype)
        b = np.ascontiguousarray(b, dtype=dtype)
        m, k = a.shape
        n = b.shape[1]
        c = np.empty((m, n), dtype=dtype)
        cnt = np.zeros(m // m_blk, dtype=np.uint64)
        self._check(getattr(self.L, f"sdref_sdd_matmul_{t}")(
            _np_ptr(a), _np_ptr(b), _np_ptr(np.ascontiguousarray(words, dtype=np.uint64)), m, n, k, m_blk, n_blk,
            k_blk, scale, threads, _np_ptr(c), _np_ptr(cnt)))
        return c, cnt

    def dense_gemm(self, a, b, m_blk, n_blk, k_blk, threads=8, dtype=np.float64):
        t = "f64" if dtype == np.float64 else "f32"
        a = np.ascontiguousarray(a, dtype=dtype)
        b = np.ascontiguousarray(b, dtype=dtype)
        m, k = a.shape
        n = b.shape[1]
        c = np.empty((m, n), dtype=dtype)
        self._check(getattr(self.L, f"sdref_dense_gemm_{t}")(_np_ptr(a), _np_ptr(b), m, n, k, m_blk, n_blk, k_blk,
                                                             threads, _np_ptr(c)))
        return c

    def layer_fwd_bwd(self, x, w, dy, p, m_blk, k_blk, n_blk, seed, step_seed, layer_index, threads=8,
                      dtype=np.float64, want_y=True, want_dx=True, want_dw=True):
        t = "f64" if dtype == np.float64 else "f32"
        x = np.ascontiguousarray(x, dtype=dtype)
        w = np.ascontiguousarray(w, dtype=dtype)
        dy = np.ascontiguousarray(dy, dtype=dtype)
        m, k = x.shape
        n = w.shape[1]
        y = np.empty((m, n), dtype=dtype) if want_y else None
        dx = np.empty((m, k), dtype=dtype) if want_dx else None
        dw = np.empty((k, n), dtype=dtype) if want_dw else None
        words = np.zeros(((m // m_blk) * (k // k_blk) + 63) // 64, dtype=np.uint64)
        self._check(getattr(self.L, f"sdref_layer_fwd_bwd_{t}")(
            _np_ptr(x), _np_ptr(w), _np_ptr(dy), m, n, k, p, m_blk, k_blk, n_blk, seed & (2**64 - 1),
            step_seed & (2**64 - 1), layer_index, threads, _np_ptr(y), _np_ptr(dx), _np_ptr(dw), _np_ptr(words)))
        return y, dx, dw, words


def oracle() -> Oracle:
    return Oracle()


def reference() -> Reference | None:
    try:
        return Reference()
    except FileNotFoundError:
        return None
