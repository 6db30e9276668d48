"""CPU: the C-ABI library loads, exports every symbol include/sparsedrop_b200.h
declares, validates arguments with the reference's error classes/messages, and
refuses to compute without a B200 (no CPU fallback)."""
import ctypes
import re

import pytest

from paper_2411_01238_b200 import _capi


@pytest.fixture(scope="module")
def lib():
    return _capi.load()


def _header_symbols():
    text = _capi.HEADER_PATH.read_text()
    return re.findall(r"SD_API\s+[\w\s\*]+?\b(sd_\w+)\s*\(", text)


def test_header_declares_api():
    syms = _header_symbols()
    assert len(syms) >= 18
    assert "sd_mask_sample" in syms and "sd_dsd_matmul" in syms and "sd_linear_backward_dw" in syms


def test_library_exports_every_header_symbol(lib):
    missing = [s for s in _header_symbols() if not hasattr(lib, s)]
    assert not missing, missing
    # and the Python binding declares a prototype for each
    assert set(_header_symbols()) <= set(_capi.PROTOTYPES)


def test_abi_version(lib):
    assert lib.sd_abi_version() == 1


def _has_gpu():
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


def _err(lib):
    return lib.sd_last_error().decode()


def test_gemm_shape_validation(lib):
    null = ctypes.c_void_p(16)  # never dereferenced: validation runs first
    rc = lib.sd_dense_gemm(null, null, null, 1, 100, 256, 128, None)
    assert rc == _capi.SD_EINVAL and "m_blk" in _err(lib) and "does not divide" in _err(lib)
    rc = lib.sd_dense_gemm(null, null, null, 1, 128, 200, 128, None)
    assert rc == _capi.SD_EINVAL and "n_blk" in _err(lib)
    rc = lib.sd_dense_gemm(null, null, null, 1, 128, 256, 100, None)
    assert rc == _capi.SD_EINVAL and "k_blk" in _err(lib)
    rc = lib.sd_dense_gemm(null, null, null, 7, 128, 256, 128, None)
    assert rc == _capi.SD_EINVAL and "dtype" in _err(lib)


def test_mask_validation(lib):
    m = _capi.SdBlockMask()
    ws = ctypes.create_string_buffer(lib.sd_mask_workspace_bytes(8, 8) + 256)
    base = (ctypes.addressof(ws) + 255) & ~255
    assert lib.sd_mask_bind(ctypes.byref(m), ctypes.c_void_p(base), 8, 8, 128, 128, 0) == 0
    assert m.block_rows == 8 and m.k_blk == 128
    assert lib.sd_mask_sample(ctypes.byref(m), 0, 1.0, 1024, 1024, None) == _capi.SD_EINVAL
    assert "dropout rate" in _err(lib)
    assert lib.sd_mask_sample(ctypes.byref(m), 0, -0.1, 1024, 1024, None) == _capi.SD_EINVAL
    assert lib.sd_mask_sample(ctypes.byref(m), 0, 0.5, 1000, 1024, None) == _capi.SD_EINVAL
    assert "m_blk" in _err(lib)
    assert lib.sd_mask_sample(ctypes.byref(m), 0, 0.5, 1024, 1000, None) == _capi.SD_EINVAL
    assert "k_blk" in _err(lib)
    assert lib.sd_mask_bind(ctypes.byref(m), ctypes.c_void_p(base), 0, 8, 128, 128, 0) == _capi.SD_EINVAL
    assert "geometry" in _err(lib)


def test_mask_geometry_mismatch(lib):
    m = _capi.SdBlockMask()
    ws = ctypes.create_string_buffer(lib.sd_mask_workspace_bytes(8, 8) + 256)
    base = (ctypes.addressof(ws) + 255) & ~255
    lib.sd_mask_bind(ctypes.byref(m), ctypes.c_void_p(base), 8, 8, 128, 128, 0)
    p = ctypes.c_void_p(16)
    rc = lib.sd_dsd_matmul(p, ctypes.byref(m), p, 1.0, p, 1, 2048, 256, 1024, None, None)
    assert rc == _capi.SD_EINVAL and "mask geometry" in _err(lib)
    rc = lib.sd_sdd_matmul(p, p, ctypes.byref(m), 1.0, p, 1, 1024, 512, 1024, None, None)
    assert rc == _capi.SD_EINVAL and "mask geometry" in _err(lib)


def test_unsupported_block_sizes_rejected(lib):
    m = _capi.SdBlockMask()
    ws = ctypes.create_string_buffer(lib.sd_mask_workspace_bytes(32, 32) + 256)
    base = (ctypes.addressof(ws) + 255) & ~255
    lib.sd_mask_bind(ctypes.byref(m), ctypes.c_void_p(base), 32, 32, 32, 32, 0)
    p = ctypes.c_void_p(16)
    rc = lib.sd_dsd_matmul(p, ctypes.byref(m), p, 1.0, p, 1, 1024, 256, 1024, None, None)
    assert rc == _capi.SD_EINVAL and "m_blk" in _err(lib)


@pytest.mark.skipif(_has_gpu(), reason="checks the no-GPU behaviour")
def test_no_cpu_fallback(lib):
    assert lib.sd_device_count() == 0
    p = ctypes.c_void_p(16)
    rc = lib.sd_dense_gemm(p, p, p, 1, 128, 256, 128, None)
    assert rc == _capi.SD_ERUNTIME and "no CPU fallback" in _err(lib)
    with pytest.raises(RuntimeError):
        _capi.check(rc)


def test_status_mapping():
    lib = _capi.load()
    p = ctypes.c_void_p(16)
    rc = lib.sd_dense_gemm(p, p, p, 1, 100, 256, 128, None)
    with pytest.raises(ValueError, match="m_blk"):
        _capi.check(rc)


def test_flops(lib):
    assert lib.sd_flops_dense(1024, 1024, 1024) == 2 * 1024**3
    # gemm.hpp:222-228
    assert lib.sd_flops_effective(1024, 1024, 128, 128, 128, 25, 0) == 2 * 1024 * 128 * 128 * 25
    assert lib.sd_flops_effective(1024, 512, 128, 128, 128, 25, 1) == 2 * 512 * 128 * 128 * 25


def test_nccl_communicator_without_gpu(lib):
    """The data-parallel backward's NCCL layer (sd_comm_*): NCCL resolves at run
    time, a unique id can be made without a GPU, and creating a communicator
    without a B200 fails loudly (no CPU fallback)."""
    import paper_2411_01238_b200 as sd

    v = sd.Communicator.nccl_version()
    assert v >= 22700, v  # NCCL >= 2.27
    uid = sd.Communicator.new_unique_id()
    assert len(uid) == 128 and uid != bytes(128)
    if not _has_gpu():
        with pytest.raises(RuntimeError):
            sd.Communicator(1, 0, uid)
    with pytest.raises(IndexError):
        sd.Communicator(2, 2, uid)
    assert lib.sd_layer_plan_backward_allreduce(None, None, 2, None, None) == _capi.SD_EINVAL
