"""BMSK mask container: save / load / replay device masks.

Byte-compatible with the reference (block_mask.cpp:137-219, block_mask.hpp:113-119):
"BMSK", version 0x01, little-endian u32 block_rows, block_cols, m_blk, k_blk,
then the mask words as little-endian u64. Reading validates magic, version,
truncation, positive geometry and zero padding bits; every failure is a
RuntimeError (std::runtime_error in the reference), prefixed by `name`.
A mask read back is re-compacted on the device (sd_mask_compact), so it can
drive the GEMMs directly (e.g. replaying a recorded training mask).
"""
from __future__ import annotations

import io
import struct
from typing import BinaryIO

from .api import BlockMask, mask_from_words

MAGIC = b"BMSK"
VERSION = 0x01


def write_mask(mask: BlockMask, out: BinaryIO) -> None:
    """block_mask.cpp:170-178."""
    out.write(MAGIC)
    out.write(bytes([VERSION]))
    out.write(struct.pack("<4I", mask.block_rows(), mask.block_cols(), mask.m_blk(), mask.k_blk()))
    out.write(struct.pack(f"<{mask.n_words()}Q", *mask.words()))


def to_bytes(mask: BlockMask) -> bytes:
    buf = io.BytesIO()
    write_mask(mask, buf)
    return buf.getvalue()


def _read_exact(inp: BinaryIO, n: int, name: str, what: str) -> bytes:
    b = inp.read(n)
    if b is None or len(b) != n:
        raise RuntimeError(f"{name}: truncated BMSK {what}")
    return b


def read_mask(inp: BinaryIO, name: str, stream=None) -> BlockMask:
    """block_mask.cpp:180-205."""
    magic = inp.read(4)
    if magic != MAGIC:
        raise RuntimeError(f"{name}: not a BMSK file (bad magic)")
    v = inp.read(1)
    version = v[0] if v else -1
    if version != VERSION:
        raise RuntimeError(f"{name}: unsupported BMSK version {version}")
    block_rows, block_cols, m_blk, k_blk = struct.unpack("<4I", _read_exact(inp, 16, name, "header"))
    if not all(0 < x < 2**31 for x in (block_rows, block_cols, m_blk, k_blk)):
        raise RuntimeError(f"{name}: BMSK header has non-positive geometry")
    n_words = (block_rows * block_cols + 63) // 64
    words = list(struct.unpack(f"<{n_words}Q", _read_exact(inp, 8 * n_words, name, "payload")))
    try:
        return mask_from_words(block_rows, block_cols, m_blk, k_blk, words, stream=stream)
    except ValueError as e:
        raise RuntimeError(f"{name}: {e}") from None


def from_bytes(data: bytes, name: str = "buffer", stream=None) -> BlockMask:
    return read_mask(io.BytesIO(data), name, stream)


def save_mask(mask: BlockMask, path: str) -> None:
    """block_mask.cpp:207-212."""
    try:
        with open(path, "wb") as f:
            write_mask(mask, f)
    except OSError as e:
        raise RuntimeError(f"cannot open {path} for writing") from e


def load_mask(path: str, stream=None) -> BlockMask:
    """block_mask.cpp:214-218."""
    try:
        f = open(path, "rb")
    except OSError as e:
        raise RuntimeError(f"cannot open {path}") from e
    with f:
        return read_mask(f, path, stream)
