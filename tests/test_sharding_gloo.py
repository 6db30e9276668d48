"""CPU, world_size 2 (gloo): the row-sharded data-parallel logic of SURVEY §8e.

Each rank takes its contiguous block rows (paper_2411_01238_b200.sharding),
generates its mask rows locally from the GLOBAL block-row index, computes its
partial dW, and the partials are summed with an all-reduce; the result must
equal the unsharded dW, and the shard masks must equal the global mask rows.
(The oracle stands in for the device kernels here; the GPU path of the same
logic is tests/test_gpu_parity.py::test_dw_linearity_in_row_shards.)
"""
import os
import socket
import sys
from pathlib import Path

import numpy as np
import pytest

from paper_2411_01238_b200.sharding import all_shards, shard_rows

ROOT = Path(__file__).resolve().parents[1]


def test_shard_rows_partition():
    for m, world in [(4096, 2), (4096, 8), (128 * 37, 4), (65536, 8), (524288, 8)]:
        shards = all_shards(m, 128, world)
        assert shards[0].row0 == 0
        for a, b in zip(shards, shards[1:]):
            assert a.row0 + a.rows == b.row0
        assert sum(s.rows for s in shards) == m
        assert all(s.row_block_offset * 128 == s.row0 for s in shards)
        assert max(s.rows for s in shards) - min(s.rows for s in shards) <= 128
    with pytest.raises(ValueError):
        shard_rows(1000, 128, 2, 0)
    with pytest.raises(ValueError):
        shard_rows(256, 128, 4, 0)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, result_path):
    sys.path.insert(0, str(ROOT))
    import torch
    import torch.distributed as dist

    from oracle.oracle import Oracle

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    o = Oracle()
    M, N, K, p, seed = 1024, 256, 512, 0.5, 17
    x = o.random_matrix(M, K, 1).astype(np.float64)
    dy = o.random_matrix(M, N, 3).astype(np.float64)
    sh = shard_rows(M, 128, world, rank)
    xs, dys = x[sh.row0:sh.row0 + sh.rows], dy[sh.row0:sh.row0 + sh.rows]
    words, _ = o.sample_mask(p, 128, 128, seed, sh.rows, K, row_block_offset=sh.row_block_offset)
    s = 1.0 / (1.0 - p)
    dw = torch.from_numpy(o.layer_dw(xs, dys, words, 128, 128, s, threads=2))
    dist.all_reduce(dw)
    # gather the shard masks (as bits, row-major: local packing differs from the
    # global words when C is not a multiple of 64) to rank 0
    nb = (sh.rows // 128) * (K // 128)
    bits = np.array([(int(words[b >> 6]) >> (b & 63)) & 1 for b in range(nb)], dtype=np.int64)
    wt = torch.from_numpy(bits)
    gathered = [torch.zeros_like(wt) for _ in range(world)] if rank == 0 else None
    dist.gather(wt, gathered, dst=0)
    if rank == 0:
        gw, _ = o.sample_mask(p, 128, 128, seed, M, K)
        full = o.layer_dw(x, dy, gw, 128, 128, s, threads=2)
        ok_dw = float(np.abs(dw.numpy() - full).max() / np.abs(full).max())
        cat = np.concatenate([g.numpy() for g in gathered])
        gbits = np.array([(int(gw[b >> 6]) >> (b & 63)) & 1 for b in range(len(cat))], dtype=np.int64)
        ok_mask = bool(np.array_equal(cat, gbits)) and len(cat) == (M // 128) * (K // 128)
        Path(result_path).write_text(f"{ok_dw} {int(ok_mask)}")
    dist.destroy_process_group()


def test_row_sharded_dw_allreduce_gloo(tmp_path):
    import torch.multiprocessing as mp

    out = tmp_path / "result.txt"
    mp.start_processes(_worker, args=(2, _free_port(), str(out)), nprocs=2, join=True, start_method="spawn")
    err, mask_ok = out.read_text().split()
    assert float(err) < 1e-12
    assert mask_ok == "1"
