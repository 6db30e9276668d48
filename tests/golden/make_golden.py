"""Generate tests/golden/ fixtures by running the UNMODIFIED reference.

Run here (where /root/reference exists) after `make -C oracle ref`:
    python tests/golden/make_golden.py
The fixtures are committed; nothing at test time reads /root/reference.

Contents
  hashes.json   mix64 / counter_hash / effective_seed / dropout_scale KATs
  masks.json    sample_mask words + keep counts for every config geometry of
                BASELINE.json (full words for small grids, sha256 of the
                little-endian words for big ones), kept_blocks_in_row lists,
                transpose_mask and retile words on small grids
  layer_256.npz reference forward + backward (sparsedrop variant, T=double) on
                bf16-rounded random_matrix inputs, M=K=N=256, 128x128 blocks
  gemm_ref32.npz reference dsd / sdd in float with 32-tiles at 128^3 (the
                reference's own test_gemm.cpp:82-90, 130-138 configuration)
"""
from __future__ import annotations

import hashlib
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
from oracle.oracle import Oracle, Reference  # noqa: E402

OUT = Path(__file__).resolve().parent


def words_sha(words: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(words, dtype="<u8").tobytes()).hexdigest()


def main():
    ref = Reference()
    orc = Oracle()

    # ---- hashes
    hashes = {
        "mix64": [[z, ref.L.sdref_mix64(z)] for z in [0, 1, 42, 2**63, 2**64 - 1]],
        "counter_hash": [[s, a, b, ref.counter_hash(s, a, b)]
                         for s, a, b in [(0, 0, 0), (42, 1, 2), (1, 7, 9), (2**64 - 1, 3, 4), (123, 4095, 63)]],
        "effective_seed": [[s, st, li, int(ref.L.sdref_effective_seed(s, st, li))]
                           for s, st, li in [(0, 0, 0), (0, 0, 1), (5, 3, 2), (0, 17, 1)]],
        "dropout_scale_f32": [[p, float(ref.L.sdref_dropout_scale_f32(p))] for p in [0.0, 0.1, 0.3, 0.5, 0.9]],
    }
    (OUT / "hashes.json").write_text(json.dumps(hashes, indent=1))

    # ---- masks
    cases = []
    eff0 = int(ref.L.sdref_effective_seed(0, 0, 0))
    eff1 = int(ref.L.sdref_effective_seed(0, 0, 1))
    geoms = [
        ("cfg1", 1024, 1024, 128, 128, 0, [0.5]),
        ("cfg2", 4096, 4096, 128, 128, 0, [round(0.1 * i, 1) for i in range(10)]),
        ("cfg3_fc1", 65536, 768, 128, 128, eff0, [0.1, 0.3, 0.5]),
        ("cfg3_fc2", 65536, 3072, 128, 128, eff1, [0.1, 0.3, 0.5]),
        ("cfg4", 65536, 8192, 128, 128, 0, [0.1, 0.3, 0.5]),
        ("cfg5", 524288, 8192, 128, 128, 0, [0.1, 0.3, 0.5]),
        ("T8", 8192, 8192, 128, 128, 0, [0.0, 0.1, 0.5]),
        ("seed1", 1024, 1024, 128, 128, 1, [0.5]),
        ("seed42", 1024, 1024, 128, 128, 42, [0.5]),
        ("ragged", 128 * 37, 128 * 19, 128, 128, 3, [0.9]),
        ("blk256", 2048, 2048, 256, 256, 11, [0.4]),
        ("small_odd", 12, 10, 3, 2, 77, [0.35]),
        ("ref_test_16x32", 16, 32, 4, 4, 123, [0.0]),
    ]
    for name, rows, cols, mb, kb, seed, ps in geoms:
        for p in ps:
            w, keep = ref.sample_mask(p, mb, kb, seed, rows, cols)
            R, C = rows // mb, cols // kb
            c = {"name": name, "p": p, "m_blk": mb, "k_blk": kb, "seed": seed, "rows": rows, "cols": cols,
                 "block_rows": R, "block_cols": C, "keep_count": keep, "sha256": words_sha(w)}
            if len(w) <= 1024:
                c["words"] = [hex(int(x)) for x in w]
            if R * C <= 4096:
                c["row_lists"] = [ref.kept_blocks_in_row(w, R, C, mb, kb, r) for r in range(R)]
                wt = ref.transpose_mask(w, R, C, mb, kb)
                c["transpose_words"] = [hex(int(x)) for x in wt]
            cases.append(c)
    retiles = []
    for seed in range(4):
        w, _ = ref.sample_mask(0.4, 4, 8, seed, 16, 32)
        for sm, sk in [(1, 1), (2, 1), (1, 2), (2, 4), (4, 8)]:
            rw = ref.retile(w, 4, 4, 4, 8, sm, sk)
            retiles.append({"seed": seed, "p": 0.4, "m_blk": 4, "k_blk": 8, "rows": 16, "cols": 32,
                            "split_m": sm, "split_k": sk, "words": [hex(int(x)) for x in rw]})
    (OUT / "masks.json").write_text(json.dumps({"cases": cases, "retile": retiles}, indent=0))

    # ---- layer fwd+bwd at 256^3 (double), bf16-rounded inputs
    M = K = N = 256
    p = 0.5
    xb = orc.bf16_bits_to_f64(orc.to_bf16_bits(ref.random_matrix(M, K, 1)))
    wb = orc.bf16_bits_to_f64(orc.to_bf16_bits(ref.random_matrix(K, N, 2)))
    dyb = orc.bf16_bits_to_f64(orc.to_bf16_bits(ref.random_matrix(M, N, 3)))
    y, dx, dw, words = ref.layer_fwd_bwd(xb, wb, dyb, p, 128, 128, 128, seed=0, step_seed=7, layer_index=1)
    np.savez_compressed(OUT / "layer_256.npz", y=y.astype(np.float32), dx=dx.astype(np.float32),
                        dw=dw.astype(np.float32), words=words,
                        meta=np.array([M, N, K, 128, 128, 0, 7, 1], dtype=np.int64), p=np.array([p]))

    # ---- reference-tile (32) dsd / sdd in float, 128^3, p=0.5 (test_gemm.cpp:82-90, 130-138)
    a = ref.random_matrix(128, 128, 11)
    b = ref.random_matrix(128, 128, 12)
    wm, _ = ref.sample_mask(0.5, 32, 32, 5, 128, 128)
    dsd, dsd_cnt = ref.dsd_matmul(a, wm, b, 32, 32, 32, 2.0, dtype=np.float32)
    sdd, sdd_cnt = ref.sdd_matmul(a, b, wm, 32, 32, 32, 1.5, dtype=np.float32)
    np.savez_compressed(OUT / "gemm_ref32.npz", dsd=dsd, sdd=sdd, words=wm, dsd_cnt=dsd_cnt, sdd_cnt=sdd_cnt)
    # ---- BMSK bytes written by the reference (block_mask.cpp:137-219)
    bm = []
    for seed, (p, mb, kb, rows, cols) in enumerate([(0.5, 128, 128, 1024, 1024), (0.4, 2, 3, 12, 12),
                                                   (0.3, 128, 128, 128 * 13, 128 * 70), (0.9, 1, 1, 5, 7),
                                                   (0.0, 4, 8, 16, 32)]):
        w, _ = ref.sample_mask(p, mb, kb, seed, rows, cols)
        R, C = rows // mb, cols // kb
        bm.append({"geom": [R, C, mb, kb], "words": [hex(int(x)) for x in w],
                   "bytes": ref.write_mask(w, R, C, mb, kb).hex()})
    (OUT / "bmsk.json").write_text(json.dumps(bm, indent=0))

    # ---- dropout_dense variant (element mask) forward/backward, double (layer.hpp:69-76,105-111,148-156)
    M2, K2, N2 = 256, 256, 128
    x2 = orc.bf16_bits_to_f64(orc.to_bf16_bits(ref.random_matrix(M2, K2, 1)))
    w2 = orc.bf16_bits_to_f64(orc.to_bf16_bits(ref.random_matrix(K2, N2, 2)))
    dy2 = orc.bf16_bits_to_f64(orc.to_bf16_bits(ref.random_matrix(M2, N2, 3)))
    y2, dx2, dw2 = ref.dropout_dense_fwd_bwd(x2, w2, dy2, 0.3, seed=11, step_seed=2, layer_index=0)
    np.savez_compressed(OUT / "dropout_dense_256.npz", y=y2.astype(np.float32), dx=dx2.astype(np.float32),
                        dw=dw2.astype(np.float32), meta=np.array([M2, N2, K2, 11, 2, 0], dtype=np.int64),
                        p=np.array([0.3]))
    print("golden fixtures written to", OUT)


if __name__ == "__main__":
    main()
