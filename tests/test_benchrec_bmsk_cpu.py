"""CPU: the bench CSV schema and the BMSK container's
host-side validation (block_mask.cpp:137-219), pinned to reference bytes."""
import io
import json
from pathlib import Path

import pytest

from paper_2411_01238_b200.benchrec import HEADER, BenchRecord, parse_csv, percentile_record, to_csv

GOLDEN = Path(__file__).resolve().parent / "golden"


def test_csv_header_exact_and_empty():
    assert to_csv([]) == ",".join(HEADER) + "\n"
    assert ",".join(HEADER) == ("method,m,n,k,sparsity,realized_sparsity,pass,nanos_median,nanos_p10,nanos_p90,"
                                "effective_gflops,repeats")


def test_csv_one_record_and_roundtrip():
    r = percentile_record("sparsedrop", 1024, 1024, 1024, 0.5, 0.609375, "total", [900.0, 1000.0, 1100.0, 1050.0],
                          3.2e12)
    text = to_csv([r])
    lines = text.split("\n")
    assert len(lines) == 3 and lines[2] == ""  # two lines + trailing LF
    assert len(lines[1].split(",")) == 12
    assert parse_csv(text) == [r]
    assert r.nanos_p10 <= r.nanos_median <= r.nanos_p90


def test_csv_invariants():
    with pytest.raises(ValueError):
        BenchRecord("sparsedrop", 1, 1, 1, 0.5, 1.5, "total", 2, 1, 3, 1.0, 3).validate()
    with pytest.raises(ValueError):
        BenchRecord("sparsedrop", 1, 1, 1, 0.5, 0.5, "total", 5, 6, 7, 1.0, 3).validate()
    with pytest.raises(ValueError):
        BenchRecord("magic", 1, 1, 1, 0.5, 0.5, "total", 5, 5, 7, 1.0, 3).validate()


def test_bmsk_oracle_bytes_match_reference(oracle):
    import numpy as np

    for c in json.loads((GOLDEN / "bmsk.json").read_text()):
        R, C, mb, kb = c["geom"]
        words = np.array([int(h, 16) for h in c["words"]], dtype=np.uint64)
        assert oracle.write_mask(words, R, C, mb, kb).hex() == c["bytes"]


def test_bmsk_reader_rejects_malformed_input():
    from paper_2411_01238_b200.bmsk import from_bytes

    with pytest.raises(RuntimeError, match="magic"):
        from_bytes(b"XMSK rest", "bad")
    good = bytes.fromhex(json.loads((GOLDEN / "bmsk.json").read_text())[1]["bytes"])
    with pytest.raises(RuntimeError, match="version"):
        from_bytes(good[:4] + b"\x02" + good[5:], "v2")
    with pytest.raises(RuntimeError, match="truncated"):
        from_bytes(good[:12], "short")
    with pytest.raises(RuntimeError, match="truncated"):
        from_bytes(good[:-1], "short")
    with pytest.raises(RuntimeError, match="non-positive"):
        from_bytes(b"BMSK\x01" + bytes(16), "zero")
