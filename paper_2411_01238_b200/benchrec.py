"""Benchmark records in the reference SPEC's CSV schema (
SPEC.md:438-463): header `method,m,n,k,sparsity,realized_sparsity,pass,
nanos_median,nanos_p10,nanos_p90,effective_gflops,repeats`, one row per
record, '.' decimal point, LF newlines, column order frozen."""
from __future__ import annotations

import csv
import dataclasses
import io
from typing import Iterable, List

HEADER = ["method", "m", "n", "k", "sparsity", "realized_sparsity", "pass", "nanos_median", "nanos_p10",
          "nanos_p90", "effective_gflops", "repeats"]
METHODS = ("dense", "dropout_dense", "block_dropout_dense", "sparsedrop")
PASSES = ("forward", "backward", "total")


@dataclasses.dataclass
class BenchRecord:
    method: str
    m: int
    n: int
    k: int
    sparsity: float
    realized_sparsity: float
    pass_: str
    nanos_median: int
    nanos_p10: int
    nanos_p90: int
    effective_gflops: float
    repeats: int

    def validate(self) -> None:
        if self.method not in METHODS:
            raise ValueError(f"unknown method {self.method!r}")
        if self.pass_ not in PASSES:
            raise ValueError(f"unknown pass {self.pass_!r}")
        if not (self.nanos_p10 <= self.nanos_median <= self.nanos_p90):
            raise ValueError("nanos_p10 <= nanos_median <= nanos_p90 violated")
        if not (0.0 <= self.realized_sparsity <= 1.0):
            raise ValueError("realized_sparsity outside [0, 1]")

    def row(self) -> list:
        return [self.method, self.m, self.n, self.k, repr(float(self.sparsity)), repr(float(self.realized_sparsity)),
                self.pass_, int(self.nanos_median), int(self.nanos_p10), int(self.nanos_p90),
                repr(float(self.effective_gflops)), int(self.repeats)]


def percentile_record(method, m, n, k, sparsity, realized, pass_, nanos: List[float], flops: float) -> BenchRecord:
    """Median / p10 / p90 over the timed repeats."""
    s = sorted(nanos)

    def pct(q):
        i = min(len(s) - 1, max(0, int(round(q * (len(s) - 1)))))
        return int(round(s[i]))

    med = pct(0.5)
    rec = BenchRecord(method, m, n, k, sparsity, realized, pass_, med, pct(0.1), pct(0.9),
                      flops / med if med > 0 else 0.0, len(s))
    rec.validate()
    return rec


def to_csv(records: Iterable[BenchRecord]) -> str:
    buf = io.StringIO()
    w = csv.writer(buf, lineterminator="\n")
    w.writerow(HEADER)
    for r in records:
        r.validate()
        w.writerow(r.row())
    return buf.getvalue()


def emit_csv(records: Iterable[BenchRecord], path: str) -> None:
    text = to_csv(records)
    try:
        with open(path, "w", newline="") as f:
            f.write(text)
    except OSError as e:
        raise RuntimeError(f"cannot write {path}: {e}") from e


def parse_csv(text: str) -> List[BenchRecord]:
    rows = list(csv.reader(io.StringIO(text)))
    if not rows or rows[0] != HEADER:
        raise ValueError("bad BenchRecord CSV header")
    out = []
    for r in rows[1:]:
        out.append(BenchRecord(r[0], int(r[1]), int(r[2]), int(r[3]), float(r[4]), float(r[5]), r[6], int(r[7]),
                               int(r[8]), int(r[9]), float(r[10]), int(r[11])))
    return out
