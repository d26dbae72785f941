"""Warp-instruction mix of an `ncu --page source --csv --print-source sass`
export: executed warp instructions per opcode (and per value when the value
count is given), plus the address ranges that hold most of them.
Measurement helper: python tools/ncu_opmix.py src.csv[.gz] [values]"""
import collections
import csv
import gzip
import sys


def main(path, values=None):
    f = gzip.open(path, "rt") if path.endswith(".gz") else open(path)
    rows = list(csv.reader(f))
    hdr = rows[1]
    ix = {h: i for i, h in enumerate(hdr)}
    ops = collections.Counter()
    samples = collections.Counter()
    total = 0
    for r in rows[2:]:
        if len(r) < len(hdr):
            continue
        src = r[ix["Source"]].strip()
        toks = src.split()
        if not toks:
            continue
        op = toks[1] if toks[0].startswith("@") and len(toks) > 1 else toks[0]
        op = op.split(".")[0]
        n = float(r[ix["Instructions Executed"]] or 0)
        ops[op] += n
        samples[op] += float(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
        total += n
    print(f"total warp instructions {total:.4g}" + (f"  per value {total * 32 / values:.2f} thread-instr" if values else ""))
    for op, n in ops.most_common(40):
        extra = f" {n * 32 / values:6.2f}/value" if values else ""
        print(f"  {op:10s} {n:12.4g} {100 * n / total:5.1f}%{extra}  samples {samples[op]:.0f}")


if __name__ == "__main__":
    main(sys.argv[1], float(sys.argv[2]) if len(sys.argv) > 2 else None)
