"""Per-instruction view of an `ncu --page source --csv --print-source sass`
export: stall samples by reason, the hottest instructions with their top
stalls, and shared-memory wavefronts (ideal vs excessive) per opcode.
Measurement helper: python tools/ncu_source.py src.csv[.gz] [top]"""
import collections
import csv
import gzip
import io
import sys


def load(path):
    f = gzip.open(path, "rt") if path.endswith(".gz") else open(path)
    rows = list(csv.reader(f))
    # first row: kernel name; second: header
    hdr = rows[1]
    return hdr, rows[2:]


def num(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


def main(path, top=40):
    hdr, rows = load(path)
    ix = {h: i for i, h in enumerate(hdr)}
    stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    tot = collections.Counter()
    samples_total = 0
    op_wf = collections.defaultdict(lambda: [0.0, 0.0, 0.0, 0])
    recs = []
    for r in rows:
        if len(r) < len(hdr):
            continue
        src = r[ix["Source"]].strip()
        s = num(r[ix["Warp Stall Sampling (All Samples)"]])
        samples_total += s
        st = {c: num(r[ix[c]]) for c in stall_cols}
        for c, v in st.items():
            tot[c] += v
        op = src.split()[0] if src else "?"
        if op.startswith("@"):
            op = src.split()[1]
        w = op_wf[op.split(".")[0]]
        w[0] += num(r[ix["L1 Wavefronts Shared"]])
        w[1] += num(r[ix["L1 Wavefronts Shared Ideal"]])
        w[2] += num(r[ix["L1 Wavefronts Shared Excessive"]])
        w[3] += int(num(r[ix["Instructions Executed"]]))
        recs.append((s, r[ix["Address"]], src, st, num(r[ix["Instructions Executed"]])))
    print(f"total samples {samples_total:.0f}")
    for c, v in tot.most_common(12):
        print(f"  {c:28s} {v:10.0f}  {100 * v / max(1, samples_total):5.1f}%")
    print("\nshared wavefronts by opcode (total / ideal / excessive / warp-instrs):")
    for op, (a, b, c, n) in sorted(op_wf.items(), key=lambda kv: -kv[1][0]):
        if a > 0:
            print(f"  {op:10s} {a:12.0f} {b:12.0f} {c:12.0f} {n:12d}")
    print(f"\ntop {top} instructions by samples:")
    for s, addr, src, st, n in sorted(recs, key=lambda t: -t[0])[:top]:
        tops = ", ".join(f"{k[6:]}={v:.0f}" for k, v in sorted(st.items(), key=lambda kv: -kv[1])[:3] if v > 0)
        print(f"  {s:7.0f} {addr[-5:]} {src[:60]:60s} {tops}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)


def by_opcode(path):
    """samples per opcode family"""
    hdr, rows = load(path)
    ix = {h: i for i, h in enumerate(hdr)}
    c = collections.Counter()
    n = collections.Counter()
    tot = 0
    for r in rows:
        if len(r) < len(hdr):
            continue
        src = r[ix["Source"]].strip().split()
        if not src:
            continue
        op = src[1] if src[0].startswith("@") else src[0]
        s = num(r[ix["Warp Stall Sampling (All Samples)"]])
        c[op.split(".")[0]] += s
        n[op.split(".")[0]] += num(r[ix["Instructions Executed"]])
        tot += s
    for op, s in c.most_common(30):
        print(f"  {op:10s} {s:8.0f} {100 * s / tot:5.1f}%  instr {n[op]:12.0f}")
