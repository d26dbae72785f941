"""Print an address range of an ncu source-page export (SASS) with executed
counts and stall samples.  Measurement helper:
python tools/ncu_range.py src.csv[.gz] START_HEX END_HEX (suffix match on the address)"""
import csv
import gzip
import sys

path, lo, hi = sys.argv[1], int(sys.argv[2], 16), int(sys.argv[3], 16)
f = gzip.open(path, "rt") if path.endswith(".gz") else open(path)
rows = list(csv.reader(f))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
for r in rows[2:]:
    if len(r) < len(hdr):
        continue
    a = int(r[ix["Address"]], 16) & 0xfffff
    if lo <= a <= hi:
        s = float(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
        top = sorted(((float(r[ix[h]] or 0), h[6:]) for h in stalls), reverse=True)[:2]
        ts = ",".join(f"{n}={int(v)}" for v, n in top if v > 0)
        print(f"{a:05x} {float(r[ix['Instructions Executed']] or 0):10.0f} {int(s):5d} {r[ix['Source']].strip()[:70]:70s} {ts}")
