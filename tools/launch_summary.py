"""Sum an `ncu --metrics gpu__time_duration.sum --csv --log-file` launch list
by kernel: count and total us (or another metric's total).  Measurement
helper: python tools/launch_summary.py launches.csv [metric]"""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
start = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr = rows[start]
ix = {h: i for i, h in enumerate(hdr)}
tot, cnt = collections.Counter(), collections.Counter()
metric = sys.argv[2] if len(sys.argv) > 2 else "gpu__time_duration.sum"
for r in rows[start + 1:]:
    if "Metric Name" in ix and r[ix["Metric Name"]] != metric:
        continue
    k = r[ix["Kernel Name"]].split("(")[0][:70]
    tot[k] += float(r[ix["Metric Value"]].replace(",", ""))
    cnt[k] += 1
for k, v in tot.most_common():
    print(f"{k:70s} n={cnt[k]:5d} total={v / 1e3:10.1f} us  mean={v / 1e3 / cnt[k]:9.2f} us")
