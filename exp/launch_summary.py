"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list: per kernel count, total, mean, and the
per-iteration profile of each kernel (first/middle/last launches)."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
h = rows[hi]
tot, cnt, seq = collections.defaultdict(float), collections.Counter(), []
for r in rows[hi + 1:]:
    d = dict(zip(h, r))
    k = d["Kernel Name"].split("(")[0].replace("void ", "")
    k = k.split("<")[0] + ("<B>" if "true>" in d["Kernel Name"] else "")
    v = float(d["Metric Value"]) / 1e3
    tot[k] += v
    cnt[k] += 1
    seq.append((k, v))
T = sum(tot.values())
for k in sorted(tot, key=lambda k: -tot[k]):
    print(f"{k:40s} n={cnt[k]:6d} total={tot[k] / 1e3:9.2f} ms ({100 * tot[k] / T:5.1f}%) mean={tot[k] / cnt[k]:8.1f} us")
for k in tot:
    v = [x for kk, x in seq if kk == k]
    if len(v) > 30:
        m = len(v) // 2
        print(k, "first", [round(x) for x in v[:6]], "mid", [round(x) for x in v[m:m + 6]], "last",
              [round(x) for x in v[-6:]])
