"""Summarise an `ncu --page source --csv --print-source cuda,sass` export by source line:
stall samples, warp instructions, average active threads; top-N lines and per-file totals."""
import collections
import csv
import sys

path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
rows = []
fname = "?"
hdr = None
csv.field_size_limit(1 << 30)
with open(path, newline="") as f:
    for r in csv.reader(f):
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or r[0] in ("", "Function Name", "Kernel Name"):
            continue
        try:
            line = int(r[0])
        except ValueError:
            continue
        d = dict(zip(hdr, r))

        def num(k):
            try:
                return float(d.get(k, 0) or 0)
            except ValueError:
                return 0.0
        rows.append((fname, line, r[1][:90], num("Warp Stall Sampling (All Samples)"), num("Instructions Executed"),
                     num("Thread Instructions Executed"), num("stall_lg"), num("stall_long_sb"), num("stall_no_inst"),
                     num("stall_barrier"), num("stall_short_sb"), num("stall_wait")))
tot_s = sum(r[3] for r in rows) or 1
tot_i = sum(r[4] for r in rows) or 1
print(f"total samples {tot_s:.0f}  warp inst {tot_i:.3e}  avg threads {sum(r[5] for r in rows) / tot_i:.2f}")
byf = collections.defaultdict(lambda: [0, 0, 0])
for r in rows:
    byf[r[0]][0] += r[3]
    byf[r[0]][1] += r[4]
    byf[r[0]][2] += r[5]
for k, v in sorted(byf.items(), key=lambda kv: -kv[1][0]):
    print(f"  {k:28s} samples {100 * v[0] / tot_s:5.1f}%  inst {100 * v[1] / tot_i:5.1f}%  thr/inst {v[2] / max(v[1], 1):5.2f}")
print("top lines by stall samples: file:line samples% inst% thr/inst lg long_sb no_inst barrier short_sb wait | src")
for r in sorted(rows, key=lambda r: -r[3])[:top]:
    print(f"  {r[0]}:{r[1]} {100 * r[3] / tot_s:5.2f}% {100 * r[4] / tot_i:5.2f}% {r[5] / max(r[4], 1):5.1f} "
          f"{r[6]:.0f} {r[7]:.0f} {r[8]:.0f} {r[9]:.0f} {r[10]:.0f} {r[11]:.0f} | {r[2]}")
