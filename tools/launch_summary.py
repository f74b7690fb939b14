"""Summarise an ncu launch list (gpu__time_duration.sum CSV) for the last full
Schur frame (the last metrics-terminated launch group holding the tile
Cholesky; bench.py's PCG-baseline frames come after it).
  python tools/launch_summary.py launches.csv [-v] [--csv frame.csv]"""
import collections
import csv
import sys

path = sys.argv[1]
rows = list(csv.reader(open(path)))
hdr, data = None, []
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
names = [d["Kernel Name"] for d in data]
idx = [i for i, n in enumerate(names) if "k_finish_metrics" in n]
bounds = [(idx[k - 1] + 1 if k else 0, idx[k] + 1) for k in range(len(idx))] or [(0, len(data))]
schur = [b for b in bounds if sum("k_cholesky" in names[i] for i in range(*b)) == 1]
start, end = (schur or bounds)[-1]
tot, cnt, seq = collections.defaultdict(float), collections.Counter(), []
for d in data[start:end]:
    n = d["Kernel Name"].split("(")[0].replace("void ", "").replace("spb::", "")
    unit = d.get("Metric Unit", "nsecond")
    v = float(d["Metric Value"]) * {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3}.get(unit, 1e-3)
    tot[n] += v
    cnt[n] += 1
    seq.append((n, v))
s = sum(tot.values())
for n, v in sorted(tot.items(), key=lambda kv: -kv[1]):
    print(f"{n:28s} {cnt[n]:3d} x {v:9.1f} us {100 * v / s:5.1f}%")
print(f"frame total {s:.1f} us over {len(seq)} launches")
if "--csv" in sys.argv:
    out = sys.argv[sys.argv.index("--csv") + 1]
    with open(out, "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(hdr)
        for d in data[start:end]:
            w.writerow([d[k] for k in hdr])
if "-v" in sys.argv:
    print([(n[:12], round(v, 1)) for n, v in seq])
