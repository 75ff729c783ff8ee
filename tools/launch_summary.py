"""Summarise an ncu --csv launch list (gpu__time_duration.sum)."""
import collections, csv, io, sys
path = sys.argv[1]
frac = float(sys.argv[2]) if len(sys.argv) > 2 else 0.5   # keep the last `frac` of launches
lines = [l for l in open(path) if not l.startswith("==")]
rows = [r for r in csv.DictReader(io.StringIO("".join(lines))) if r["Metric Name"] == "gpu__time_duration.sum"]
rows = rows[int(len(rows) * (1 - frac)):]
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows:
    v = float(r["Metric Value"].replace(",", ""))
    u = r["Metric Unit"]
    v *= {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "second": 1e6, "s": 1e6}[u]
    name = r["Kernel Name"].split("(")[0][:60]
    agg[name][0] += 1
    agg[name][1] += v
tot = sum(v[1] for v in agg.values())
print(f"total GPU time {tot/1e3:.3f} ms over {len(rows)} launches")
for k, (c, v) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:int(sys.argv[3]) if len(sys.argv) > 3 else 30]:
    print(f"{v/1e3:8.3f} ms {100*v/tot:5.1f}%  x{c:5d}  avg {v/c:8.2f} us  {k}")
