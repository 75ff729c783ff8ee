"""Per-launch list of the measured rep of tools/one_step.py (second
k_strength onwards), filtered by regex; with --agg, per-kernel totals."""
import csv, collections, re, sys
rows = [l for l in open(sys.argv[1]) if not l.startswith("==")]
r = list(csv.reader(rows)); hdr = r[0]; data = r[1:]
ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
gi = hdr.index("Grid Size") if "Grid Size" in hdr else None
vals = [(d[ki].split("(")[0], float(d[vi].replace(",", "")) * {"ns": 1e-3, "us": 1, "ms": 1e3}[d[ui]],
         d[gi] if gi is not None else "") for d in data if len(d) > ui]
starts = [i for i, v in enumerate(vals) if v[0].startswith("k_strength")]
rep = vals[starts[len(starts) // 2] - 0:]
pat = re.compile(sys.argv[2] if len(sys.argv) > 2 and sys.argv[2] != "--agg" else ".")
if "--agg" in sys.argv:
    agg = collections.defaultdict(lambda: [0, 0.0])
    for k, v, g in rep:
        agg[k][0] += 1; agg[k][1] += v
    print(f"total {sum(v for _, v, _ in rep):.1f} us over {len(rep)} launches")
    for k, (c, v) in sorted(agg.items(), key=lambda x: -x[1][1])[:30]:
        print(f"{v:9.1f} us x{c:4d} {k[:80]}")
else:
    for i, (k, v, g) in enumerate(rep):
        if pat.search(k):
            print(i, k[:34], round(v, 1), g)
