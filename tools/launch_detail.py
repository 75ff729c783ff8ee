"""Per-launch list (second half = measured rep) filtered by kernel-name regex."""
import csv, io, re, sys
lines = [l for l in open(sys.argv[1]) if not l.startswith("==")]
rows = [r for r in csv.DictReader(io.StringIO("".join(lines))) if r["Metric Name"] == "gpu__time_duration.sum"]
rows = rows[len(rows) // 2:]
pat = re.compile(sys.argv[2] if len(sys.argv) > 2 else ".")
for i, r in enumerate(rows):
    n = r["Kernel Name"]
    if pat.search(n):
        v = float(r["Metric Value"]) * {"ns": 1e-3, "us": 1, "ms": 1e3}.get(r["Metric Unit"], 1)
        print(i, n.split("(")[0][:40], f"{v:.1f} us", r.get("Grid Size", ""))
