"""Aggregate ncu source-page stall samples per CUDA source line.
usage: ncu -i rep --page source --csv --print-source cuda,sass > x.csv; python ncu_lines.py x.csv [func-substr]"""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
want = sys.argv[2] if len(sys.argv) > 2 else ""
cur_file = cur_func = None
hdr = None
agg = collections.defaultdict(lambda: [0, 0, collections.Counter(), ""])
for r in rows:
    if not r: continue
    if r[0] == "File Path": cur_file = r[1].split("/")[-1]; continue
    if r[0] == "Function Name": cur_func = r[1]; continue
    if r[0] == "Line No": hdr = r; continue
    if hdr is None or want not in (cur_func or ""): continue
    try:
        ln = int(r[0])
    except ValueError:
        continue
    d = dict(zip(hdr, r))
    try:
        s = int(d.get("Warp Stall Sampling (All Samples)") or 0)
        ex = int(d.get("Instructions Executed") or 0)
    except ValueError:
        continue
    key = (cur_file, ln)
    agg[key][0] += s; agg[key][1] += ex; agg[key][3] = r[1][:80]
    for k, v in d.items():
        if k.startswith("stall_") and "Not Issued" not in k and v and v.isdigit():
            agg[key][2][k] += int(v)
tot = sum(v[0] for v in agg.values()) or 1
for key, (s, ex, st, src) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:25]:
    top = ", ".join(f"{k[6:]}:{v}" for k, v in st.most_common(3))
    print(f"{100*s/tot:5.1f}% ex={ex:9d} {key[0]}:{key[1]:<4d} {src.strip()[:60]:60s} [{top}]")
