"""Top source lines of an ncu report by warp-stall samples and instructions
(ncu --page source --print-source cuda,sass)."""
import csv, io, subprocess, sys, collections
rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
cur_file = None
rows = []
lines = out.splitlines()
i = 0
agg = collections.defaultdict(lambda: [0, 0, ""])
hdr = None
for ln in lines:
    if ln.startswith('"File Path"'):
        cur_file = next(csv.reader([ln]))[1].split("/")[-1]
        continue
    if ln.startswith('"Line No"'):
        hdr = next(csv.reader([ln]))
        continue
    if ln.startswith('"Function Name"') or hdr is None:
        continue
    r = next(csv.reader([ln]))
    if len(r) < len(hdr):
        continue
    try:
        samp = int(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
        inst = int(r[hdr.index("Instructions Executed")] or 0)
    except ValueError:
        continue
    key = (cur_file, r[0])
    agg[key][0] += samp
    agg[key][1] += inst
    agg[key][2] = r[1][:90]
tot_s = sum(v[0] for v in agg.values()) or 1
tot_i = sum(v[1] for v in agg.values()) or 1
print(f"total samples {tot_s}, instructions {tot_i}")
for (f, l), (s, n, src) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{100*s/tot_s:5.1f}% stall {100*n/tot_i:5.1f}% inst  {f}:{l}  {src}")
