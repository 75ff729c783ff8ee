#!/bin/bash
# usage: tools/ncu_summary.sh <rep.ncu-rep> "<description>" > profiles/<name>.txt
rep=$1; desc=$2
echo "# ncu --set full --clock-control none: $desc"
ncu -i "$rep" --page details --csv 2>/dev/null | python3 -c "
import sys,csv
rows=list(csv.reader(sys.stdin)); h=rows[0]
last=None
for r in rows[1:]:
    kid=(r[h.index('ID')], r[h.index('Kernel Name')])
    if kid!=last:
        print(f'## launch {kid[0]}: {kid[1][:110]}'); last=kid
    print(f'{r[h.index(\"Section Name\")]:35s} {r[h.index(\"Metric Name\")]:45s} {r[h.index(\"Metric Value\")]:>14s} {r[h.index(\"Metric Unit\")]}')
"
echo "# raw (first launch; per-launch lines follow)"
ncu -i "$rep" --page raw --csv 2>/dev/null | python3 -c "
import sys,csv
rows=list(csv.reader(sys.stdin)); hdr=rows[0]; units=rows[1]
want=['dram__bytes_read.sum','dram__bytes_write.sum','gpu__time_duration.sum','lts__t_sector_hit_rate.pct','sm__warps_active.avg.pct_of_peak_sustained_active','launch__grid_size','launch__registers_per_thread']
vals=rows[2]
for w in want:
    if w in hdr: i=hdr.index(w); print(w, vals[i], units[i])
kn=hdr.index('Kernel Name') if 'Kernel Name' in hdr else None
for k,vals in enumerate(rows[2:]):
    name=vals[kn][:60] if kn is not None else ''
    out=[]
    for w in want[:3]:
        if w in hdr: i=hdr.index(w); out.append(f'{w}={vals[i]} {units[i]}')
    print(f'# launch {k}: {name}: '+'; '.join(out))
"
