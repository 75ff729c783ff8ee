#!/bin/bash
# usage: tools/ncu_summary.sh <rep.ncu-rep> "<description>" > profiles/<name>.txt
rep=$1; desc=$2
echo "# ncu --set full --clock-control none: $desc"
ncu -i "$rep" --page details --csv 2>/dev/null | python3 -c "
import sys,csv
rows=list(csv.reader(sys.stdin)); h=rows[0]
for r in rows[1:]:
    print(f'{r[h.index(\"Section Name\")]:35s} {r[h.index(\"Metric Name\")]:45s} {r[h.index(\"Metric Value\")]:>14s} {r[h.index(\"Metric Unit\")]}')
"
echo "# raw"
ncu -i "$rep" --page raw --csv 2>/dev/null | python3 -c "
import sys,csv
rows=list(csv.reader(sys.stdin)); hdr=rows[0]; units=rows[1]; vals=rows[2]
for w in ['dram__bytes_read.sum','dram__bytes_write.sum','gpu__time_duration.sum','lts__t_sector_hit_rate.pct','sm__warps_active.avg.pct_of_peak_sustained_active','launch__grid_size','launch__registers_per_thread']:
    if w in hdr: i=hdr.index(w); print(w, vals[i], units[i])
"
