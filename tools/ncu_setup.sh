#!/bin/bash
# ncu --set full of the setup kernels in their closing state (emin classes,
# Galerkin fills, segmented sort) at C4; text summaries only in gpurun_out/.
tag=${1:-r02i}
mkdir -p gpurun_out
python tools/one_step.py C4 - 1 > /tmp/${tag}_plain.log 2>&1 || { echo "plain run failed"; exit 1; }
NCU="ncu --set full --clock-control none"
REP=/tmp/ncu_rep; mkdir -p $REP
cap() {  # name regex skip count
  $NCU -k "regex:$2" --launch-skip $3 -c $4 -o $REP/${tag}_c4_$1 -f \
      python tools/one_step.py C4 - 1 > $REP/ncu_$1.log 2>&1
  echo "$1 rc=$?"
  bash tools/ncu_summary.sh $REP/${tag}_c4_$1.ncu-rep "C4 $1 (launch-skip $3, $4 launch(es))" \
      > gpurun_out/${tag}_c4_$1_full.txt
}
cap k_emin_step      '^k_emin_step'      0 2
cap k_emin_setup     '^k_emin_setup'     0 4
cap k_spgemm_fill    '^k_spgemm_fill$'   0 1
cap k_spgemm_fill_cta '^k_spgemm_fill_cta' 0 1
cap k_sort_rows      '^k_sort_rows'      0 2
ls -la gpurun_out/${tag}_c4_*_full.txt
