#!/bin/bash
# ncu --set full captures of every hot-path kernel class at C4 (one GPU, one
# process per kernel; run only after the same program exited 0 without ncu).
# usage (on the GPU box): bash tools/ncu_all.sh <tag>   -> gpurun_out/<tag>_c4_<kernel>_full.txt
# (the .ncu-rep files stay in /tmp on the box: gpurun_out is capped at 64 MiB)
tag=${1:-r02c}
mkdir -p gpurun_out
python tools/one_step.py C4 - 1 > gpurun_out/${tag}_plain.log 2>&1 || { echo "plain run failed"; exit 1; }
NCU="ncu --set full --clock-control none"
REP=/tmp/ncu_rep; mkdir -p $REP
cap() {  # name regex skip count
  $NCU -k "regex:$2" --launch-skip $3 -c $4 -o $REP/${tag}_c4_$1 -f \
      python tools/one_step.py C4 - 1 > $REP/ncu_$1.log 2>&1
  echo "$1 rc=$?"
  bash tools/ncu_summary.sh $REP/${tag}_c4_$1.ncu-rep "C4 $1 (launch-skip $3, $4 launch(es))" \
      > gpurun_out/${tag}_c4_$1_full.txt
}
# solve (the second k_sell_cheb launch is the first full pass over A_e)
cap k_sell_cheb      '^k_sell_cheb'      1 1
cap k_sell_hipt_mid  '^k_sell_hipt_mid'  0 1
cap k_sell_spmv      '^k_sell_spmv'      0 1
cap k_spmv           '^k_spmv'           0 4
cap k_dense_gemv     '^k_dense_gemv'     0 1
# the PCG vector kernels only run inside the WHILE graph: capture them on the host loop
SPHC_PCG_GRAPH=0 cap k_pcg            '^k_pcg_'           0 3
cap k_reduce         '^k_reduce'         0 2
# setup
cap k_spgemm_thin_fill '^k_spgemm_thin_fill' 0 1
cap k_spgemm_thin_count '^k_spgemm_thin_count' 0 1
cap k_spgemm_fill    '^k_spgemm_fill$'   0 1
cap k_spgemm_fill_cta '^k_spgemm_fill_cta' 0 1
cap k_spgemm_count   '^k_spgemm_count$'  0 1
cap k_emin_step      '^k_emin_step'      0 2
cap k_emin_setup     '^k_emin_setup'     0 2
cap k_agg_roots      '^k_agg_roots'      0 1
cap k_hsw_dot        '^k_hsw_dot'        0 1
cap k_lanczos_coop   '^k_lanczos_coop'   0 1
cap k_pc_fixpoint    '^k_pc_fixpoint'    1 1
cap k_nodal_smooth   '^k_nodal_smooth'   0 2
ls -la gpurun_out/${tag}_c4_*_full.txt
