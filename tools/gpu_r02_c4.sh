#!/bin/bash
# Round-2 C4 measurement: bench line, launch list, ncu --set full captures of
# the solve's and setup's dominant kernels at C4 (one GPU).
set -x
mkdir -p gpurun_out
python bench.py --steps 5 --warmup 3 > gpurun_out/r02_bench_c4.json 2> gpurun_out/r02_bench_c4.err
NCU="ncu --clock-control none"
$NCU --metrics gpu__time_duration.sum --csv --log-file gpurun_out/r02_c4_launches.csv \
    python tools/one_step.py C4 - 2 > gpurun_out/ncu_launch.log 2>&1
for k in k_sell_cheb k_emin_step; do
  $NCU --set full --import-source on -k regex:$k -c 1 -o gpurun_out/r02_c4_$k \
      python tools/one_step.py C4 - 1 > gpurun_out/ncu_$k.log 2>&1
done
$NCU --set full --import-source on -k regex:k_spgemm_fill -c 4 -o gpurun_out/r02_c4_k_spgemm_fill \
    python tools/one_step.py C4 - 1 > gpurun_out/ncu_fill.log 2>&1
ls -la gpurun_out
