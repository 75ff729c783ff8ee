#!/bin/bash
# Round-2 closing measurements (delta-coded SELL kernels in): bench lines, the
# C4 launch list and setup timeline, ncu --set full of the three 16-bit
# kernels. Text only in gpurun_out/.
tag=${1:-r02f}
mkdir -p gpurun_out
run() { name=$1; shift; timeout 900 "$@" > gpurun_out/${tag}_$name.json 2> gpurun_out/${tag}_$name.err; echo "$name rc=$? $(grep '^{' gpurun_out/${tag}_$name.json | tail -1 | head -c 120)"; }
run bench_c4 python bench.py --steps 5 --warmup 3
run reference_arm_c4 python bench.py --impl reference --steps 5 --warmup 3
run bench_c2 python bench.py --config C2 --steps 20 --warmup 5
run bench_c3 python bench.py --config C3 --steps 10 --warmup 3
run bench_c5 python bench.py --config C5 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline
run bench_c4_partitioned python bench.py --partitioned --steps 3 --warmup 3 --no-cpu-baseline
timeout 900 ncu --clock-control none --metrics gpu__time_duration.sum --csv \
    --log-file /tmp/${tag}_c4_launches.csv python tools/one_step.py C4 - 1 > /tmp/ncu_launch.log 2>&1
python tools/launch_summary.py /tmp/${tag}_c4_launches.csv 1.0 60 > gpurun_out/${tag}_c4_launch_summary.txt 2>&1
TOPGAPS=10 MIN_MS=1.0 timeout 300 python tools/setup_timeline.py C4 2>&1 | grep -v -i warn > gpurun_out/${tag}_c4_setup_timeline.txt
NCU="ncu --set full --clock-control none"
REP=/tmp/ncu_rep; mkdir -p $REP
cap() {  # name regex skip count outname
  $NCU -k "regex:$2" --launch-skip $3 -c $4 -o $REP/${tag}_c4_$1 -f \
      python tools/one_step.py C4 - 1 > $REP/ncu_$1.log 2>&1
  echo "$1 rc=$?"
  bash tools/ncu_summary.sh $REP/${tag}_c4_$1.ncu-rep "C4 $1 (launch-skip $3, $4 launch(es))" \
      > gpurun_out/${tag}_c4_${5:-$1}_full.txt
}
# the roofline kernel: bench.py reads profiles/r*_c4_k_sell_cheb_full.txt
cap k_sell_cheb16 '^k_sell_cheb16$' 0 1 k_sell_cheb
cap k_sell_spmv16 '^k_sell_spmv16$' 0 1
cap k_sell_hipt_mid16 '^k_sell_hipt_mid16$' 0 1
ls -la gpurun_out | tail -24
