set -x
timeout 400 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
timeout 600 python bench.py --config C4 --steps 3 --warmup 3 --no-cpu-baseline --no-scale-roofline > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c2_launches.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-scale-roofline > gpurun_out/ncu.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k "regex:k_sell_cheb<false, 2>" -s 10 -c 1 -o gpurun_out/sell_cheb_l0_c2 python tools/one_step.py C2 > gpurun_out/ncu_sell.log 2>&1
echo done
