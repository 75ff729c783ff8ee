set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo tests_exit=$? >> gpurun_out/gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
for k in 1 0; do echo K8=$k; SPHC_SELL_K8=$k timeout 120 python tools/solve_timing.py C2 2>&1 | sed -n 3p; done > gpurun_out/k8b.txt 2>&1
timeout 400 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
timeout 600 python bench.py --config C4 --steps 3 --warmup 3 --no-cpu-baseline --no-scale-roofline > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c2_launches.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-scale-roofline > gpurun_out/ncu.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_sell_cheb -s 40 -c 1 -o gpurun_out/sell_cheb_c2 python tools/one_step.py C2 > gpurun_out/ncu_sell.log 2>&1
timeout 900 python bench.py --config C5 --steps 2 --warmup 3 --no-cpu-baseline --no-scale-roofline > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
echo done
