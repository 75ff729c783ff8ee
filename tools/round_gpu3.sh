set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo tests_exit=$? >> gpurun_out/gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 400 python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
timeout 600 python bench.py --config C4 --steps 3 --warmup 3 --no-cpu-baseline --no-scale-roofline > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c2_launches.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-scale-roofline > gpurun_out/ncu.log 2>&1
echo done
