mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 2400 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py --no-cpu-baseline --no-sweep > gpurun_out/bench_v15.json 2> gpurun_out/bench_v15.err; echo "bench rc=$?" >> gpurun_out/bench_v15.err
FETIGPU_EAGER=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_v15.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-sweep > gpurun_out/ncu_l.log 2>&1
