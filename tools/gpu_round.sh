mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py --no-cpu-baseline --no-sweep > gpurun_out/bench_v20.json 2> gpurun_out/bench_v20.err; echo "bench rc=$?" >> gpurun_out/bench_v20.err
FETIGPU_NO_SPLIT=1 timeout 900 python bench.py --no-cpu-baseline --no-sweep > gpurun_out/bench_v20_nosplit.json 2>/dev/null
