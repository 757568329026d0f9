mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py --no-cpu-baseline --no-sweep > gpurun_out/bench_v19.json 2> gpurun_out/bench_v19.err; echo "bench rc=$?" >> gpurun_out/bench_v19.err
FETIGPU_NO_ELIM_REUSE=1 timeout 900 python bench.py --no-cpu-baseline --no-sweep > gpurun_out/bench_v19_noreuse.json 2>/dev/null
