mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_golden.py tests/test_gpu3d.py -m gpu -x -q > gpurun_out/pytest_v32.log 2>&1; echo rc=$? >> gpurun_out/pytest_v32.log
timeout 900 python bench.py --no-cpu-baseline --no-sweep > gpurun_out/bench_v32.json 2>/dev/null
FETIGPU_PHASE_TIMES=1 timeout 300 python tools/profile_step.py > gpurun_out/phases_v32.log 2>&1
