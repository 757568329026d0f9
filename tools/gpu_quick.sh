mkdir -p gpurun_out
python -c "from paper_1312_5653_b200 import build; build.build()"
timeout 900 python bench.py --no-cpu-baseline --no-sweep > gpurun_out/bench_v29.json 2> gpurun_out/bench_v29.err
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_fullspace.py tests/test_golden.py tests/test_sharding.py tests/test_experiments.py -m gpu -x -q > gpurun_out/pytest_v29.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_v29.log
FETIGPU_NO_FDM=1 timeout 900 python bench.py --no-cpu-baseline --no-sweep > gpurun_out/bench_v29_nofdm.json 2>/dev/null
