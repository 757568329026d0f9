mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu3d.py tests/test_sharding3d.py -m gpu -x -q > gpurun_out/pytest_fdm3.log 2>&1; echo rc=$? >> gpurun_out/pytest_fdm3.log
timeout 900 python bench.py --config 4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/c4_fdm.json 2>gpurun_out/c4_fdm.err
FETIGPU3D_NO_FDM=1 timeout 900 python bench.py --config 4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/c4_nofdm.json 2>/dev/null
