mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu3d.py tests/test_sharding3d.py -m gpu -x -q > gpurun_out/pytest_fdm3b.log 2>&1; echo rc=$? >> gpurun_out/pytest_fdm3b.log
timeout 900 python bench.py --config 4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/c4_fdmb.json 2>/dev/null
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k3_fdm_solve --csv python tools/run3d.py --config 4 --solves 1 2>/dev/null | grep gpu__time_duration > gpurun_out/fdm3b_ncu.log
