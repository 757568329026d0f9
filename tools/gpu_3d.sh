mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu3d.py -m gpu -x -q > gpurun_out/pytest_gpu3d.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu3d.log
timeout 900 python tools/run3d.py --config 4 --solves 2 > gpurun_out/run3d_c4.log 2>&1; echo "rc=$?" >> gpurun_out/run3d_c4.log
