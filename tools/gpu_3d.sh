mkdir -p gpurun_out
python -c "from paper_1312_5653_b200 import build; build.build()"
timeout 600 python tools/run3d.py --config 4 --n 32 --s 2 --solves 1 > gpurun_out/run3d_small.log 2>&1; echo "rc=$?" >> gpurun_out/run3d_small.log
timeout 1200 python -m pytest tests/test_gpu3d.py tests/test_sharding3d.py -m gpu -x -q > gpurun_out/pytest_gpu3d.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu3d.log
timeout 900 python tools/run3d.py --config 4 --solves 2 > gpurun_out/run3d_c4.log 2>&1
timeout 900 python tools/run3d.py --config 5 --solves 2 > gpurun_out/run3d_c5.log 2>&1
