mkdir -p gpurun_out
python -c "from paper_1312_5653_b200 import build; build.build()"
timeout 1200 python -m pytest tests/test_gpu3d.py tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/pytest_gpu3d.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu3d.log
timeout 600 python tools/run3d.py --config 4 --solves 1 > gpurun_out/run3d_c4.log 2>&1
FETIGPU3D_GJ=ffma timeout 600 python tools/run3d.py --config 4 --solves 1 > gpurun_out/run3d_c4_ffma.log 2>&1
timeout 900 python tools/run3d.py --config 5 --solves 1 > gpurun_out/run3d_c5.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:"k3_gj_update64_tc" --launch-skip 10 -c 1 -o gpurun_out/gj_tc python tools/run3d.py --config 4 --solves 0 > gpurun_out/ncu_gj.log 2>&1
