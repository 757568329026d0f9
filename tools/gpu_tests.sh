mkdir -p gpurun_out
python -c "from paper_1312_5653_b200 import build; build.build()"
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_all.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu_all.log
