mkdir -p gpurun_out
python -c "from paper_1312_5653_b200 import build; build.build()"
timeout 1200 python -m pytest tests/test_gpu3d.py tests/test_sharding3d.py -m gpu -x -q > gpurun_out/pytest_gpu3d.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu3d.log
timeout 900 python bench.py --config 4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo "rc=$?" >> gpurun_out/bench_c4.err
timeout 1500 python bench.py --config 5 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo "rc=$?" >> gpurun_out/bench_c5.err
