mkdir -p gpurun_out
python -c "from paper_1312_5653_b200 import build; build.build()"
timeout 1200 python -m pytest tests/test_sharding3d.py tests/test_gpu3d.py -m gpu -x -q > gpurun_out/pytest_gpu3d.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu3d.log
timeout 900 python bench.py --config 4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo "rc=$?" >> gpurun_out/bench_c4.err
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-sweep > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo "rc=$?" >> gpurun_out/bench_c2.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k3_sym_rows|k3_bb_solve1" --launch-skip 4 -c 2 -o gpurun_out/full3d_c5 python tools/run3d.py --config 5 --solves 1 > gpurun_out/ncu3d_f5.log 2>&1; echo "rc=$?" >> gpurun_out/ncu3d_f5.log
