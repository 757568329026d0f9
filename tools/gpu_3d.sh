mkdir -p gpurun_out
python -c "from paper_1312_5653_b200 import build; build.build()"
timeout 900 python bench.py --config 4 --steps 5 --warmup 3 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo "rc=$?" >> gpurun_out/bench_c4.err
timeout 1500 python bench.py --config 5 --steps 3 --warmup 3 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo "rc=$?" >> gpurun_out/bench_c5.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k3_bb_solve_tma|k3_bb_msolve2|k3_gj_update64" --launch-skip 2 -c 3 -o gpurun_out/full3d_c4_aux python tools/run3d.py --config 4 --solves 1 > gpurun_out/ncu3d_aux.log 2>&1; echo "rc=$?" >> gpurun_out/ncu3d_aux.log
