mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench_v10.json 2> gpurun_out/bench_v10.err; echo "bench rc=$?" >> gpurun_out/bench_v10.err
FETIGPU_EAGER=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_v10.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-sweep > gpurun_out/ncu_l.log 2>&1; echo "ncu rc=$?" >> gpurun_out/ncu_l.log
FETIGPU_EAGER=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_sym_gemv|k_arnoldi_tail|k_bt_solve" --launch-skip 200 -c 6 -o gpurun_out/full_v10 python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-sweep > gpurun_out/ncu_f.log 2>&1; echo "ncuf rc=$?" >> gpurun_out/ncu_f.log
