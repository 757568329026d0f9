mkdir -p gpurun_out
python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-sweep > gpurun_out/r02_pt_bench.json 2> gpurun_out/r02_pt_bench.err
FETIGPU_EAGER=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_arnoldi_tail|k_sym_gemv" --launch-skip 60 -c 6 -o gpurun_out/r02_tail_full python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-sweep > gpurun_out/r02_pt_ncu.log 2>&1
FETIGPU_TAIL_TIMES=1 timeout 300 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-sweep > /dev/null 2> gpurun_out/r02_tail_times.txt
