# Round-end profile capture (each ncu pass only after the same command ran clean).
mkdir -p gpurun_out
python -c "from paper_1312_5653_b200 import build; build.build()"
FETIGPU_EAGER=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/p_launches_c2.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-sweep > gpurun_out/p_ncu1.log 2>&1
FETIGPU_EAGER=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_sym_gemv|k_arnoldi_tail" --launch-skip 200 -c 3 -o gpurun_out/p_full_c2 python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-sweep > gpurun_out/p_ncu2.log 2>&1
FETIGPU_EAGER=1 timeout 900 ncu --set full --clock-control none -k regex:"k_fdm_solve" --launch-skip 2 -c 1 -o gpurun_out/p_full_c2_bt python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-sweep > gpurun_out/p_ncu3.log 2>&1
