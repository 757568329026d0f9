# Round-end profile capture (each ncu pass only after the same command ran clean).
mkdir -p gpurun_out
python -c "from paper_1312_5653_b200 import build; build.build()"
timeout 900 python bench.py --impl reference > gpurun_out/p_bench_ref.json 2> gpurun_out/p_bench_ref.err
timeout 900 python bench.py > gpurun_out/p_bench_c2.json 2> gpurun_out/p_bench_c2.err
FETIGPU_EAGER=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/p_launches_c2.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-sweep > gpurun_out/p_ncu1.log 2>&1
FETIGPU_EAGER=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_sym_gemv|k_arnoldi_tail" --launch-skip 200 -c 3 -o gpurun_out/p_full_c2 python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-sweep > gpurun_out/p_ncu2.log 2>&1
FETIGPU_EAGER=1 timeout 900 ncu --set full --clock-control none -k regex:"k_fdm_solve" --launch-skip 2 -c 1 -o gpurun_out/p_full_c2_bt python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-sweep > gpurun_out/p_ncu3.log 2>&1
timeout 900 python bench.py --config 4 --steps 5 --warmup 3 > gpurun_out/p_bench_c4.json 2> gpurun_out/p_bench_c4.err
timeout 1500 python bench.py --config 5 --steps 3 --warmup 3 > gpurun_out/p_bench_c5.json 2> gpurun_out/p_bench_c5.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:"k3_(sym|bb_solve|fdm|lam|gather|mdot|mupdate|gcp|coarse_rhs|dense_gemv|norm|scale|axpby|mcombine|sub|split|tb_minus|ri_rhs|assemble_x|apply_global|tridiag|real|conj|imag|recover|ub_correct)" --log-file gpurun_out/p_launches_c4.csv python tools/run3d.py --config 4 --solves 1 > gpurun_out/p_ncu4.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k3_sym_rows" --launch-skip 4 -c 2 -o gpurun_out/p_full_c4 python tools/run3d.py --config 4 --solves 1 > gpurun_out/p_ncu5.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:"k3_fdm_solve" -c 1 -o gpurun_out/p_full_c4_bt python tools/run3d.py --config 4 --solves 1 > gpurun_out/p_ncu6.log 2>&1
