# Round-2 profile capture of the final code (each ncu pass only after the same command ran
# clean without ncu).  Outputs into gpurun_out/; summaries are copied to profiles/ by hand.
mkdir -p gpurun_out
python -c "from paper_1312_5653_b200 import build; build.build()"
timeout 900 python bench.py --impl reference > gpurun_out/f_bench_ref.json 2> gpurun_out/f_bench_ref.err
timeout 900 python bench.py > gpurun_out/f_bench_c2.json 2> gpurun_out/f_bench_c2.err
FETIGPU_NO_FDM=1 timeout 900 python bench.py --no-cpu-baseline --no-sweep > gpurun_out/f_bench_c2_nofdm.json 2>/dev/null
timeout 900 python bench.py --config 3 --no-cpu-baseline > gpurun_out/f_bench_c3.json 2> gpurun_out/f_bench_c3.err
timeout 900 python bench.py --config 4 --steps 5 > gpurun_out/f_bench_c4.json 2> gpurun_out/f_bench_c4.err
timeout 1500 python bench.py --config 5 --steps 3 > gpurun_out/f_bench_c5.json 2> gpurun_out/f_bench_c5.err
# launch list of the bench command (eager: ncu cannot profile conditional-graph kernel nodes)
FETIGPU_EAGER=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/f_launches_c2.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-sweep > gpurun_out/f_ncu1.log 2>&1
# full capture of the per-step kernels (GEMVs, tail) and the setup / elimination kernels
FETIGPU_EAGER=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_sym_gemv|k_arnoldi_tail" --launch-skip 200 -c 4 -o gpurun_out/f_full_c2 python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-sweep > gpurun_out/f_ncu2.log 2>&1
M=gpu__time_duration.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_tensor_subpipe_dmma.sum,sm__sass_thread_inst_executed_op_dfma_pred_on.sum,sm__sass_thread_inst_executed_op_dmul_pred_on.sum,sm__sass_thread_inst_executed_op_dadd_pred_on.sum,dram__bytes_read.sum,dram__bytes_write.sum
timeout 900 ncu --metrics $M --clock-control none -k regex:"k_assemble|k_fdm_solve|k_sym_sweep_inverse|k_schur_bb|k_coupling|k_band_ldlt|k_coarse|k_gauss_jordan|k_pack_sym" -c 16 --csv --log-file gpurun_out/f_fp64_setup_c2.csv python -c "import paper_1312_5653_b200 as F; p=F.make_seeded_problem(1024,1e-4); s=F.SchurSolver(p,32,32,tol=1e-10,max_iter=2000); s.close()" > gpurun_out/f_ncu3.log 2>&1
# plane strain (no separable solve: banded LDL^T, multi-RHS band solve, Gauss-Jordan in global memory)
timeout 900 ncu --metrics $M --clock-control none -k regex:"k_band_ldlt|k_band_solve|k_bt_factor|k_gauss_jordan|k_sym_sweep_inverse" -c 12 --csv --log-file gpurun_out/f_fp64_setup_ps.csv python -c "import paper_1312_5653_b200 as F; p=F.make_cantilever_problem(64,1e-4); s=F.SchurSolver(p,12,4,tol=1e-10,max_iter=2000); s.close()" > gpurun_out/f_ncu4.log 2>&1
# phase timings: tail phases + the coarse CTAs of the dual GEMV's launch; Schur-solve phases
FETIGPU_TAIL_TIMES=1 timeout 300 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-sweep 2>&1 >/dev/null | grep fetigpu | tail -2 > gpurun_out/f_tail_times.txt
FETIGPU_PHASE_TIMES=1 timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-sweep 2>&1 >/dev/null | grep fetigpu | tail -3 >> gpurun_out/f_tail_times.txt
echo done > gpurun_out/f_done.txt
