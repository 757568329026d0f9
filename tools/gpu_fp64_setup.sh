# FP64 evidence for the 2D setup (factorization) kernels: the FP64 pipe utilisation and the
# executed DFMA/DMMA counts per launch (ncu), config 2; plus the metric names available.
mkdir -p gpurun_out
ncu --query-metrics 2>/dev/null | grep -i -E "fp64|dmma|dfma|dadd|dmul" > gpurun_out/r02_metrics_fp64.txt
M=gpu__time_duration.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__sass_thread_inst_executed_op_dfma_pred_on.sum,sm__sass_thread_inst_executed_op_dadd_pred_on.sum,sm__sass_thread_inst_executed_op_dmul_pred_on.sum,sm__inst_executed_pipe_fp64.sum,dram__bytes_read.sum,dram__bytes_write.sum
timeout 900 ncu --metrics $M --clock-control none -k regex:"k_band_solve|k_gauss_jordan|k_bt_factor|k_band_ldlt|k_schur_bb|k_coupling|k_fdm_solve" -c 14 --csv --log-file gpurun_out/r02_fp64_setup.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-sweep > gpurun_out/r02_fp64_setup.log 2>&1
echo rc=$? >> gpurun_out/r02_fp64_setup.log
