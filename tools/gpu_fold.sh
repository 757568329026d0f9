mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_golden.py -m gpu -x -q > gpurun_out/pytest_fold.log 2>&1; echo rc=$? >> gpurun_out/pytest_fold.log
bash tools/gpu_env_ab.sh FETIGPU_FDM_NOFOLD=1
rm -f gpurun_out/fdm_ab.log; bash tools/gpu_fdm_ab.sh
