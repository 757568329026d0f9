mkdir -p gpurun_out
FETIGPU_PHASE_TIMES=1 timeout 300 python tools/profile_step.py > gpurun_out/phases.log 2>&1
FETIGPU_PHASE_TIMES=1 timeout 300 python tools/profile_step.py >> gpurun_out/phases.log 2>&1
