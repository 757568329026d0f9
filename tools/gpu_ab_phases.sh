# Per-phase tail timestamps and per-kernel step spans of two prebuilt libraries
# (paper_1312_5653_b200/_lib/libfetigpu_{base,new}.so).  Usage: bash tools/gpu_ab_phases.sh <tag>
mkdir -p gpurun_out
L=paper_1312_5653_b200/_lib
for v in base new; do
  cp $L/libfetigpu_$v.so $L/libfetigpu.so
  FETIGPU_TAIL_TIMES=1 timeout 300 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-sweep > /dev/null 2> gpurun_out/ph_$1_tail_$v.txt
  FETIGPU_STEP_TIMES=1 timeout 300 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-sweep > /dev/null 2> gpurun_out/ph_$1_step_$v.txt
done
cp $L/libfetigpu_new.so $L/libfetigpu.so
