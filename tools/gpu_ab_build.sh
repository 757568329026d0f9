# A/B of a build-time define (e.g. a launch-bounds experiment): bench with the default build, then with $1 (e.g.
# "-DFETIGPU_TAIL_MINB=2"), then restore the default build.  Usage: bash tools/gpu_ab_build.sh "<defines>" <tag>
mkdir -p gpurun_out
python -c "from paper_1312_5653_b200 import build; build.build(force=True)"
for k in 1 2; do timeout 600 python bench.py --no-cpu-baseline --no-sweep --steps 30 > gpurun_out/ab_$2_base_$k.json 2>/dev/null; done
FETIGPU_NVCC_DEFINES="$1" python -c "from paper_1312_5653_b200 import build; build.build(force=True)"
for k in 1 2; do timeout 600 python bench.py --no-cpu-baseline --no-sweep --steps 30 > gpurun_out/ab_$2_var_$k.json 2>/dev/null; done
FETIGPU_NVCC_DEFINES="$1" FETIGPU_STEP_TIMES=1 timeout 300 python bench.py --no-cpu-baseline --no-sweep --steps 2 > /dev/null 2> gpurun_out/ab_$2_var_spans.txt
python -c "from paper_1312_5653_b200 import build; build.build(force=True)"
