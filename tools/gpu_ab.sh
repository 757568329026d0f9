# A/B/C.. of experiment builds: the default library and FETIGPU_LIB=<variant .so>, alternated
mkdir -p gpurun_out
for r in 1 2; do
timeout 600 python bench.py --no-cpu-baseline --no-sweep > gpurun_out/ab_base$r.json 2>/dev/null
for v in "$@"; do
FETIGPU_LIB=paper_1312_5653_b200/_lib/libfetigpu_$v.so timeout 600 python bench.py --no-cpu-baseline --no-sweep > gpurun_out/ab_$v$r.json 2>/dev/null
done
done
