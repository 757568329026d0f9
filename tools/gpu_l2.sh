mkdir -p gpurun_out
python -c "from paper_1312_5653_b200 import build; build.build()"
timeout 600 python bench.py --no-cpu-baseline --no-sweep > gpurun_out/l2_off.json 2>/dev/null
FETIGPU_L2_PERSIST=1 timeout 600 python bench.py --no-cpu-baseline --no-sweep > gpurun_out/l2_on.json 2> gpurun_out/l2_on.err
timeout 600 python bench.py --no-cpu-baseline --no-sweep > gpurun_out/l2_off2.json 2>/dev/null
