mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py --no-cpu-baseline --no-sweep > gpurun_out/bench_v17.json 2> gpurun_out/bench_v17.err; echo "bench rc=$?" >> gpurun_out/bench_v17.err
for kb in 0 32 128; do FETIGPU_PAIR_PF_KB=$kb timeout 600 python bench.py --no-cpu-baseline --no-sweep --steps 20 > gpurun_out/bench_v17_pf$kb.json 2>/dev/null; done
FETIGPU_NO_PAIR=1 timeout 600 python bench.py --no-cpu-baseline --no-sweep --steps 20 > gpurun_out/bench_v17_nopair.json 2>/dev/null
