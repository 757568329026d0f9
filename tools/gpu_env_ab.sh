# A/B of an environment switch on the config-2 bench: bash tools/gpu_env_ab.sh VAR=value
mkdir -p gpurun_out
for r in 1 2; do
timeout 600 python bench.py --no-cpu-baseline --no-sweep > gpurun_out/eab_base$r.json 2>/dev/null
env "$@" timeout 600 python bench.py --no-cpu-baseline --no-sweep > gpurun_out/eab_var$r.json 2>gpurun_out/eab_var$r.err
done
