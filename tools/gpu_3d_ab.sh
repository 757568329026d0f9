# config-4 bench under environment variants: bash tools/gpu_3d_ab.sh "VAR=a" "VAR=b" ...
mkdir -p gpurun_out
timeout 900 python bench.py --config 4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ab3_base.json 2>/dev/null
i=0
for v in "$@"; do i=$((i+1)); env $v timeout 900 python bench.py --config 4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ab3_v$i.json 2>/dev/null; done
