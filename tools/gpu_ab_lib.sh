# A/B of two prebuilt libraries (paper_1312_5653_b200/_lib/libfetigpu_{base,new}.so), bench
# alternating base/new twice each; restores the new build.  Usage: bash tools/gpu_ab_lib.sh <tag>
mkdir -p gpurun_out
L=paper_1312_5653_b200/_lib
for k in 1 2; do
  for v in base new; do
    cp $L/libfetigpu_$v.so $L/libfetigpu.so
    timeout 600 python bench.py --no-cpu-baseline --no-sweep --steps 30 > gpurun_out/ab_$1_${v}_$k.json 2>/dev/null
  done
done
cp $L/libfetigpu_new.so $L/libfetigpu.so
