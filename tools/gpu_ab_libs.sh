# A/B of prebuilt libraries paper_1312_5653_b200/_lib/libfetigpu_<name>.so: bench each, twice, alternating.
# Usage: bash tools/gpu_ab_libs.sh <tag> <name1> <name2> ...   (the first one is restored at the end)
mkdir -p gpurun_out
L=paper_1312_5653_b200/_lib
tag=$1; shift
for k in 1 2; do
  for v in "$@"; do
    cp $L/libfetigpu_$v.so $L/libfetigpu.so
    timeout 600 python bench.py --no-cpu-baseline --no-sweep --steps 30 > gpurun_out/abl_${tag}_${v}_$k.json 2>/dev/null
    python - $v gpurun_out/abl_${tag}_${v}_$k.json <<'P'
import json,sys
try:
    d=json.load(open(sys.argv[2])); print(sys.argv[1], round(d['value'],2), round(d['e2e']['value'],2), d['roofline'].get('in_graph',{}).get('spans_us'))
except Exception as e: print(sys.argv[1], 'ERR', e)
P
  done
done
cp $L/libfetigpu_$1.so $L/libfetigpu.so
