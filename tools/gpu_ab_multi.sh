# bench under several environment settings.  Usage: bash tools/gpu_ab_multi.sh <tag> "ENV1=.." "ENV2=.." ...
mkdir -p gpurun_out
tag=$1; shift
i=0
for e in "$@"; do
  i=$((i+1))
  env $e timeout 600 python bench.py --no-cpu-baseline --no-sweep --steps 30 > gpurun_out/abm_${tag}_$i.json 2>/dev/null
  python - "$e" gpurun_out/abm_${tag}_$i.json <<'P'
import json,sys
try:
    d=json.load(open(sys.argv[2])); print(sys.argv[1], round(d['value'],2), round(d['e2e']['value'],2), d['roofline'].get('in_graph',{}).get('spans_us'))
except Exception as e: print(sys.argv[1], 'ERR', e)
P
done
