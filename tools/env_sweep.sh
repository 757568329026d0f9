#!/bin/bash
# Runs bench.py (no sweep / cpu baseline) once per environment setting given as arguments;
# prints value, e2e and per-class ms per step.  Usage: tools/env_sweep.sh "A=1 B=2" "A=3" ...
for cfg in "$@"; do
  echo "== $cfg"
  env $cfg timeout 300 python bench.py --no-sweep --no-cpu-baseline --steps 10 2>&1 | python -c "
import json, sys
for l in sys.stdin:
    try:
        d = json.loads(l)
    except Exception:
        print(l.rstrip()[:300]); continue
    print(round(d['value'], 2), round(d['e2e']['value'], 2), round(d['roofline']['frac'], 3),
          {k: round(v['ms_per_step'], 3) for k, v in d['config']['kernel_ms_per_step'].items()})
"
done
