#!/bin/bash
# single-CTA tier threshold vs input size (tools only)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
for mm in ${MMS:-0 24576}; do
  for n in 4194304 8388608 16777216 33554432; do
    IPS4O_MEDIUM_MAX=$mm timeout 300 python bench.py --config H --n $n --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-verify --no-kernel-events > /tmp/v.json 2>/tmp/v.err
    python -c "
import json
d=json.loads(open('/tmp/v.json').read().strip().splitlines()[-1]); st=d['sort_stats']
print('$mm', '$n', round(d['ms_per_step'],3), 'med', st['medium_tasks'], 'levels', st['levels'])" || tail -2 /tmp/v.err
  done
done
