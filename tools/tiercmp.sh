#!/bin/bash
# Single-CTA tier threshold sweep (IPS4O_MEDIUM_MAX) over the configs (tools only).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
for mm in ${MMS:-0 65536 131072}; do
  for cfg in ${CFGS:-H C3_rootdup C3_twodup C3_eightdup C4}; do
    IPS4O_MEDIUM_MAX=$mm timeout 300 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-verify > /tmp/v.json 2>/tmp/v.err
    python -c "
import json,sys
d=json.loads(open('/tmp/v.json').read().strip().splitlines()[-1]); st=d['sort_stats']
print('$mm', '$cfg', round(d['ms_per_step'],3), 'med', st['medium_tasks'], st['medium_partitions'], st['medium_marks'], 'levels', st['levels'], 'batches', st['batches'], 'mcta_ms', round(d['kernels_ms_per_step'].get('medium_cta',0),3))" || tail -3 /tmp/v.err
  done
done
