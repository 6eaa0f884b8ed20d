#!/bin/bash
# Tuning sweep on the GPU over environment settings of the default library:
#   ENVS="IPS4O_WAVE=0 IPS4O_WAVE=8388608,IPS4O_WAVE_STRIPE=32768"  CFG="H C4"  [VERIFY=1]
# (comma-separated assignments inside one setting)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
out=gpurun_out/envsweep.log
: > $out
nv="--no-verify"; [ -n "$VERIFY" ] && nv=""
for e in $ENVS; do
  for c in ${CFG:-H}; do
    env $(echo $e | tr ',' ' ') timeout 300 python bench.py --config $c --steps ${STEPS:-10} --warmup 3 --no-cpu-baseline --e2e-steps 0 $nv > /tmp/v.json 2>/tmp/v.err
    python - "$e" "$c" >> $out <<'PY'
import json, sys
try:
    d = json.loads(open('/tmp/v.json').read().strip().splitlines()[-1])
    k = {a: round(b, 3) for a, b in d['kernels_ms_per_step'].items()}
    print(sys.argv[1], sys.argv[2], round(d['ms_per_step'], 3), 'ms', round(d['value'], 2), d['unit'], 'verified' if d.get('verified') else 'unverified', 'batches', d['sort_stats'].get('batches'), k)
except Exception as e:
    print(sys.argv[1], sys.argv[2], 'FAILED', e, open('/tmp/v.err').read()[-400:].replace('\n', ' | '))
PY
  done
done
cat $out
