#!/bin/bash
# Tuning sweep on the GPU: bench one config with each built variant library (IPS4O_LIB).
#   VARIANTS="k3s2 k3s8"  CFG=H  [TESTS=1 runs pytest -m gpu on the default library first]
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
if [ -n "$TESTS" ]; then
  timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
fi
: > gpurun_out/variants.log
for v in default $VARIANTS; do
  if [ "$v" = default ]; then lib=paper_1705_02257_b200/libips4o.so; else lib=paper_1705_02257_b200/libips4o_$v.so; fi
  for c in ${CFG:-H}; do
    IPS4O_LIB=$PWD/$lib timeout 300 python bench.py --config $c --steps ${STEPS:-5} --warmup 3 --no-cpu-baseline --e2e-steps 0 ${NOVERIFY:+--no-verify} > /tmp/v.json 2>/tmp/v.err
    python - "$v" "$c" >> gpurun_out/variants.log <<'PY'
import json, sys
try:
    d = json.loads(open('/tmp/v.json').read().strip().splitlines()[-1])
    k = {a: round(b, 3) for a, b in d['kernels_ms_per_step'].items()}
    print(sys.argv[1], sys.argv[2], round(d['ms_per_step'], 3), 'ms', round(d['value'], 2), d['unit'], 'ok' if d.get('verified') else 'BAD', k, 'lv', d['sort_stats']['levels'], 'b', d['sort_stats']['batches'], d['sort_stats']['base_tasks_by_class'], 'fb', d['sort_stats']['base_fallback_tasks'])
except Exception as e:
    print(sys.argv[1], sys.argv[2], 'FAILED', e, open('/tmp/v.err').read()[-300:].replace('\n', ' | '))
PY
  done
done
cat gpurun_out/variants.log
