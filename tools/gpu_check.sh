#!/bin/bash
# One GPU session: parity tests, smoke, bench lines, optional ncu (never timed under ncu).
#   TESTS=1            run pytest -m gpu
#   BENCH_CONFIGS="H…"  bench lines (gpurun_out/bench_<cfg>.json)
#   NCU=1              launch list of one H sort (gpurun_out/launches_H.csv)
#   NCU_FULL="regex" NCU_COUNT=n   ncu --set full of the first n matching launches of one H sort
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
if [ -n "$TESTS" ]; then
  timeout ${TEST_TIMEOUT:-1200} python -m pytest tests -m gpu -x -q ${TEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
fi
for c in ${BENCH_CONFIGS}; do
  timeout 600 python bench.py --config $c --steps ${STEPS:-5} --warmup 3 ${BENCH_ARGS} > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
done
PCFG=${PROFILE_CONFIG:-H}
if [ -n "$NCU" ]; then
  timeout 300 python tools/profile_run.py --config $PCFG --sorts 1 > gpurun_out/plain_launch.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_$PCFG.csv python tools/profile_run.py --config $PCFG --sorts 1 > gpurun_out/ncu_launch.log 2>&1
fi
if [ -n "$NCU_FULL" ]; then
  timeout 300 python tools/profile_run.py --config $PCFG --sorts 1 > gpurun_out/plain_full.log 2>&1 && \
  timeout 1500 ncu --set full --clock-control none --import-source on -k "regex:$NCU_FULL" -c ${NCU_COUNT:-3} \
    -o gpurun_out/full_$PCFG -f python tools/profile_run.py --config $PCFG --sorts 1 > gpurun_out/ncu_full.log 2>&1
fi
exit 0
