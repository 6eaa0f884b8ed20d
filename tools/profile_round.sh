#!/bin/bash
# Round evidence on one GPU: the bench line (no profiler), then the ncu launch list with DRAM
# bytes of one sort of the same workload, then a full ncu capture of the top kernels.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
CFG=${CFG:-H}
timeout 900 python bench.py --config $CFG > gpurun_out/bench_round_$CFG.json 2> gpurun_out/bench_round_$CFG.err
timeout 300 python tools/profile_run.py --config $CFG --sorts 1 > gpurun_out/plain_round.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -k regex:k_ --csv --log-file gpurun_out/launches_dram_$CFG.csv python tools/profile_run.py --config $CFG --sorts 1 \
  > gpurun_out/ncu_round.log 2>&1
if [ -n "$FULL" ]; then
  timeout 1500 ncu --set full --clock-control none --import-source on -k "regex:$FULL" -c ${FULLC:-4} \
    -o gpurun_out/full_round_$CFG -f python tools/profile_run.py --config $CFG --sorts 1 > gpurun_out/ncu_full_round.log 2>&1
fi
exit 0
