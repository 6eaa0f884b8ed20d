#!/bin/bash
# Round evidence on one GPU: the bench line (no profiler), then the ncu launch list with DRAM
# bytes of one sort of the same workload, then a full ncu capture of the top kernels (with
# branch-divergence counters).  ncu cannot profile kernels inside graphs with conditional nodes,
# so the captures run the same loop host-driven (IPS4O_EAGER=1: same kernels, same grids).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
CFG=${CFG:-H}
TAG=${TAG:-r02}
timeout 900 python bench.py --config $CFG > gpurun_out/${TAG}_bench_$CFG.json 2> gpurun_out/${TAG}_bench_$CFG.err
export IPS4O_EAGER=1
timeout 300 python tools/profile_run.py --config $CFG --sorts 1 > gpurun_out/plain_round.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -k regex:k_ --csv --log-file gpurun_out/${TAG}_launches_$CFG.csv python tools/profile_run.py --config $CFG --sorts 1 \
  > gpurun_out/ncu_round.log 2>&1
if [ -n "$FULL" ]; then
  timeout 1800 ncu --set full --metrics smsp__sass_branch_targets.sum,smsp__sass_branch_targets_threads_divergent.sum,smsp__sass_branch_targets_threads_uniform.sum \
    --clock-control none --import-source on -k "regex:$FULL" -c ${FULLC:-6} \
    -o gpurun_out/${TAG}_full_$CFG -f python tools/profile_run.py --config $CFG --sorts 1 > gpurun_out/ncu_full_round.log 2>&1
fi
exit 0
