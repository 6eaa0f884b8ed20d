#!/bin/bash
# One full ncu capture (source-level) of kernels matching $K (regex) in one host-driven sort of $CFG.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
export IPS4O_EAGER=1
timeout 300 python tools/profile_run.py --config ${CFG:-H} --sorts 1 > gpurun_out/plain_one.log 2>&1 && \
timeout 1500 ncu --set full --import-source on --clock-control none -k "regex:$K" -s ${SKIP:-0} -c ${COUNT:-1} \
  -o gpurun_out/${OUT:-one} -f python tools/profile_run.py --config ${CFG:-H} --sorts 1 > gpurun_out/ncu_one.log 2>&1
tail -3 gpurun_out/ncu_one.log
