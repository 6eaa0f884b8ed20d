cd "${GRAFT_REPO_ROOT:-/root/repo}"
VARIANTS="${V:-celltile celltile4 c3t512}" CFG="${C:-H C2a C3_eightdup C4}" STEPS=10 bash tools/variants.sh > /dev/null 2>&1
if [ -n "$EDUP" ]; then
export IPS4O_EAGER=1
timeout 300 python tools/profile_run.py --config C3_eightdup --sorts 1 > gpurun_out/plain_e.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_ --csv \
    --log-file gpurun_out/launches_C3_eightdup.csv python tools/profile_run.py --config C3_eightdup --sorts 1 > gpurun_out/ncu_e.log 2>&1
fi
cat gpurun_out/variants.log
