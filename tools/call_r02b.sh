cd "${GRAFT_REPO_ROOT:-/root/repo}"
VARIANTS="leaf8k leaf8k512 leaf8k768" CFG="H C2a C3_eightdup" STEPS=10 bash tools/variants.sh > /dev/null 2>&1
export IPS4O_EAGER=1
timeout 300 python tools/profile_run.py --config H --sorts 1 > gpurun_out/plain_full.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k "regex:k_base_cell" -c 8 \
    -o gpurun_out/full_base_H -f python tools/profile_run.py --config H --sorts 1 > gpurun_out/ncu_full.log 2>&1
ls -la gpurun_out
