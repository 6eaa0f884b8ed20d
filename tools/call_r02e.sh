# Final evidence of the round: full GPU suite, smoke, the H bench line + ncu launch list + full
# capture (tools/profile_round.sh), then every configuration (tools/variants.sh).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
TAG=r02 CFG=H FULL="k_classify|k_permute_tma|k_base_cell" FULLC=12 bash tools/profile_round.sh
VARIANTS="" CFG="H C1 C2a C2b C3_rootdup C3_twodup C3_eightdup C3_almostsorted C3_reversesorted C3_zeros F3_sorted F3_ones C4 C4_kv C5 F3_pair_f64 F3_quartet" STEPS=10 bash tools/variants.sh > /dev/null 2>&1
tail -3 gpurun_out/pytest_gpu.log; tail -1 gpurun_out/smoke.log; cat gpurun_out/variants.log
