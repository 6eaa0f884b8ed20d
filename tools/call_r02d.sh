cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/pytest_parity.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_parity.log
VARIANTS="${V}" CFG="${C:-H C2b C3_eightdup C3_twodup C3_rootdup C4}" STEPS=10 bash tools/variants.sh > /dev/null 2>&1
tail -3 gpurun_out/pytest_parity.log
cat gpurun_out/variants.log
