set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_balanced.py -x -q -s --timeout 120 > gpurun_out/pytest_bal.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_bal.log
grep "balanced n=" gpurun_out/pytest_bal.log | tail -30; tail -15 gpurun_out/pytest_bal.log
