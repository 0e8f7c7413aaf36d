set -x
mkdir -p gpurun_out
timeout 200 python scripts/dbg_balanced.py 33 100 1000 1025 2049 4096 16384 65536 100000 131072 > gpurun_out/dbg_bal.log 2>&1; echo rc=$? >> gpurun_out/dbg_bal.log
cat gpurun_out/dbg_bal.log
timeout 900 python -m pytest tests/test_gpu_balanced.py -x -q -s --timeout 300 > gpurun_out/pytest_bal.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_bal.log
grep "balanced n=" gpurun_out/pytest_bal.log | tail -14; tail -4 gpurun_out/pytest_bal.log
