set -x
mkdir -p gpurun_out
timeout 600 python scripts/dbg_balanced.py 1000 131072 262144 524288 1048576 > gpurun_out/dbg_bal.log 2>&1; echo rc=$? >> gpurun_out/dbg_bal.log
cat gpurun_out/dbg_bal.log
