mkdir -p gpurun_out
timeout 120 python scripts/prof_run.py 30 3 --u64 > gpurun_out/u64_stages.log 2>&1
timeout 120 python scripts/prof_run.py 29 3 --u64 >> gpurun_out/u64_stages.log 2>&1
timeout 300 python scripts/rs_run.py 30 3 >> gpurun_out/u64_stages.log 2>&1
cat gpurun_out/u64_stages.log
