# whole GPU suite + stage timings + every config with the warp-specialised decode
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/ws_pytest_all.log 2>&1; echo "pytest rc=$?" >> gpurun_out/ws_pytest_all.log
tail -3 gpurun_out/ws_pytest_all.log
for n in 20 26 30 30 31; do timeout 300 python scripts/prof_run.py $n 5 --check; done > gpurun_out/ws_stages.log 2>&1
timeout 900 python scripts/configs_timing.py > gpurun_out/ws_configs.jsonl 2>&1
cat gpurun_out/ws_stages.log gpurun_out/ws_configs.jsonl
