# round-2 final check: all GPU tests, smoke, the bench, every config, ncu of the speculative decode
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q --timeout 900 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo rc=$?
timeout 900 python scripts/configs_timing.py > gpurun_out/configs.jsonl 2> gpurun_out/configs.err; echo rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:leaf_decode_spec -s 1 -c 1 -o gpurun_out/spec -f python scripts/prof_run.py 20 1 > gpurun_out/ncu_spec.log 2>&1; echo rc=$?
tail -3 gpurun_out/pytest_gpu.log; cat gpurun_out/smoke.log; cat gpurun_out/bench.json; cat gpurun_out/configs.jsonl
