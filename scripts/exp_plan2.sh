# rounds' plans on two side streams (knob 10): parity + graph tests, then A/B stage timings
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_graph.py tests/test_gpu_edges.py tests/test_gpu_multiprocess.py -x -q -m gpu --timeout 300 > gpurun_out/plan2_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/plan2_pytest.log
tail -5 gpurun_out/plan2_pytest.log
for rep in 1 2; do for k in 1 2; do timeout 120 python scripts/prof_run.py 30 5 10=$k --check; done; done > gpurun_out/plan2_stages.log 2>&1
for k in 1 2; do timeout 120 python scripts/prof_run.py 28 5 10=$k; done >> gpurun_out/plan2_stages.log 2>&1
cat gpurun_out/plan2_stages.log
