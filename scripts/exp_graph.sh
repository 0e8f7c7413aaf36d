set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_graph.py -x -q > gpurun_out/pytest_graph.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_graph.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo rc=$?
tail -5 gpurun_out/pytest_graph.log; cat gpurun_out/bench.json
