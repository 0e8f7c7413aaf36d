# warp-per-leaf speculative decode: parity tests, then stage timings with the leaf-count threshold on / off
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edges.py tests/test_gpu_rs.py tests/test_gpu_graph.py -x -q -m gpu --timeout 120 > gpurun_out/spec_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/spec_pytest.log
tail -15 gpurun_out/spec_pytest.log
if grep -q "pytest rc=0" gpurun_out/spec_pytest.log; then
for n in 20 22 24 26 27 28; do
  for k in 0 1000000; do timeout 60 python scripts/prof_run.py $n 5 8=$k --check; done
done > gpurun_out/spec_stages.log 2>&1
cat gpurun_out/spec_stages.log
fi
