# A/B: leaf decode variants (sk_debug_set 8: 0 single-warp lanes, 1 warp-specialised, 2 + lookahead)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edges.py tests/test_gpu_rs.py -x -q -m gpu > gpurun_out/ws_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/ws_pytest.log
tail -3 gpurun_out/ws_pytest.log
for v in ${VARS:-1 2 1 2}; do timeout 300 python scripts/prof_run.py 30 5 8=$v --check; echo "variant=$v"; done > gpurun_out/ws.log 2>&1
for v in ${VARS:-1 2}; do timeout 300 python scripts/prof_run.py 20 20 8=$v --check; echo "variant=$v n=2^20"; done >> gpurun_out/ws.log 2>&1
cat gpurun_out/ws.log
