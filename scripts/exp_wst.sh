# flag-synchronised warp-specialised decode: epochs of 16 / 32 / 64 trips
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edges.py tests/test_gpu_rs.py -x -q -m gpu > gpurun_out/ws_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/ws_pytest.log
tail -2 gpurun_out/ws_pytest.log
for v in f16 f32 f64 t32; do SK_LIB_PATH=build/variants/$v.so timeout 300 python scripts/prof_run.py 20 20 --check; echo "variant=$v n=2^20"; done > gpurun_out/wst.log 2>&1
for v in f16 f32 f64 t32; do SK_LIB_PATH=build/variants/$v.so timeout 300 python scripts/prof_run.py 30 5 --check; echo "variant=$v n=2^30"; done >> gpurun_out/wst.log 2>&1
for v in f16 f32 f64; do SK_LIB_PATH=build/variants/$v.so timeout 300 python scripts/prof_run.py 31 3; echo "variant=$v n=2^31"; done >> gpurun_out/wst.log 2>&1
for v in f16 f32 f64; do SK_LIB_PATH=build/variants/$v.so timeout 600 python scripts/configs_timing.py 2>&1 | grep "config\": \"5"; echo "variant=$v configs"; done >> gpurun_out/wst.log 2>&1
cat gpurun_out/wst.log
