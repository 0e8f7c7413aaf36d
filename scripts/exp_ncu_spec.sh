mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:leaf_decode_spec -s 1 -c 1 -o gpurun_out/spec -f python scripts/prof_run.py 20 1 > gpurun_out/ncu_spec.log 2>&1; echo rc=$?
