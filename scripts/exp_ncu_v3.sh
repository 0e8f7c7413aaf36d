mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:leaf_apply_v3 -s 1 -c 1 -o gpurun_out/leafv3c -f python scripts/prof_run.py 30 1 > gpurun_out/ncu_v3.log 2>&1
tail -1 gpurun_out/ncu_v3.log
