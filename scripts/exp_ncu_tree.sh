mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:merge_tree_kernel -s 20 -c 1 -o gpurun_out/tree -f python scripts/prof_run.py 30 1 > gpurun_out/ncu_tree.log 2>&1
tail -1 gpurun_out/ncu_tree.log
