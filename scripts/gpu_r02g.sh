# round-2 final-code measurement set: bench, reference arm, launch list, ncu of the three top kernels
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo rc=$?
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/ncu.log 2>&1; echo rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:merge_tree_kernel -s 20 -c 1 -o gpurun_out/tree -f python scripts/prof_run.py 30 1 > gpurun_out/ncu_tree.log 2>&1; echo rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:leaf_apply_v3 -s 1 -c 1 -o gpurun_out/leaf -f python scripts/prof_run.py 30 1 > gpurun_out/ncu_leaf.log 2>&1; echo rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:leaf_decode_ws -s 1 -c 1 -o gpurun_out/dec -f python scripts/prof_run.py 30 1 > gpurun_out/ncu_dec.log 2>&1; echo rc=$?
cat gpurun_out/smoke.log; cat gpurun_out/bench.json; cat gpurun_out/bench_ref.json
