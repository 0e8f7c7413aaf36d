# A/B: leaf apply with / without L2 eviction hints (sk_debug_set(7, v)), then the parity tests
set -x
mkdir -p gpurun_out
for v in 0 1 0 1; do timeout 300 python scripts/prof_run.py 30 5 7=$v --check; done > gpurun_out/l2pol.jsonl 2>gpurun_out/l2pol.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:leaf_apply_v3 -s 1 -c 1 -o gpurun_out/leafpol -f python scripts/prof_run.py 30 1 > gpurun_out/ncu_leafpol.log 2>&1; echo rc=$?
timeout 1200 python -m pytest tests -m gpu -x -q -k "leaf or fisher or parity or fullsize" > gpurun_out/pytest_sub.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_sub.log
cat gpurun_out/l2pol.jsonl; tail -3 gpurun_out/pytest_sub.log
