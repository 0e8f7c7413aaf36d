# cumulative leaf-apply time with the pipeline cut after phase k (sk_debug_set(1, k)), 2^30 u32
set -x
mkdir -p gpurun_out
for k in 1 2 3 4 5 6 7 99; do timeout 300 python scripts/prof_run.py 30 3 1=$k; done > gpurun_out/leafphases.jsonl 2> gpurun_out/leafphases.err
cat gpurun_out/leafphases.jsonl
