# A/B: decode with running pointer (decptr) vs step-index addresses (decidx)
set -x
for v in decptr decidx decptr decidx; do SK_LIB_PATH=build/variants/$v.so timeout 300 python scripts/prof_run.py 30 3 --check; echo "variant=$v"; done > gpurun_out/decidx.log 2>&1
for v in decptr decidx; do SK_LIB_PATH=build/variants/$v.so timeout 300 python scripts/prof_run.py 20 5; echo "variant=$v"; done >> gpurun_out/decidx.log 2>&1
cat gpurun_out/decidx.log | grep -v "^+"
