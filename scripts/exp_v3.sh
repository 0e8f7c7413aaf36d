python -m pytest tests/test_gpu_parity.py -q -x -k "leaf_apply_variants or small or config1 or config2" 2>&1 | tail -2
for s in 4 5 99; do python scripts/prof_run.py 30 3 1=$s; done
python scripts/prof_run.py 30 3 --check
