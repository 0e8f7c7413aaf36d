python -m pytest tests/test_gpu_parity.py -q -x -k "leaf_apply_variants or small or config1 or config2" 2>&1 | tail -2
for s in 1 2 3 4 5 6 7 10 11 99; do python scripts/prof_run.py 30 3 1=$s; done
python scripts/prof_run.py 30 3 5=10 --check
python scripts/prof_run.py 30 3 5=10 1=7
python scripts/prof_run.py 30 3 --check
