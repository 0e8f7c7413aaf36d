python -m pytest tests/test_gpu_parity.py tests/test_gpu_edges.py -q -x 2>&1 | tail -2
python scripts/prof_batched.py 65536 4096 5
python scripts/prof_batched.py 65536 4096 5 5=1
python scripts/prof_batched.py 32768 8192 5
python scripts/prof_batched.py 32768 8192 5 5=1
python scripts/prof_run.py 30 3 --check
