python -m pytest tests/test_gpu_parity.py tests/test_gpu_edges.py tests/test_gpu_rs.py -q -x 2>&1 | tail -2
python scripts/prof_run.py 30 3 --check
python scripts/prof_run.py 30 3
python scripts/prof_run.py 30 3 --u64 --check
