python -m pytest tests/test_gpu_parity.py -q -x -k "host_entry or numpy_host or config1" 2>&1 | tail -2
python bench.py --steps 3 --no-cpu-baseline --e2e-steps 3 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e'], d['roofline']['stage_ms_per_step'])"
