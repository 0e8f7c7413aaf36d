python scripts/prof_run.py 30 3 --check
python scripts/prof_run.py 30 3 1=13 --check
python scripts/prof_run.py 30 3
python scripts/prof_run.py 30 3 1=13
