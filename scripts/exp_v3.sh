python scripts/prof_run.py 30 3 --check
SK_LIB_PATH=build/variants/sstop.so python scripts/prof_run.py 30 3 --check
SK_LIB_PATH=build/variants/noknob.so python scripts/prof_run.py 30 3 --check
python scripts/prof_run.py 30 3
SK_LIB_PATH=build/variants/sstop.so python scripts/prof_run.py 30 3
SK_LIB_PATH=build/variants/noknob.so python scripts/prof_run.py 30 3
