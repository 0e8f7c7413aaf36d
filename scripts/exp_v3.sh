python scripts/prof_run.py 30 3 --check
for v in scat8 quad4; do SK_LIB_PATH=build/variants/$v.so python scripts/prof_run.py 30 3 --check; done
for v in scat8 quad4; do SK_LIB_PATH=build/variants/$v.so python scripts/prof_run.py 30 3 1=4; done
python scripts/prof_run.py 30 3 1=4
