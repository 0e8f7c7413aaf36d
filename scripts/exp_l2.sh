for n in 22 23 24 25 26 27 28; do python scripts/prof_run.py $n 10; done
