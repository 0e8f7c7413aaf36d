# leaf-apply phase timing: cumulative stage time with the pipeline cut after phase k
for v in 1 0; do for s in 1 2 3 4 5 6 99; do
  python scripts/prof_run.py 30 3 5=$v 1=$s
done; done
python scripts/prof_run.py 30 3 --check
