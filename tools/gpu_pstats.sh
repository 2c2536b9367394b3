IPS4O_EXTRA_NVCC_FLAGS="-DIPS4O_PERM_STATS $EXTRA" python -m paper_2009_13569_b200.build --force > gpurun_out/build.log 2>&1 || exit 1
for a in tree digit; do echo "== $a"; python tools/prof_run.py --n 30 --reps 1 --algo $a --max-levels 2 2>&1 | tail -3; done
