for v in "$@"; do
IPS4O_EXTRA_NVCC_FLAGS="$v" python -m paper_2009_13569_b200.build --force > gpurun_out/build.log 2>&1 || exit 1
for a in digit tree; do echo "== $v $a"; python tools/prof_run.py --n 30 --reps 2 --algo $a --max-levels 2 2>&1 | grep -v "^0 " | cut -c1-200; done
done
