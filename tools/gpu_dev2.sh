# dev_check (u64) + base-case phase timing
bash tools/gpu_dev.sh 0 "$@"
IPS4O_EXTRA_NVCC_FLAGS="-DIPS4O_ONLY_DT=0 -DIPS4O_PHASE_TIMING $*" python -m paper_2009_13569_b200.build >/dev/null 2>&1 && timeout 120 python tools/prof_run.py --n 30 --reps 2 2>&1 | grep cycles | tail -1
