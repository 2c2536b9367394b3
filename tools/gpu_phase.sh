# base-case phase timing (clock64 per phase, CTA 0), 2^30 u64
IPS4O_EXTRA_NVCC_FLAGS=-DIPS4O_PHASE_TIMING python -m paper_2009_13569_b200.build --force > gpurun_out/build.log 2>&1 || exit 1
timeout 300 python tools/prof_run.py --n 30 --reps 2 2>&1 | tail -12
