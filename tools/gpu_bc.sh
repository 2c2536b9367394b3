IPS4O_EXTRA_NVCC_FLAGS=-DIPS4O_PHASE_TIMING python -m paper_2009_13569_b200.build --force > gpurun_out/build.log 2>&1 || exit 1
timeout 300 python tools/prof_run.py --n 30 --reps 2 2>&1 | grep -v "cycles: zero 0 " | tail -4
python -m paper_2009_13569_b200.build --force > gpurun_out/build.log 2>&1 || exit 1
bash tools/gpu_prof1.sh basecase 4
