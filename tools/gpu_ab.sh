# A/B: default build (parity + timing), then a build with $VARIANT flags (timing only)
bash tools/gpu_quick.sh
IPS4O_EXTRA_NVCC_FLAGS="$VARIANT" python -m paper_2009_13569_b200.build --force > gpurun_out/build_b.log 2>&1 || { tail -5 gpurun_out/build_b.log; exit 1; }
echo "variant: $VARIANT"
timeout 300 python tools/prof_run.py --n 30 --reps 3 --check 2>&1 | tail -2
