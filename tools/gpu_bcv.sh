# base-case micro variants (u64 dev builds)
for V in "-DIPS4O_BC_HEVEC=0 -DIPS4O_BC_STCHG=0" "-DIPS4O_BC_HEVEC=1 -DIPS4O_BC_STCHG=0" "-DIPS4O_BC_HEVEC=1 -DIPS4O_BC_STCHG=1"; do
  IPS4O_EXTRA_NVCC_FLAGS="-DIPS4O_ONLY_DT=0 $V" python -m paper_2009_13569_b200.build > gpurun_out/build_v.log 2>&1 || { echo "build failed: $V"; tail -5 gpurun_out/build_v.log; continue; }
  echo "variant: [$V]"
  if [ "$V" = "-DIPS4O_BC_HEVEC=1 -DIPS4O_BC_STCHG=1" ]; then
    timeout 600 python tools/dev_check.py --dt 0 --n 30 --dists uniform_u64,twodup_u64 --reps 5 2>&1 | tail -3
  else
    timeout 300 python tools/dev_check.py --dt 0 --n 30 --no-check --dists uniform_u64,twodup_u64 --reps 5 2>&1 | tail -2
  fi
done
