# base-case parking A/B (u64 dev builds): PARK=0 vs PARK=1, with correctness check on the PARK=1 build
for V in "-DIPS4O_BC_PARK=0" "-DIPS4O_BC_PARK=1"; do
  IPS4O_EXTRA_NVCC_FLAGS="-DIPS4O_ONLY_DT=0 $V" python -m paper_2009_13569_b200.build > gpurun_out/build_v.log 2>&1 || { echo "build failed: $V"; tail -5 gpurun_out/build_v.log; continue; }
  echo "variant: [$V]"
  grep -A2 "basecase_kernelILi0ELb0" gpurun_out/build_v.log | grep -E "registers|spill" | head -2
  if [ "$V" = "-DIPS4O_BC_PARK=1" ]; then
    timeout 600 python tools/dev_check.py --dt 0 --n 30 --dists uniform_u64,twodup_u64,zipf_u64 --reps 4 2>&1 | tail -5
  else
    timeout 300 python tools/dev_check.py --dt 0 --n 30 --no-check --dists uniform_u64,twodup_u64,zipf_u64 --reps 4 2>&1 | tail -4
  fi
done
