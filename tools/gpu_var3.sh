# variants of the u64 dev build: gpu_var3.sh "<flags A>" "<flags B>" ...  (2^30 uniform + rootdup timing)
for V in "$@"; do
  IPS4O_EXTRA_NVCC_FLAGS="-DIPS4O_ONLY_DT=0 $V" python -m paper_2009_13569_b200.build > gpurun_out/build_v.log 2>&1 || { echo "build failed: $V"; tail -5 gpurun_out/build_v.log; continue; }
  echo "variant: [$V]"
  timeout 300 python tools/dev_check.py --no-check --dists uniform_u64,rootdup_u64 --reps 3 2>&1 | tail -2
done
