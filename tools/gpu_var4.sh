# variants of a one-dtype dev build: gpu_var4.sh <dt> <log2 n> <dists> "<flags A>" "<flags B>" ...
DT=$1; N=$2; DISTS=$3; shift 3
for V in "$@"; do
  IPS4O_EXTRA_NVCC_FLAGS="-DIPS4O_ONLY_DT=$DT $V" python -m paper_2009_13569_b200.build > gpurun_out/build_v.log 2>&1 || { echo "build failed: $V"; tail -5 gpurun_out/build_v.log; continue; }
  echo "variant: [$V]"
  timeout 300 python tools/dev_check.py --dt $DT --n $N --no-check --dists $DISTS --reps 3 2>&1 | tail -2
done
