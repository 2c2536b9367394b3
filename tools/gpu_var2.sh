# timing of several build variants over several inputs: gpu_var2.sh "<dist:algo ...>" "<flags A>" "<flags B>" ...
CASES=$1; shift
for V in "$@"; do
  IPS4O_EXTRA_NVCC_FLAGS="$V" python -m paper_2009_13569_b200.build --force > gpurun_out/build_v.log 2>&1 || { echo "build failed: $V"; tail -5 gpurun_out/build_v.log; continue; }
  for c in $CASES; do
    d=${c%%:*}; a=${c##*:}
    echo "variant: [$V] $d $a $(timeout 300 python tools/prof_run.py --n 30 --dist $d --algo $a --reps 2 2>&1 | tail -1 | cut -c1-400)"
  done
done
