# timing of several build variants: gpu_var.sh "<prof_run args>" "<flags A>" "<flags B>" ...
ARGS=$1; shift
for V in "$@"; do
  IPS4O_EXTRA_NVCC_FLAGS="$V" python -m paper_2009_13569_b200.build --force > gpurun_out/build_v.log 2>&1 || { echo "build failed: $V"; tail -5 gpurun_out/build_v.log; continue; }
  echo "variant: [$V]"
  timeout 300 python tools/prof_run.py $ARGS 2>&1 | grep -v "sorted ok" | tail -1
done
