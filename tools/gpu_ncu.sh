# ncu --set full of the classify (L1, L2) and base-case launches of the 2nd 2^N u64 sort
# (host-launched rounds so that ncu sees every kernel): gpu_ncu.sh <tag> [N] [extra nvcc flags]
TAG=$1; N=${2:-30}; shift; shift
IPS4O_EXTRA_NVCC_FLAGS="-DIPS4O_ONLY_DT=0 $*" python -m paper_2009_13569_b200.build > gpurun_out/build_ncu.log 2>&1 || exit 1
timeout 300 python tools/prof_run.py --n $N --reps 2 > gpurun_out/prof_plain_$TAG.log 2>&1 || { cat gpurun_out/prof_plain_$TAG.log; exit 1; }
IPS4O_HOST_LEVELS=1 timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"basecase|classify_v2" -s 4 -c 3 \
  -o gpurun_out/ncu_$TAG python tools/prof_run.py --n $N --reps 2 > gpurun_out/ncu_$TAG.log 2>&1
echo ncu_rc=$?
tail -3 gpurun_out/ncu_$TAG.log
