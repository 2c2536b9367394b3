# dev iteration on one element type: gpu_dev.sh <dt> [extra nvcc flags...]; builds -DIPS4O_ONLY_DT=<dt>
DT=$1; shift
IPS4O_EXTRA_NVCC_FLAGS="-DIPS4O_ONLY_DT=$DT $*" python -m paper_2009_13569_b200.build > gpurun_out/build_dev.log 2>&1 || { tail -30 gpurun_out/build_dev.log; exit 1; }
timeout 600 python tools/dev_check.py --dt $DT ${DEV_ARGS} 2>&1 | tail -12
