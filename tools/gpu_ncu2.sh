# ncu --set full of classify + permute, both levels, of the 2nd 2^30 u64 sort (host-launched rounds)
TAG=$1
IPS4O_EXTRA_NVCC_FLAGS="-DIPS4O_ONLY_DT=0" python -m paper_2009_13569_b200.build > gpurun_out/build_ncu.log 2>&1 || exit 1
cp paper_2009_13569_b200/lib/libips4o.so gpurun_out/libips4o_$TAG.so
IPS4O_HOST_LEVELS=1 timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"classify_v2|permute_kernel" -s 4 -c 4 \
  -o gpurun_out/ncu_$TAG python tools/prof_run.py --n 30 --reps 2 > gpurun_out/ncu_$TAG.log 2>&1
echo ncu_rc=$?
