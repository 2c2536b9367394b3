# ncu --set full of classify L2, permute L2 and the base case of the 2nd 2^30 u64 sort (host-launched rounds)
IPS4O_HOST_LEVELS=1 timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"classify_v2|permute_kernel|basecase_kernel<0, 0>" -s 8 -c 3 \
  -o gpurun_out/ncu_full_r2c python tools/prof_run.py --n 30 --reps 2 > gpurun_out/ncu_full_r2c.log 2>&1; echo full_rc=$?
