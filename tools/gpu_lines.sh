# ncu source-level captures (SASS csv) of the u64 base case and the level-2 classification at 2^30
python -c "import paper_2009_13569_b200 as p; p.load()" || exit 1
IPS4O_HOST_LEVELS=1 timeout 1200 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k regex:"basecase_kernel<0, false>" -s 1 -c 1 -o /tmp/ncu_bc python tools/prof_run.py --n 30 --reps 2 > gpurun_out/ncu_bc.log 2>&1; echo ncu_rc=$?
ncu -i /tmp/ncu_bc.ncu-rep --page source --csv --print-source sass > gpurun_out/ncu_bc_sass.csv 2>gpurun_out/exp.err; echo exp_rc=$?
IPS4O_HOST_LEVELS=1 timeout 1200 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k regex:"classify_v2_kernel<0, 0>" -s 1 -c 1 -o /tmp/ncu_cl python tools/prof_run.py --n 30 --reps 2 > gpurun_out/ncu_cl.log 2>&1; echo ncu2_rc=$?
ncu -i /tmp/ncu_cl.ncu-rep --page source --csv --print-source sass > gpurun_out/ncu_cl_sass.csv 2>>gpurun_out/exp.err; echo exp2_rc=$?
ls -la gpurun_out/*.csv
