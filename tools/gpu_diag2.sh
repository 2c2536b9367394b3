# ncu source-level capture of the u64 base case (2^30) + classify L1/L2 + permute (full set)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
IPS4O_HOST_LEVELS=1 timeout 1200 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k regex:"basecase_kernel<0, false>" -s 1 -c 1 -o gpurun_out/ncu_bc python tools/prof_run.py --n 30 --reps 2 > gpurun_out/ncu_bc.log 2>&1; echo ncu_rc=$?
if [ ! -f gpurun_out/ncu_bc.ncu-rep ]; then
IPS4O_HOST_LEVELS=1 timeout 1200 ncu --set full --clock-control none --import-source on -k regex:basecase_kernel -s 6 -c 4 \
  -o gpurun_out/ncu_bc python tools/prof_run.py --n 30 --reps 2 > gpurun_out/ncu_bc2.log 2>&1; echo ncu2_rc=$?
fi
ncu -i gpurun_out/ncu_bc.ncu-rep --page source --csv --print-source sass > gpurun_out/ncu_bc_sass.csv 2>gpurun_out/exp.err; echo exp_rc=$?
ncu -i gpurun_out/ncu_bc.ncu-rep --page raw --csv > gpurun_out/ncu_bc_raw.csv 2>>gpurun_out/exp.err
IPS4O_HOST_LEVELS=1 timeout 1500 ncu --set full --clock-control none -k regex:"classify_v2|permute_kernel" -s 4 -c 4 \
  -o gpurun_out/ncu_cp python tools/prof_run.py --n 30 --reps 2 > gpurun_out/ncu_cp.log 2>&1; echo ncu3_rc=$?
ncu -i gpurun_out/ncu_cp.ncu-rep --page raw --csv > gpurun_out/ncu_cp_raw.csv 2>>gpurun_out/exp.err
rm -f gpurun_out/*.ncu-rep
