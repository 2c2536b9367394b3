# EightDup level structure + ncu source-level capture of the u64 base case (2^30)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 600 python tools/exp/eightdup_levels.py eightdup_u64 30 > gpurun_out/eightdup_levels.log 2>&1; echo diag_rc=$?
timeout 300 python tools/rounds.py eightdup_u64 30 > gpurun_out/eightdup_rounds.log 2>&1
IPS4O_HOST_LEVELS=1 timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"basecase_kernel<0, 0>" -s 1 -c 1 \
  -o gpurun_out/ncu_bc python tools/prof_run.py --n 30 --reps 2 > gpurun_out/ncu_bc.log 2>&1; echo ncu_rc=$?
ncu -i gpurun_out/ncu_bc.ncu-rep --page source --csv --print-source sass > gpurun_out/ncu_bc_sass.csv 2>/dev/null; echo exp_rc=$?
ncu -i gpurun_out/ncu_bc.ncu-rep --page raw --csv > gpurun_out/ncu_bc_raw.csv 2>/dev/null
