# ncu --set full of the level-1/2 classify, level-2 permute and level-2 base case at 2^30 u64
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 300 python tools/prof_run.py --n 30 --reps 2 > gpurun_out/prof_plain.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"classify_reg|basecase|permute_kernel" -s 9 -c 6 -o gpurun_out/prof_full python tools/prof_run.py --n 30 --reps 2 > gpurun_out/ncu_full.log 2>&1
echo rc=$?
