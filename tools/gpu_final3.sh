# final round-2 measurement on the in-tree library: GPU tests, bench, smoke, launch list, ncu full (raw CSV -> summary), all configs
python -c "import paper_2009_13569_b200 as p; p.load()" || exit 1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench_rc=$?
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?
IPS4O_HOST_LEVELS=1 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/launches_r2.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --no-c1 --stat-steps 1 > gpurun_out/ncu_bench.log 2>&1; echo launches_rc=$?
IPS4O_HOST_LEVELS=1 timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"classify_v2|permute_kernel|basecase_kernel" -s 8 -c 8 \
  -o /tmp/ncu_full_head python tools/prof_run.py --n 30 --reps 2 > gpurun_out/ncu_full_head.log 2>&1; echo full_rc=$?
ncu -i /tmp/ncu_full_head.ncu-rep --page raw --csv > gpurun_out/ncu_full_head_raw.csv 2>/dev/null
python tools/ncu_summary.py gpurun_out/ncu_full_head_raw.csv > gpurun_out/ncu_full_head_summary.txt 2>&1
timeout 900 python tools/bench_configs.py --reps 3 > gpurun_out/cfg_tree.jsonl 2>&1; echo tree_rc=$?
timeout 900 python tools/bench_configs.py --reps 3 --algo digit > gpurun_out/cfg_digit.jsonl 2>&1; echo digit_rc=$?
