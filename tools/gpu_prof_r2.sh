# round-2 measurement: configs check, ncu launch list of the bench workload, ncu --set full of the hot kernels
timeout 600 python tools/bench_configs.py --reps 3 --only c4 > gpurun_out/cfg_c4.jsonl 2>&1
timeout 600 python tools/bench_configs.py --reps 3 --only next2 > gpurun_out/cfg_next2.jsonl 2>&1
timeout 600 python tools/bench_configs.py --reps 3 --only head > gpurun_out/cfg_head.jsonl 2>&1
IPS4O_HOST_LEVELS=1 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/launches_r2.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --no-c1 --stat-steps 0 > gpurun_out/ncu_bench.log 2>&1; echo launches_rc=$?
IPS4O_HOST_LEVELS=1 timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"classify_v2|permute_kernel|basecase_kernel" -s 6 -c 5 \
  -o gpurun_out/ncu_full_r2 python tools/prof_run.py --n 30 --reps 2 > gpurun_out/ncu_full_r2.log 2>&1; echo full_rc=$?
