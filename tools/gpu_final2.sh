# bench + smoke + launch list (small outputs), records tests, records config
python -c "import paper_2009_13569_b200 as p; p.load()" || exit 1
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench_rc=$?
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?
IPS4O_HOST_LEVELS=1 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/launches_r2.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --no-c1 --stat-steps 1 > gpurun_out/ncu_bench.log 2>&1; echo launches_rc=$?
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x -k "REC100 or 3- or -3 or records or rec100" > gpurun_out/pytest_rec.log 2>&1; echo rec_rc=$?; tail -2 gpurun_out/pytest_rec.log
timeout 300 python tools/bench_configs.py --reps 3 --only c5 > gpurun_out/cfg_c5.jsonl 2>&1
