# baseline of the current library: non-slow GPU tests, every config (tree + digit)
python -c "import paper_2009_13569_b200 as p; p.load()" || exit 1
timeout 900 python -m pytest tests -m "gpu and not slow" -x -q > gpurun_out/pytest_quick.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_quick.log
timeout 600 python tools/bench_configs.py --reps 3 > gpurun_out/cfg_tree.jsonl 2>&1; echo cfg_tree=$?
timeout 600 python tools/bench_configs.py --reps 3 --algo digit > gpurun_out/cfg_digit.jsonl 2>&1; echo cfg_digit=$?
