# full GPU round on the in-tree library: all GPU tests, bench, configs (tree)
python -c "import paper_2009_13569_b200 as p; p.load()" || exit 1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench_rc=$?
timeout 900 python tools/bench_configs.py --reps 3 > gpurun_out/cfg_tree.jsonl 2>&1; echo cfg=$?
