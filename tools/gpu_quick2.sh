# quick check of the in-tree library: parity tests (no full-size files), smoke, a short bench
python -c "import paper_2009_13569_b200 as p; p.load()" || exit 1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_boundary.py -m gpu -x -q > gpurun_out/pytest_quick.log 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/pytest_quick.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python bench.py --no-cpu --no-e2e --no-c1 --steps 10 --warmup 3 2>/dev/null | cut -c1-400
