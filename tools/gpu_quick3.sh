# check of the in-tree library: parity + boundary tests, smoke, the full bench line
python -c "import paper_2009_13569_b200 as p; p.load()" || exit 1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_boundary.py -m gpu -x -q > gpurun_out/pytest_quick.log 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/pytest_quick.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench_rc=$?
cut -c1-300 gpurun_out/bench.json
IPS4O_SOAK_SECONDS=200 IPS4O_SOAK_START=50000 timeout 900 python -m pytest tests/test_gpu_soak.py -m gpu -x -q -s -k "soak_" > gpurun_out/pytest_soak3.log 2>&1; echo soak_rc=$?; tail -3 gpurun_out/pytest_soak3.log
