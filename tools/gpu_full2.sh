# all GPU tests on the in-tree library (HEAD)
python -c "import paper_2009_13569_b200 as p; p.load()" || exit 1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/pytest_gpu.log
