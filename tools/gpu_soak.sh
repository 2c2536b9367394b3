# soak run (tests/test_gpu_soak.py): randomized differential cases past the fixed 240 + repeated large sorts
python -c "import paper_2009_13569_b200 as p; p.load()" || exit 1
IPS4O_SOAK_START=${2:-240} IPS4O_SOAK_SECONDS=${1:-720} timeout 1500 python -m pytest tests/test_gpu_soak.py -m gpu -x -q -s > gpurun_out/pytest_soak.log 2>&1; echo soak_rc=$?
tail -40 gpurun_out/pytest_soak.log
