# near-maximum n (2^32 - 4097 elements of U32 and U64), tests/test_gpu_soak.py::test_near_maximum_n
python -c "import paper_2009_13569_b200 as p; p.load()" || exit 1
IPS4O_SOAK_SECONDS=1 timeout 1200 python -m pytest tests/test_gpu_soak.py -m gpu -x -q -s -k near_maximum > gpurun_out/pytest_nearmax.log 2>&1; echo nearmax_rc=$?
tail -30 gpurun_out/pytest_nearmax.log
nvidia-smi --query-gpu=memory.used,memory.total --format=csv
