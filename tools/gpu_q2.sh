# build check, parity + boundary tests, 2^30 u64 timing by kernel family
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_boundary.py -x -q > gpurun_out/q2_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/q2_pytest.log
timeout 300 python tools/prof_run.py --n 30 --reps 3 --check ${ALGO:+--algo $ALGO} 2>&1 | tail -3
