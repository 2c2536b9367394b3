python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/quick_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/quick_pytest.log
timeout 900 python -m pytest tests/test_gpu_fullsize.py -x -q -k "u32 or eightdup or zero" > gpurun_out/fs_pytest.log 2>&1; echo "fullsize rc=$?"; tail -3 gpurun_out/fs_pytest.log
python tools/prof_run.py --n 30 --reps 2 --dist uniform_u32 2>&1 | tail -1
python tools/prof_run.py --n 30 --reps 2 --dist uniform_u32 --algo digit 2>&1 | tail -1
