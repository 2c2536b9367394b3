python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/quick_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/quick_pytest.log
timeout 900 python -m pytest tests/test_gpu_fullsize.py -x -q -k "quartet" > gpurun_out/fs_pytest.log 2>&1; echo "fullsize rc=$?"; tail -3 gpurun_out/fs_pytest.log
python tools/bench_configs.py --only quartets --reps 2; python tools/bench_configs.py --only quartets --reps 2 --algo digit
