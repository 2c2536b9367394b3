# quick GPU check: build, parity tests, 2^30 timing by kernel family
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -15
timeout 300 python tools/prof_run.py --n 30 --reps 3 --check 2>&1 | tail -4
