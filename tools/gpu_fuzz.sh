# randomized differential test with guard bands (tests/test_gpu_parity.py::test_random_cases_with_guard_bands)
python -c "import paper_2009_13569_b200 as p; p.load()" || exit 1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "random_cases" > gpurun_out/pytest_fuzz.log 2>&1; echo fuzz_rc=$?
tail -30 gpurun_out/pytest_fuzz.log
