# quick: build, selected GPU tests (-k expression), then optional extra command
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -x -q -k "$1" > gpurun_out/t1_pytest.log 2>&1; echo pytest_rc=$?
tail -5 gpurun_out/t1_pytest.log
