# A/B timing of prof_run args $ARGS: default build vs $VARIANT build (no tests)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 300 python tools/prof_run.py $ARGS 2>&1 | tail -1
IPS4O_EXTRA_NVCC_FLAGS="$VARIANT" python -m paper_2009_13569_b200.build --force > gpurun_out/build_b.log 2>&1 || { tail -5 gpurun_out/build_b.log; exit 1; }
echo "variant: $VARIANT"
timeout 300 python tools/prof_run.py $ARGS 2>&1 | tail -1
