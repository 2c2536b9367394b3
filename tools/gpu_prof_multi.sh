# ncu --set full of several kernels (one launch each) of a prof_run: gpu_prof_multi.sh "<prof_run args>" regex:skip ...
ARGS=$1; shift
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 300 python tools/prof_run.py $ARGS > gpurun_out/prof_plain.log 2>&1 || { echo plain failed; exit 1; }
for ks in "$@"; do K=${ks%%:*}; S=${ks##*:}
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"$K" -s $S -c 1 -o gpurun_out/prof_$K python tools/prof_run.py $ARGS > gpurun_out/ncu_$K.log 2>&1; echo "$K rc=$?"
done
