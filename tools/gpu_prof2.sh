# ncu --set full of one kernel launch with extra prof_run args: gpu_prof2.sh <kernel regex> <skip> "<args>"
K=$1; S=$2; ARGS=$3
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 300 python tools/prof_run.py $ARGS > gpurun_out/prof_plain.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"$K" -s $S -c 1 -o gpurun_out/prof_$K python tools/prof_run.py $ARGS > gpurun_out/ncu_$K.log 2>&1
echo rc=$?
tail -2 gpurun_out/prof_plain.log
