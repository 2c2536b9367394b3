# ncu --set full of one kernel launch: gpu_prof1.sh <kernel regex> <skip> [n]
K=$1; S=$2; N=${3:-30}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 300 python tools/prof_run.py --n $N --reps 2 > gpurun_out/prof_plain.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"$K" -s $S -c 1 -o gpurun_out/prof_$K python tools/prof_run.py --n $N --reps 2 > gpurun_out/ncu_$K.log 2>&1
echo rc=$?
tail -3 gpurun_out/prof_plain.log
