# timing of several compile variants: gpu_var.sh "<flags1>" "<flags2>" ...  (ARGS = prof_run args)
for v in "$@"; do
IPS4O_EXTRA_NVCC_FLAGS="$v" python -m paper_2009_13569_b200.build --force > gpurun_out/build.log 2>&1 || { tail -3 gpurun_out/build.log; exit 1; }
echo "== [$v]"; python tools/prof_run.py ${ARGS:---n 30 --reps 2} 2>&1 | grep -v "^0 " | cut -c1-220
done
