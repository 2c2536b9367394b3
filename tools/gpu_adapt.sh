# adaptive IPS2Ra extractor: new parity tests, the digit step/sort tests, Zipf / Exponential / uniform digit timings, misalignment A/B
python -c "import paper_2009_13569_b200 as p; p.load()" || exit 1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "digit" > gpurun_out/pytest_digit.log 2>&1; echo digit_rc=$?; tail -5 gpurun_out/pytest_digit.log
timeout 600 python tools/bench_configs.py --reps 3 --algo digit --only c3 > gpurun_out/cfg_digit_c3.jsonl 2>&1; echo c3_rc=$?
timeout 600 python tools/bench_configs.py --reps 3 --algo digit --only c2 > gpurun_out/cfg_digit_c2.jsonl 2>&1; echo c2_rc=$?
timeout 300 python tools/misalign.py > gpurun_out/misalign.log 2>&1; echo mis_rc=$?
