mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q -rA --durations=10 > gpurun_out/pytest_r2c.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_r2c.log
python bench.py --steps 10 --warmup 3 > gpurun_out/bench_r2c.json 2> gpurun_out/bench_r2c.err; echo "bench rc=$?" >> gpurun_out/bench_r2c.err
CMD2="python bench.py --steps 1 --warmup 1 --frames 16 --no-extras --no-cpu-baseline --no-e2e"
$CMD2 > gpurun_out/plain_full.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_envelope_tc -s 1 -c 1 -o gpurun_out/prof_env_r02c $CMD2 > gpurun_out/ncu_env.log 2>&1
echo done
