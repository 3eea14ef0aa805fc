mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q -rA --durations=10 > gpurun_out/pytest_r2b.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_r2b.log
python tools/ubench.py r02 > gpurun_out/ubench.log 2>&1; echo "ubench rc=$?" >> gpurun_out/ubench.log
python bench.py --steps 10 --warmup 3 > gpurun_out/bench_r2b.json 2> gpurun_out/bench_r2b.err; echo "bench rc=$?" >> gpurun_out/bench_r2b.err
CMD="python bench.py --steps 2 --warmup 1 --no-extras --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/plain_launch.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_r02.csv $CMD > gpurun_out/ncu_launch.log 2>&1
CMD2="python bench.py --steps 1 --warmup 1 --frames 16 --no-extras --no-cpu-baseline --no-e2e"
$CMD2 > gpurun_out/plain_full.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_beamform_lds64 -s 1 -c 1 -o gpurun_out/prof_bf_r02 $CMD2 > gpurun_out/ncu_bf.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_envelope_tc -s 1 -c 1 -o gpurun_out/prof_env_r02 $CMD2 > gpurun_out/ncu_env.log 2>&1
echo done
