mkdir -p gpurun_out
python -m pytest tests/test_gpu_quality.py -m gpu -x -q -rA > gpurun_out/pytest_quality.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_quality.log
python tools/ubench.py r02 > gpurun_out/ubench.log 2>&1; echo "ubench rc=$?" >> gpurun_out/ubench.log
python bench.py --workload C4 --steps 5 --warmup 3 --no-cpu-baseline --no-extras > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
echo done
