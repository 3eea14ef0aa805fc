mkdir -p gpurun_out
timeout 900 python bench.py --steps 3 --warmup 2 --force-sharded --no-cpu-baseline --no-extras --e2e-frames 32 > gpurun_out/bench_sharded1.json 2> gpurun_out/bench_sharded1.err; echo "rc=$?" >> gpurun_out/bench_sharded1.err
echo done
