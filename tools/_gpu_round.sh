mkdir -p gpurun_out
timeout 900 python bench.py --steps 2 --warmup 1 --force-sharded --no-cpu-baseline --no-extras --no-e2e --frames 32 > gpurun_out/bench_sharded3.json 2> gpurun_out/bench_sharded3.err; echo "rc=$?" >> gpurun_out/bench_sharded3.err
echo done
