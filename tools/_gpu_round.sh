mkdir -p gpurun_out
S=$(date +%s); python bench.py --steps 10 --warmup 3 > gpurun_out/bench_r2d.json 2> gpurun_out/bench_r2d.err; echo "bench rc=$? wall=$(( $(date +%s) - S ))s" >> gpurun_out/bench_r2d.err
echo done
