mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py -m gpu -x -q -k "C3 or slice or lds64 or fuzz or random_multi or high_orders" > gpurun_out/pytest_p5.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_p5.log
echo done
