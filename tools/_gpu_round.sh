mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_fuzz.py -m gpu -q -rf > gpurun_out/pytest_fuzz.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_fuzz.log
echo done
