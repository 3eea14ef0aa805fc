mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "all_kinds_whole_frame" --durations=3 > gpurun_out/pytest_c5all.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_c5all.log
echo done
