python -m pytest tests/test_gpu_parity.py tests/test_gpu_modes.py tests/test_gpu_errors.py -q -x 2>&1 | tail -3
bash tools/qbench.sh 3 5 4 2
