python -m pytest tests/test_gpu_errors.py tests/test_gpu_baselines.py tests/test_cpp_dropin.py -q -s > gpurun_out/r02b_new.log 2>&1
tail -50 gpurun_out/r02b_new.log
python -m pytest tests -q -m gpu > gpurun_out/r02b_all.log 2>&1
tail -5 gpurun_out/r02b_all.log
