export WALLACE_B200_LIB=$PWD/paper_1005_2314_b200/variants/lib_q.so
python -m pytest tests/test_gpu_parity.py -q -k "(pool_size1024 or pool_size2048 or pool_size4096) and latency and not huge" 2>&1 | tail -1
unset WALLACE_B200_LIB
python tools/tune_variants.py 1
