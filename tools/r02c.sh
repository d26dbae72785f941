make -s -C tests/cpp
for b in 65536 262144 1048576 4194304; do echo "block $b"; WALLACE_B200_LOOKAHEAD=$b ./tests/cpp/test_dropin 2>&1 | grep "drop-in\|checks"; done
python -m pytest tests/test_gpu_errors.py -q 2>&1 | tail -3
