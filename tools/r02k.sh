python tools/tune_variants.py 1
for v in qc qc0; do WALLACE_B200_LIB=$PWD/paper_1005_2314_b200/variants/lib_$v.so WALLACE_B200_PROFILE_DUMP=1 python bench.py --config 1 --steps 1 --warmup 1 --no-cpu --no-e2e --no-configs --no-sustained 2>&1 >/dev/null | grep "timeline pool" | head -2; done
