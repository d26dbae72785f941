python tools/tune_variants.py 2,3,4 2>&1
