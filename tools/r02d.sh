( time python bench.py ) > gpurun_out/r02d_bench.json 2> gpurun_out/r02d_bench.err
tail -3 gpurun_out/r02d_bench.err
