# round-2 session-2 baseline: full GPU suite, full bench line, per-config quick timings
python -m pytest tests -q -m gpu -x > gpurun_out/r02h_all.log 2>&1
tail -5 gpurun_out/r02h_all.log
python bench.py > gpurun_out/r02h_bench.json 2> gpurun_out/r02h_bench.err
tail -c 600 gpurun_out/r02h_bench.err
bash tools/qbench.sh 2 3 4 5 1
