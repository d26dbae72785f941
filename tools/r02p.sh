# full GPU suite + per-config quick timings of the current build
python -m pytest tests -q -m gpu -x > gpurun_out/r02p_all.log 2>&1
tail -3 gpurun_out/r02p_all.log
bash tools/qbench.sh 2 3 4 5 1
