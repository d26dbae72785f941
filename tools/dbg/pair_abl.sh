export WALLACE_B200_PAIR=1
for m in 0 2 3 4; do
  echo "== PAIR_DEBUG=$m"
  WALLACE_B200_PAIR_DEBUG=$m bash tools/qbench.sh 3
done
