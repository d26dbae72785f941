# timing-only ablations of pair_kernel (WALLACE_B200_PAIR_DEBUG): 2 no bulk
# copies, 3 no staging, 4 every row aligned, 5 output rows resident in L2, 6 rows handed back before their copy has read them
for m in ${@:-0 2 3 4 5}; do
  echo "== PAIR_DEBUG=$m"
  WALLACE_B200_PAIR_DEBUG=$m bash tools/qbench.sh 3
done
