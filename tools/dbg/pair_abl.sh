# timing-only ablations of pair_kernel (WALLACE_B200_PAIR_DEBUG, honoured by
# builds with -DWB_PAIR_DEBUGKNOBS=1 only): 2 no bulk copies, 3 no staging,
# 4 every row aligned, 5 output rows resident in L2, 6 rows handed back
# before their copy has read them.  Build the variant first:
#   bash tools/mkpair.sh "dbg:-DWB_PAIR_DEBUGKNOBS=1"
export WALLACE_B200_LIB=$PWD/paper_1005_2314_b200/variants/lib_dbg.so
for m in ${@:-0 2 3 4 5 6}; do
  echo "== PAIR_DEBUG=$m"
  WALLACE_B200_PAIR_DEBUG=$m bash tools/qbench.sh 3
done
