# the C++ drop-in's timed call patterns (tests/cpp/test_dropin.cpp) with the
# main library and with every built variant
cd "$(dirname "$0")/../.." || exit 1
echo "== main"; tests/cpp/test_dropin | grep "drop-in\|failed"
for lib in paper_1005_2314_b200/variants/lib_*.so; do
  echo "== $lib"; WALLACE_B200_LIB=$PWD/$lib LD_PRELOAD=$PWD/$lib tests/cpp/test_dropin | grep "drop-in\|failed"
done
