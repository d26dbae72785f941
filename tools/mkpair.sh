# pair_kernel measurement variants: only pool_pair.cu is recompiled, the other
# objects come from the main build.  bash tools/mkpair.sh "name:FLAGS" ...
cd "$(dirname "$0")/../paper_1005_2314_b200/csrc" || exit 1
make > /tmp/mkpair_main.log 2>&1 || { tail -20 /tmp/mkpair_main.log; exit 1; }
mkdir -p ../variants
ARCH="-gencode arch=compute_100a,code=sm_100a"
for v in "$@"; do
  n=${v%%:*}; f=${v#*:}
  ( nvcc -O3 -std=c++17 $ARCH -lineinfo -fmad=false -Xcompiler -fPIC,-O2,-ffp-contract=off -Xptxas -v \
      --expt-relaxed-constexpr $f -c -o /tmp/pool_pair_$n.o pool_pair.cu 2> ../variants/ptxas_pair_$n.log \
    && nvcc $ARCH -shared -o ../variants/lib_$n.so /tmp/pool_pair_$n.o $(ls obj/*.o | grep -v pool_pair) -lpthread \
    && echo "$n: $(grep -A3 pair_kernel ../variants/ptxas_pair_$n.log | grep -o 'Used [0-9]* registers') $(grep -o '[0-9]* bytes spill stores' ../variants/ptxas_pair_$n.log | sort -u | tr '\n' ' ')" ) &
done
wait
