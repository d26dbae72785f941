# build measurement variants: bash tools/mkvar.sh "name:FLAGS" ...  (quick builds: -DWB_QUICK=1 added)
cd "$(dirname "$0")/../paper_1005_2314_b200/csrc" || exit 1
for v in "$@"; do
  n=${v%%:*}; f=${v#*:}
  make variant VNAME=$n VFLAGS="-DWB_QUICK=1 $f" > /tmp/mkvar_$n.log 2>&1 || { echo "build failed: $n"; tail -20 /tmp/mkvar_$n.log; }
done
rm -rf ../variants/obj_*
ls ../variants
