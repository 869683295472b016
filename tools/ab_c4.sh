# A/B of library variants on the batched c4 path (16384 columns; exact and FAST).
# usage (under gpurun): bash tools/ab_c4.sh <variant>...   ("base" = the in-tree build)
O=gpurun_out/ab
mkdir -p $O
for v in "$@"; do
  if [ $v = base ]; then L=""; else L=build/var/$v/libalnnls.so; fi
  ALNNLS_LIB=$L timeout 300 python tools/quick_c4.py 16384 > $O/c4_$v.txt 2>&1
  ALNNLS_LIB=$L timeout 300 python tools/quick_c4.py 16384 fast > $O/c4fast_$v.txt 2>&1
done
