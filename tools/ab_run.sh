# A/B of library variants built by tools/build_variant.sh (run under gpurun).
# usage: bash tools/ab_run.sh <workload> <variant>...   ("base" = the in-tree build)
O=gpurun_out/ab
mkdir -p $O
w=$1; shift
for v in "$@"; do
  if [ $v = base ]; then L=""; else L=build/var/$v/libalnnls.so; fi
  ALNNLS_LIB=$L timeout 300 python tools/quick_phases.py $w > $O/phases_${w}_$v.txt 2>&1
done
