# A/B of FAST-loop library variants (tools/build_variant.sh) at one workload, under gpurun.
# usage: bash tools/fast_ab.sh <workload> <variant>...   ("base" = the in-tree build)
w=$1; shift
for v in "$@"; do
  L=""; [ "$v" != base ] && L=build/var/$v/libalnnls.so
  echo "== $v"; ALNNLS_LIB=$L python tools/fast_phases.py $w
done
