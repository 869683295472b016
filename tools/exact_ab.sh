# A/B of exact-loop library variants (tools/build_variant.sh) on loop phases, under gpurun.
# usage: bash tools/exact_ab.sh "<workload>[:d:n] ..." <variant>...   ("base" = in-tree build)
ws=$1; shift
for v in "$@"; do
  L=""; [ "$v" != base ] && L=build/var/$v/libalnnls.so
  for w in $ws; do
    IFS=: read -r wn wd wnn <<< "$w"
    echo "== $v $w"; ALNNLS_LIB=$L timeout 600 python tools/quick_phases.py $wn $wd $wnn 2>&1 | head -3
  done
done
