# A/B of library variants built by tools/build_variant.sh (run under gpurun).
# usage: bash tools/ab_run.sh <workload>[:d:n] <variant>...   ("base" = the in-tree build)
O=gpurun_out/ab
mkdir -p $O
w=$1; shift
IFS=: read -r wn wd wnn <<< "$w"
tag=$(echo $w | tr ':' '_')
for v in "$@"; do
  if [ $v = base ]; then L=""; else L=build/var/$v/libalnnls.so; fi
  ALNNLS_LIB=$L timeout 300 python tools/quick_phases.py $wn $wd $wnn > $O/phases_${tag}_$v.txt 2>&1
done
