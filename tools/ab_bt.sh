# Batched EXACT: chain-lane sum variants x 256-/128-thread CTAs. Under gpurun.
O=gpurun_out/ab; mkdir -p $O
for v in base sqmap sq3; do
  if [ $v = base ]; then L=""; else L=build/var/$v/libalnnls.so; fi
  for n in 8192 65536; do
    ALNNLS_LIB=$L timeout 600 python tools/quick_c4.py $n > $O/v${v}_bt256_n$n.txt 2>&1
    ALNNLS_LIB=$L ALNNLS_BATCH_BT=128 timeout 600 python tools/quick_c4.py $n > $O/v${v}_bt128_n$n.txt 2>&1
  done
done
for f in $O/v*_bt*.txt; do echo $f; grep '"rep": 1' $f | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['loop_s'], d['total_s'], d['iters_mean'])"; done
