O=gpurun_out/ab; mkdir -p $O
for v in base u2 u4; do
  if [ $v = base ]; then L=""; else L=build/var/$v/libalnnls.so; fi
  for n in 2368 8192; do
    ALNNLS_LIB=$L timeout 600 python tools/quick_c4.py $n fast > $O/fast5_${v}_n$n.txt 2>&1
  done
done
for f in $O/fast5_*.txt; do echo $f; grep '"rep": 1' $f | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['loop_s'], d['total_s'], d['iters_mean'], d['loop_TFLOPs_algorithmic'])"; done
