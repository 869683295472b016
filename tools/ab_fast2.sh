O=gpurun_out/ab; mkdir -p $O
for v in u1 u4; do for t in 1 2; do
  ALNNLS_FAST_TPW=$t ALNNLS_LIB=build/var/$v/libalnnls.so timeout 600 python tools/quick_c4.py 65536 fast > $O/fast2_${v}_t${t}.txt 2>&1
done; done
for f in $O/fast2_u*.txt; do echo $f; grep '"rep": 1' $f | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['loop_s'], d['total_s'], d['iters_mean'], d['loop_TFLOPs_algorithmic'])"; done
