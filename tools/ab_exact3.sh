O=gpurun_out/ab; mkdir -p $O
for v in "$@"; do
  L=build/var/$v/libalnnls.so
  ALNNLS_LIB=$L timeout 600 python tools/quick_c4.py 65536 > $O/exact3_${v}_n65536.txt 2>&1
done
for v in "$@"; do f=$O/exact3_${v}_n65536.txt; echo $f; grep '"rep": 1' $f | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['loop_s'], d['total_s'], d['iters_mean'], d['loop_TFLOPs_algorithmic'])"; done
