O=gpurun_out/ab; mkdir -p $O
timeout 300 python tools/fast2_check.py > $O/fast6_check.txt 2>&1; tail -n 5 $O/fast6_check.txt
for n in 2369 8192 65536; do for k in 1 0; do
  ALNNLS_FAST_NO_TAIL_COMPACT=$k timeout 600 python tools/quick_c4.py $n fast > $O/fast6_nocompact${k}_n$n.txt 2>&1
done; done
for f in $O/fast6_no*.txt; do echo $f; grep '"rep": 1' $f | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['loop_s'], d['total_s'], d['iters_mean'], d['loop_TFLOPs_algorithmic'])"; done
