O=gpurun_out/ab; mkdir -p $O
timeout 600 python tools/fast2_check.py > $O/fast2_check.txt 2>&1; tail -n 2 $O/fast2_check.txt
for n in 8192 16384 32768 65536; do
  ALNNLS_FAST_2CTA=0 timeout 600 python tools/quick_c4.py $n fast > $O/fast1_n$n.txt 2>&1
  timeout 600 python tools/quick_c4.py $n fast > $O/fast2_t1_n$n.txt 2>&1
done
for f in $O/fast1_n*.txt $O/fast2_t1*.txt; do echo $f; grep '"rep": 1' $f | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['loop_s'], d['total_s'], d['iters_mean'], d['loop_TFLOPs_algorithmic'])"; done
