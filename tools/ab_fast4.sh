O=gpurun_out/ab; mkdir -p $O
timeout 300 python tools/fast2_check.py > $O/fast4_check.txt 2>&1; tail -n 2 $O/fast4_check.txt
for n in 8192 65536; do
  timeout 600 python tools/quick_c4.py $n fast > $O/fast4_n$n.txt 2>&1
done
for f in $O/fast4_n*.txt; do echo $f; grep '"rep": 1' $f | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['loop_s'], d['total_s'], d['iters_mean'], d['loop_TFLOPs_algorithmic'])"; done
