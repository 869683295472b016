O=gpurun_out/ab; mkdir -p $O
for n in 4096 8192 16384 32768; do for two in 0 1; do
  ALNNLS_FAST_2CTA=$two timeout 600 python tools/quick_c4.py $n fast > $O/fast3_n${n}_two${two}.txt 2>&1
done; done
for f in $O/fast3_n*.txt; do echo $f; grep '"rep": 1' $f | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['loop_s'], d['total_s'], d['iters_mean'], d['loop_TFLOPs_algorithmic'])"; done
