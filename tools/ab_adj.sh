O=gpurun_out/ab; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_batched.py tests/test_gpu_c4_full.py tests/test_gpu_edges.py -m gpu -x -q 2>&1 | tail -n 2
for n in 8192 65536; do
  timeout 600 python tools/quick_c4.py $n > $O/adj_n$n.txt 2>&1
done
for f in $O/adj_n*.txt; do echo $f; grep '"rep": 1' $f | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['loop_s'], d['total_s'], d['iters_mean'], d['loop_TFLOPs_algorithmic'])"; done
