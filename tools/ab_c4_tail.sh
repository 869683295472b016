# Batched tail A/B (under gpurun): a rank-sized 8192-column shard vs the full 65536
# columns, for the in-tree build and one variant (build/var/noskip).
mkdir -p gpurun_out/ab
for v in base noskip; do
  if [ $v = base ]; then L=""; else L=build/var/$v/libalnnls.so; fi
  for n in 8192 65536; do ALNNLS_LIB=$L timeout 300 python tools/quick_c4.py $n > gpurun_out/ab/c4n${n}_$v.txt 2>&1; done
done
timeout 300 python -m pytest tests/test_gpu_batched.py tests/test_sharding.py -x -q > gpurun_out/ab/tests_skip.log 2>&1
