O=gpurun_out/ab
mkdir -p $O
for v in base cg16 cg16jb16; do
  if [ $v = base ]; then L=""; else L=build/var/$v/libalnnls.so; fi
  ALNNLS_LIB=$L timeout 300 python tools/quick_c4.py 16384 > $O/c4_$v.txt 2>&1
done
ALNNLS_LIB=build/var/cg16/libalnnls.so timeout 300 python -m pytest tests/test_gpu_batched.py -x -q > $O/tests_cg16.log 2>&1
