# Round-2 (last session) ncu --set full captures of the batched kernels (one launch each, after
# the same command ran clean without ncu). Run under gpurun.
O=gpurun_out
CMDF="python bench.py --workload c4 --nrhs 8192 --profile fast --steps 1 --warmup 1 --no-cpu-baseline"
CMDE="python bench.py --workload c4 --nrhs 8192 --steps 1 --warmup 1 --no-cpu-baseline"
$CMDF > $O/r02c_c4_8192_fast.json 2> $O/r02c_c4_8192_fast.err || exit 1
$CMDE > $O/r02c_c4_8192_exact.json 2> $O/r02c_c4_8192_exact.err || exit 1
ncu --set full --import-source on --clock-control none -k regex:batched_fast -c 1 -o $O/r02c_batched_fast $CMDF > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:residual_dmma -c 1 -o $O/r02c_residual_dmma $CMDF > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:batched_nqp -c 1 -o $O/r02c_batched_exact $CMDE > /dev/null 2>&1
ls -la $O/*.ncu-rep
