# Round-2 measurement sweep (run under gpurun): bench lines per workload/profile into
# gpurun_out/r02_bench_*.json, the default command's ncu launch list, and one
# ncu --set full capture per top kernel (each command first ran clean without ncu).
O=gpurun_out
mkdir -p $O
set -x
python bench.py --steps 20 --warmup 5 > $O/r02_bench_c2.json 2> $O/r02_bench_c2.err
python bench.py --workload c2 --profile fast --steps 20 --warmup 5 --no-cpu-baseline > $O/r02_bench_c2_fast.json 2>&1
python bench.py --workload c1 --steps 20 --warmup 5 > $O/r02_bench_c1.json 2>&1
python bench.py --workload c1 --profile fast --steps 20 --warmup 5 --no-cpu-baseline > $O/r02_bench_c1_fast.json 2>&1
python bench.py --workload c3 --steps 3 --warmup 3 --no-cpu-baseline > $O/r02_bench_c3.json 2>&1
python bench.py --workload c3 --profile fast --steps 3 --warmup 3 --no-cpu-baseline > $O/r02_bench_c3_fast.json 2>&1
python bench.py --workload c4 --steps 3 --warmup 3 > $O/r02_bench_c4.json 2>&1
python bench.py --workload c4 --profile fast --steps 3 --warmup 3 --no-cpu-baseline > $O/r02_bench_c4_fast.json 2>&1
python bench.py --workload c4 --nrhs 8192 --steps 3 --warmup 3 --no-cpu-baseline > $O/r02_bench_c4_nrhs8192.json 2>&1
python bench.py --workload c5 --steps 3 --warmup 3 --no-cpu-baseline > $O/r02_bench_c5.json 2>&1
python bench.py --workload c5 --profile fast --steps 3 --warmup 3 --no-cpu-baseline > $O/r02_bench_c5_fast.json 2>&1
python bench.py --workload c5 --c5-setup allreduce --profile fast --steps 3 --warmup 3 --no-cpu-baseline > $O/r02_bench_c5_allreduce_fast.json 2>&1
ALNNLS_FORCE_ROWBLOCK=1 python bench.py --workload c5 --steps 3 --warmup 3 --no-cpu-baseline > $O/r02_bench_c5_rowblock_n1.json 2>&1
python bench.py --solver anti_acc --steps 5 --warmup 3 --no-cpu-baseline > $O/r02_bench_c2_anti_acc.json 2>&1
python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/r02_launches_plain.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/r02_c2_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/r02_ncu_launches.log 2>&1
