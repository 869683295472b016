# Round profiling batch (run under gpurun): bench lines + ncu launch lists + full captures.
set -x
O=gpurun_out/prof
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q > $O/gpu_tests.log 2>&1
timeout 600 python bench.py > $O/bench_c2.json 2> $O/bench_c2.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_ref_c2.json 2> $O/bench_ref_c2.err
timeout 600 python bench.py --profile fast > $O/bench_c2_fast.json 2> $O/bench_c2_fast.err
timeout 900 python bench.py --workload c4 --steps 3 --warmup 3 > $O/bench_c4.json 2> $O/bench_c4.err
timeout 900 python bench.py --workload c4 --profile fast --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_c4_fast.json 2> $O/bench_c4_fast.err
timeout 900 python bench.py --workload c4 --impl reference --steps 1 --warmup 1 > $O/bench_ref_c4.json 2> $O/bench_ref_c4.err
timeout 900 python bench.py --workload c5 --steps 2 --warmup 1 --no-cpu-baseline > $O/bench_c5.json 2> $O/bench_c5.err
timeout 900 python bench.py --workload c5 --c5-setup allreduce --profile fast --steps 2 --warmup 1 > $O/bench_c5_allreduce_fast.json 2> $O/bench_c5_allreduce_fast.err
timeout 900 python bench.py --workload c3 --steps 2 --warmup 1 --no-cpu-baseline > $O/bench_c3.json 2> $O/bench_c3.err
timeout 900 python bench.py --workload c1 --steps 5 --warmup 3 > $O/bench_c1.json 2> $O/bench_c1.err
timeout 900 python bench.py --solver anti_acc --steps 2 --warmup 1 --no-cpu-baseline > $O/bench_c2_anti_acc.json 2> $O/bench_c2_anti_acc.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/c2_launches.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > $O/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"nqp_loop|syrk_streamk|colchain" -c 3 -o $O/c2_full python bench.py --steps 1 --warmup 1 --no-cpu-baseline > $O/ncu_full.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/c4_launches.csv python bench.py --workload c4 --nrhs 8192 --steps 1 --warmup 1 --no-cpu-baseline > $O/ncu_launch_c4.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"batched_nqp|residual_batched" -c 2 -o $O/c4_full python bench.py --workload c4 --nrhs 8192 --steps 1 --warmup 1 --no-cpu-baseline > $O/ncu_full_c4.log 2>&1
ls -la $O
