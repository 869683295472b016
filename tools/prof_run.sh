set -x
mkdir -p gpurun_out/prof
timeout 600 python bench.py > gpurun_out/prof/bench_c2.json 2> gpurun_out/prof/bench_c2.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/prof/bench_ref_c2.json 2> gpurun_out/prof/bench_ref_c2.err
timeout 900 python bench.py --workload c4 --steps 3 --warmup 3 > gpurun_out/prof/bench_c4.json 2> gpurun_out/prof/bench_c4.err
timeout 900 python bench.py --workload c4 --impl reference --steps 1 --warmup 1 > gpurun_out/prof/bench_ref_c4.json 2> gpurun_out/prof/bench_ref_c4.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/prof/c2_launches.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/prof/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"nqp_loop|syrk_exact|colchain" -c 3 -o gpurun_out/prof/c2_full python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/prof/ncu_full.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/prof/c4_launches.csv python bench.py --workload c4 --nrhs 8192 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/prof/ncu_launch_c4.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"batched_nqp|syrk_exact|residual_batched" -c 3 -o gpurun_out/prof/c4_full python bench.py --workload c4 --nrhs 8192 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/prof/ncu_full_c4.log 2>&1
ls -la gpurun_out/prof
