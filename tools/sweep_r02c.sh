# Last-session c4 sweep (run under gpurun): bench lines for the batched workload and the
# launch list of the FAST command (after it ran clean without ncu).
O=gpurun_out
python bench.py --workload c4 --steps 3 --warmup 3 > $O/r02_bench_c4.json 2> $O/r02_bench_c4.err
python bench.py --workload c4 --profile fast --steps 3 --warmup 3 --no-cpu-baseline > $O/r02_bench_c4_fast.json 2> $O/r02_bench_c4_fast.err
python bench.py --workload c4 --nrhs 8192 --steps 3 --warmup 3 --no-cpu-baseline > $O/r02_bench_c4_nrhs8192.json 2> /dev/null
python bench.py --workload c4 --nrhs 8192 --profile fast --steps 3 --warmup 3 --no-cpu-baseline > $O/r02_bench_c4_nrhs8192_fast.json 2> /dev/null
python bench.py --workload c4 --nrhs 8192 --profile fast --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file $O/r02_c4_fast_launches.csv python bench.py --workload c4 --nrhs 8192 --profile fast --steps 1 --warmup 3 --no-cpu-baseline > $O/r02_ncu_c4_launches.log 2>&1
for f in c4 c4_fast c4_nrhs8192 c4_nrhs8192_fast; do python -c "
import json; d=json.load(open('$O/r02_bench_$f.json')); print('$f', round(d['value']), round(d['ms_per_step'],1), round(d['loop_ms'],1), round(d['e2e']['value']), d['roofline']['frac'], d['gpu_launches'])"; done
