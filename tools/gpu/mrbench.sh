# MR workloads: bench lines + one cfg3 launch list
python bench.py --workload cfg2 --steps 500 --warmup 5 --no-cpu-baseline > gpurun_out/r02_cfg2.json 2>gpurun_out/r02_cfg2.err; tail -c 1500 gpurun_out/r02_cfg2.json
python bench.py --workload cfg3 --steps 64 --warmup 3 --no-cpu-baseline > gpurun_out/r02_cfg3.json 2>gpurun_out/r02_cfg3.err; tail -c 1500 gpurun_out/r02_cfg3.json
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_cfg3_launches.csv python bench.py --workload cfg3 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
echo done
