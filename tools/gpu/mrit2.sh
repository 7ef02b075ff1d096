python -m pytest tests/test_mr_switches_gpu.py -q -x 2>&1 | tail -3
python -m pytest tests/test_mr_gpu.py tests/test_digests_gpu.py tests/test_mr_dist_gpu.py tests/test_kats_gpu.py tests/test_fullsize_gpu.py tests/test_shim_gpu.py -q -x 2>&1 | tail -3
python bench.py --workload cfg3 --steps 16 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/c3.json 2>gpurun_out/c3.err; python -c "import json;d=json.load(open('gpurun_out/c3.json'));print('cfg3', d['value'], d['ms_per_step'])"
AF_MR_NO_FULLK=1 python bench.py --workload cfg3 --steps 16 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/c3b.json 2>gpurun_out/c3b.err; python -c "import json;d=json.load(open('gpurun_out/c3b.json'));print('cfg3 nofullk', d['value'], d['ms_per_step'])"
python bench.py --workload cfg2 --steps 500 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/c2.json 2>gpurun_out/c2.err; python -c "import json;d=json.load(open('gpurun_out/c2.json'));print('cfg2', d['value'], d['ms_per_step'])"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c3_launches.csv python tools/prof_mr.py --workload cfg3 --warmup 2 --steps 1 > gpurun_out/c3_l.log 2>&1; tail -1 gpurun_out/c3_l.log
