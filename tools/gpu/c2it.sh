python -m pytest tests/test_mr_switches_gpu.py tests/test_mr_gpu.py tests/test_digests_gpu.py tests/test_mr_dist_gpu.py -q -x 2>&1 | tail -2
python bench.py --workload cfg2 --steps 500 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/c2.json 2>gpurun_out/c2.err; python -c "import json;d=json.load(open('gpurun_out/c2.json'));print('cfg2', d['value'], d['ms_per_step'])"
AF_MR_NO_SUBTREE=1 python bench.py --workload cfg2 --steps 500 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/c2b.json 2>gpurun_out/c2b.err; python -c "import json;d=json.load(open('gpurun_out/c2b.json'));print('cfg2 no-subtree', d['value'], d['ms_per_step'])"
AF_MR_PHASES=1 python tools/prof_mr.py --workload cfg2 --warmup 3 --steps 30 > gpurun_out/c2_phases.txt 2>&1; cat gpurun_out/c2_phases.txt
