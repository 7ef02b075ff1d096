python -m pytest tests -q -m gpu -x --timeout 1200 > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -5 gpurun_out/gpu_tests.log
python bench.py --workload cfg3 --steps 16 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/c3.json 2>gpurun_out/c3.err; python -c "import json;d=json.load(open('gpurun_out/c3.json'));print('cfg3', d['value'], d['ms_per_step'])"
python bench.py --workload cfg2 --steps 500 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/c2.json 2>gpurun_out/c2.err; python -c "import json;d=json.load(open('gpurun_out/c2.json'));print('cfg2', d['value'], d['ms_per_step'])"
