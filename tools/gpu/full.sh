# full GPU test suite + default bench line
python -m pytest tests -q -m gpu -x --timeout 1200 > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -15 gpurun_out/gpu_tests.log
python bench.py --steps 20 --warmup 3 > gpurun_out/r02_bench.json 2> gpurun_out/r02_bench.err; echo "bench rc=$?"; cat gpurun_out/r02_bench.json; tail -3 gpurun_out/r02_bench.err
