# re-entry check: full GPU suite at HEAD + default bench line + fv3d check
python -m pytest tests -q -m gpu -x --timeout 1200 > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -15 gpurun_out/gpu_tests.log
python tools/gpu/fv3d_check.py > gpurun_out/fv3d_check.log 2>&1; tail -12 gpurun_out/fv3d_check.log
python bench.py --steps 20 --warmup 3 > gpurun_out/r02c_bench.json 2> gpurun_out/r02c_bench.err; echo "bench rc=$?"; cat gpurun_out/r02c_bench.json; tail -3 gpurun_out/r02c_bench.err
