python -m pytest tests/test_amr_gpu.py -q -x --timeout 900 > gpurun_out/amr2.log 2>&1; echo "rc=$?"; tail -30 gpurun_out/amr2.log
python tools/gpu/amr_time.py 2 6 10 64 2.5e-4 0 1 1; python tools/gpu/amr_time.py 3 3 7 32 7e-4 3 1 1; python tools/gpu/amr_time.py 3 3 8 32 3.5e-4 3 1 1
