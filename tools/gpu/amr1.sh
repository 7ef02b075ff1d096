python -m pytest tests/test_amr_gpu.py -q --timeout 900 > gpurun_out/amr1.log 2>&1; echo "rc=$?"; tail -40 gpurun_out/amr1.log
