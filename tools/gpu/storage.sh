python -m pytest tests/test_mr_storage_gpu.py -x -q -s --timeout 900 > gpurun_out/storage.log 2>&1; echo "rc=$?"; tail -30 gpurun_out/storage.log
