python tools/gpu/fv3d_time.py auto > gpurun_out/t_tol.log 2>&1; cat gpurun_out/t_tol.log
python tools/gpu/fv3d_time.py exact auto > gpurun_out/t_ex.log 2>&1; cat gpurun_out/t_ex.log
python -m pytest tests/test_tolerance_gpu.py tests/test_uniform_gpu.py tests/test_digests_gpu.py -q -x -k "cfg4 or cfg1 or tile or tol or u3d or 3d" 2>&1 | tail -2
