python tools/gpu/fv3d_time.py auto > gpurun_out/t_tol.log 2>&1; cat gpurun_out/t_tol.log
python tools/gpu/fv3d_time.py exact auto > gpurun_out/t_ex.log 2>&1; cat gpurun_out/t_ex.log
python tools/gpu/fv3d_check.py > gpurun_out/fv3d_check.log 2>&1; head -16 gpurun_out/fv3d_check.log | grep -c "tile==legacy True"; grep "tile==legacy False" gpurun_out/fv3d_check.log; tail -2 gpurun_out/fv3d_check.log
python -m pytest tests/test_tolerance_gpu.py tests/test_uniform_gpu.py tests/test_digests_gpu.py tests/test_multigpu.py tests/test_fullsize_gpu.py -q -x 2>&1 | tail -2
