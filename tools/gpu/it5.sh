python tools/gpu/fv3d_time.py auto > gpurun_out/t_tol.log 2>&1; cat gpurun_out/t_tol.log
python tools/gpu/fv3d_check.py > gpurun_out/fv3d_check.log 2>&1; grep -c "tile==legacy True" gpurun_out/fv3d_check.log; grep "tile==legacy False" gpurun_out/fv3d_check.log; grep "tol rel" gpurun_out/fv3d_check.log | sort | tail -3; tail -2 gpurun_out/fv3d_check.log
python -m pytest tests/test_tolerance_gpu.py tests/test_mr_tolerance_gpu.py -q -x 2>&1 | tail -2
