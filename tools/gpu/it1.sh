python tools/gpu/fv3d_time.py auto 1 2 5 8 > gpurun_out/t_tol.log 2>&1; cat gpurun_out/t_tol.log
python tools/gpu/fv3d_time.py exact auto 2 > gpurun_out/t_ex.log 2>&1; cat gpurun_out/t_ex.log
python tools/gpu/fv3d_check.py > gpurun_out/fv3d_check.log 2>&1; cat gpurun_out/fv3d_check.log
