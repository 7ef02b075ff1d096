# one ncu --set full capture of the exact-mode fv3d kernel + SASS/source export
ncu --set full --import-source on --clock-control none -k regex:fv3d -s 2 -c 1 -o gpurun_out/p_ex -f python tools/gpu/fv3d_one.py 9 2 > gpurun_out/p_ex.log 2>&1
ncu -i gpurun_out/p_ex.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/p_ex_mix.csv 2>/dev/null
ncu -i gpurun_out/p_ex.ncu-rep --page raw --csv > gpurun_out/p_ex_raw.csv 2>/dev/null
