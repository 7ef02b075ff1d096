ncu --set full --import-source on --clock-control none -k regex:"mr_coarsen_level|mr_count_speed|mr_virtual_mark" -c 4 -o gpurun_out/p_coarsen -f python tools/prof_mr.py --workload cfg3 --warmup 1 --steps 1 > gpurun_out/p_coarsen.log 2>&1
ncu -i gpurun_out/p_coarsen.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/p_coarsen_mix.csv 2>/dev/null
