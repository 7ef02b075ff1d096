ncu --set full --import-source on --clock-control none -k regex:mr_stage_full2d -s 0 -c 1 -o gpurun_out/p_full -f python tools/prof_mr.py --workload cfg3 --warmup 1 --steps 1 > gpurun_out/p_full.log 2>&1
ncu -i gpurun_out/p_full.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/p_full_mix.csv 2>/dev/null
