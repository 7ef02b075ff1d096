python tools/gpu/amr_time.py 3 3 8 32 3.5e-4 3 1 1 > gpurun_out/amr_prof_run.log 2>&1; echo "rc=$?"; cat gpurun_out/amr_prof_run.log
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/amr_launches_3d_L8.csv python tools/gpu/amr_time.py 3 3 8 32 3.5e-4 3 1 1 > gpurun_out/amr_prof_ncu.log 2>&1; echo "ncu rc=$?"
python tools/launch_summary.py gpurun_out/amr_launches_3d_L8.csv | head -40
