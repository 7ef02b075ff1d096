python tools/gpu/c3gap.py
ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/c3gap.csv python tools/gpu/c3gap.py > gpurun_out/c3gap.log 2>&1; tail -1 gpurun_out/c3gap.log
