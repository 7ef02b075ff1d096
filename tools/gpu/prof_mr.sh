ncu --set full --import-source on --clock-control none -k regex:mr_stage_kernel -s 0 -c 2 -o gpurun_out/p_cfg3_stage -f python bench.py --workload cfg3 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/p_cfg3_stage.log 2>&1
tail -3 gpurun_out/p_cfg3_stage.log
