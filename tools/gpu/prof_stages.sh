# both RK-stage launches of the 3D tile kernel (tolerance mode) at 512^3, full set
ncu --set full --import-source on --clock-control none -k regex:fv3d -s 2 -c 2 -o gpurun_out/p_stages -f python tools/gpu/fv3d_one.py 9 2 tol > gpurun_out/p_stages.log 2>&1
python bench.py --steps 20 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/bench_launches.csv python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --no-other-numerics > /dev/null 2>&1; echo "launches rc=$?"
