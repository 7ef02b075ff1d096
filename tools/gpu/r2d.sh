python -m pytest tests -q -m gpu -x --timeout 1200 > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -5 gpurun_out/gpu_tests.log
for v in tol exact; do
  arg=""; [ $v = tol ] && arg=tol
  ncu --set full --import-source on --clock-control none -k regex:fv3d -s 2 -c 2 -o gpurun_out/p2_$v -f python tools/gpu/fv3d_one.py 9 2 $arg > gpurun_out/p2_$v.log 2>&1
done
python bench.py --steps 20 --warmup 3 > gpurun_out/r02d_bench.json 2> gpurun_out/r02d_bench.err; echo "bench rc=$?"; cat gpurun_out/r02d_bench.json
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02d_cfg4_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo "launches rc=$?"
