# round-2 closing run: roofline inputs from one ncu capture of both RK stages,
# the full GPU suite, smoke, the default bench line, the reference arm, the
# launch list of the bench command, the secondary workloads
bash tools/gpu/prof_stages.sh
python tools/roofline_inputs.py gpurun_out/p_stages.ncu-rep "fv3d_tile<minmod,16x15,tolerance>"; cp profiles/traffic_cfg4.json profiles/fp64_peaks.json gpurun_out/
ncu -i gpurun_out/p_stages.ncu-rep --page details --csv > gpurun_out/r02j_fv3d_tile_stages_details.csv 2>/dev/null
python -m pytest tests -q -m gpu --timeout 1200 > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -4 gpurun_out/gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -3 gpurun_out/smoke.log
python bench.py --impl reference --steps 20 --warmup 3 > gpurun_out/r02j_bench_reference_cfg4.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
python bench.py --steps 20 --warmup 3 > gpurun_out/r02j_bench_cfg4.json 2> gpurun_out/bench.err; echo "bench rc=$?"; cat gpurun_out/r02j_bench_cfg4.json
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02j_cfg4_launches.csv python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --no-other-numerics > /dev/null 2>&1; echo "launches rc=$?"
python bench.py --workload cfg3 --steps 16 --warmup 3 --no-cpu-baseline > gpurun_out/r02j_bench_cfg3.json 2>/dev/null; echo "cfg3 rc=$?"
python bench.py --workload cfg3 --numerics tolerance --steps 16 --warmup 3 --no-cpu-baseline > gpurun_out/r02j_bench_cfg3_tolerance.json 2>/dev/null; echo "cfg3 tol rc=$?"
python bench.py --workload cfg2 --no-cpu-baseline > gpurun_out/r02j_bench_cfg2.json 2>/dev/null; echo "cfg2 rc=$?"
