for w in amr3d amr2d; do
python bench.py --workload $w > gpurun_out/r02f_bench_$w.json 2> gpurun_out/r02f_bench_$w.err; echo "$w rc=$?"; cat gpurun_out/r02f_bench_$w.json; tail -3 gpurun_out/r02f_bench_$w.err
done
python bench.py --workload amr3d --impl reference > gpurun_out/r02f_bench_reference_amr3d.json 2>/dev/null; cat gpurun_out/r02f_bench_reference_amr3d.json
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02f_amr3d_launches.csv python bench.py --workload amr3d --steps 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo "launches rc=$?"
python tools/launch_summary.py gpurun_out/r02f_amr3d_launches.csv > gpurun_out/r02f_amr3d_launch_summary.txt; head -12 gpurun_out/r02f_amr3d_launch_summary.txt
