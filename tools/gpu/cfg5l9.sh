( while true; do nvidia-smi --query-gpu=memory.used --format=csv,noheader,nounits >> gpurun_out/mem.log; sleep 1; done ) &
MP=$!
timeout 900 python bench.py --workload cfg5 --level 9 --steps 4 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/c5l9.json 2> gpurun_out/c5l9.err; echo "rc=$?"
kill $MP
tail -c 1500 gpurun_out/c5l9.json; tail -3 gpurun_out/c5l9.err; sort -n gpurun_out/mem.log | tail -1
