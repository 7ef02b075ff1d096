set -x
nproc; free -g; lscpu | grep -i "model name"
python -c "import paper_1603_05211_b200 as P; P.load_library(); print('lib ok')"
python bench.py --steps 20 --warmup 3 > gpurun_out/r02_b_cfg4.json 2> gpurun_out/r02_b_cfg4.err
tail -c 3000 gpurun_out/r02_b_cfg4.json
( time python bench.py --impl reference --steps 20 --warmup 3 ) > gpurun_out/r02_ref_cfg4.json 2> gpurun_out/r02_ref_cfg4.err
cat gpurun_out/r02_ref_cfg4.json; tail -5 gpurun_out/r02_ref_cfg4.err
