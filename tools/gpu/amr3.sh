python -m pytest tests/test_amr_gpu.py -q -x --timeout 900 > gpurun_out/amr3.log 2>&1; echo "rc=$?"; tail -5 gpurun_out/amr3.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -5
