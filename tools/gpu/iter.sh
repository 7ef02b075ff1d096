# build-measure iteration: correctness vs legacy, timing, one ncu capture per mode
python tools/gpu/fv3d_check.py > gpurun_out/fv3d_check.log 2>&1; tail -8 gpurun_out/fv3d_check.log
for v in exact tol; do
  arg=""; [ $v = tol ] && arg=tol
  ncu --set full --import-source on --clock-control none -k regex:fv3d -s 2 -c 1 -o gpurun_out/p_$v -f python tools/gpu/fv3d_one.py 9 2 $arg > gpurun_out/p_$v.log 2>&1
done
