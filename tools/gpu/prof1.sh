for v in legacy exact tol; do
  arg=""; [ $v = legacy ] && arg=legacy; [ $v = tol ] && arg=tol
  ncu --set full --import-source on --clock-control none -k regex:fv3d -s 2 -c 1 -o gpurun_out/p_$v -f python tools/gpu/fv3d_one.py 9 2 $arg > gpurun_out/p_$v.log 2>&1
done
ls -la gpurun_out/
