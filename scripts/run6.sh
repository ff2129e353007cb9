for v in "" c2 cvt s4 cvt_s4; do
  if [ -z "$v" ]; then export HH_LIB=""; tag=default; else export HH_LIB=$PWD/paper_2604_09147_b200/libhh_$v.so; tag=$v; fi
  for c in 3d_exp_proxy 3d_laplace; do
    echo "[$tag] $(timeout 300 python scripts/profile_matvec.py $c 1 3 2>&1 | tail -1)"
  done
done
unset HH_LIB
timeout 1200 python -m pytest tests -m gpu -x -q -k "not 3d_large" > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc $?
tail -3 gpurun_out/pytest_gpu.log
