./scripts/fp64_peak
for v in "" nomma; do
  if [ -z "$v" ]; then export HH_LIB=""; tag=default; else export HH_LIB=$PWD/paper_2604_09147_b200/libhh_$v.so; tag=$v; fi
  for r in 1 4 8 16; do echo "[$tag] $(timeout 300 python scripts/profile_matvec.py 3d_exp_proxy $r 3 2>&1 | tail -1)"; done
  for r in 1 16; do echo "[$tag] $(timeout 300 python scripts/profile_matvec.py 3d_laplace $r 3 2>&1 | tail -1)"; done
done
unset HH_LIB
timeout 2400 python -m pytest tests -m gpu -x -q -k "not 3d_large" > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc $?
tail -3 gpurun_out/pytest_gpu.log
