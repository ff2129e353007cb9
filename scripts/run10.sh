for v in "" s2_wd48_x6 s3_wd32 s2_wd40_x5 s2_wd28 s2_wd64_x8; do
  if [ -z "$v" ]; then export HH_LIB=""; tag=default; else export HH_LIB=$PWD/paper_2604_09147_b200/libhh_$v.so; tag=$v; fi
  for c in 3d_exp_proxy 3d_laplace 2d_medium; do
    echo "[$tag] $(timeout 300 python scripts/profile_matvec.py $c 1 3 2>&1 | tail -1)"
  done
done
unset HH_LIB
for r in 2 4 8 16; do echo "[default] $(timeout 300 python scripts/profile_matvec.py 3d_exp_proxy $r 3 2>&1 | tail -1)"; done
timeout 1200 python -m pytest tests -m gpu -x -q -k "not 3d_large" > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc $?
tail -3 gpurun_out/pytest_gpu.log
