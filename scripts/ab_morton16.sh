timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2
for i in 1 2; do
for v in "" morton; do
  if [ -z "$v" ]; then export HH_LIB=""; tag=lpt; else export HH_LIB=$PWD/paper_2604_09147_b200/libhh_$v.so; tag=$v; fi
  for c in 3d_exp_proxy 3d_laplace; do echo "[$tag] $(timeout 300 python scripts/profile_matvec.py $c 16 3 2>&1 | tail -1)"; done
done
done
unset HH_LIB
HH_PROFILE_BUILD=1 timeout 900 python scripts/profile_matvec.py 3d_large 1 3 2>&1 | tail -3
