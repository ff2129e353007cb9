for i in 1 2; do
for v in base ""; do
  if [ -z "$v" ]; then export HH_LIB=""; tag=prefetch; else export HH_LIB=$PWD/paper_2604_09147_b200/libhh_$v.so; tag=$v; fi
  for c in 3d_exp_proxy 3d_laplace 2d_medium; do echo "[$tag] $(timeout 300 python scripts/profile_matvec.py $c 1 3 2>&1 | tail -1)"; done
  echo "[$tag] $(timeout 300 python scripts/profile_matvec.py 3d_exp_proxy 16 3 2>&1 | tail -1)"
done
done
