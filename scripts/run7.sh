for v in "" c1_s4 s4 c2_s4 s3 w16_s6 w16_s4 w12_s5; do
  if [ -z "$v" ]; then export HH_LIB=""; tag=default; else export HH_LIB=$PWD/paper_2604_09147_b200/libhh_$v.so; tag=$v; fi
  for c in 3d_exp_proxy 3d_laplace; do
    echo "[$tag] $(timeout 300 python scripts/profile_matvec.py $c 1 3 2>&1 | tail -1)"
  done
  echo "[$tag] $(timeout 300 python scripts/profile_matvec.py 3d_exp_proxy 16 3 2>&1 | tail -1)"
done
