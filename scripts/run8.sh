for v in c1_s4 c1_s3 c1_s3_wd12_b5 c1_s2_b5 c1_s2_wd12_b6 c1_s4_wd8_b4; do
  export HH_LIB=$PWD/paper_2604_09147_b200/libhh_$v.so; tag=$v
  for c in 3d_exp_proxy 3d_laplace 2d_medium; do
    echo "[$tag] $(timeout 300 python scripts/profile_matvec.py $c 1 3 2>&1 | tail -1)"
  done
done
