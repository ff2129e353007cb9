# A/B of the phase-2 NR=16 stage geometry: adopted default vs the previous one (libhh_p2old).
cd "$(dirname "$0")/.."
for r in 1 2; do
  for v in default p2old; do
    if [ "$v" = default ]; then lib=paper_2604_09147_b200/libhh.so; else lib=paper_2604_09147_b200/libhh_$v.so; fi
    for c in "3d_exp_proxy 16" "3d_laplace 16" "3d_sphere 16" "3d_laplace 20"; do
      HH_LIB=$PWD/$lib timeout 300 python scripts/profile_matvec.py $c 3 2>&1 | grep nrhs= | sed "s/^/[$v] /"
    done
  done
done
