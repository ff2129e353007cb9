# Time the phase-1 NR>=8 variants (scripts/variants_p1.sh) with CUDA events, two rounds.
cd "$(dirname "$0")/.."
for r in 1 2; do
  for v in default p1_w40_x12 p1_w48_x8 p1_w36_x16 p1_w44_x10; do
    if [ "$v" = default ]; then lib=paper_2604_09147_b200/libhh.so; else lib=paper_2604_09147_b200/libhh_$v.so; fi
    for c in "3d_exp_proxy 16" "3d_laplace 16" "3d_sphere 16"; do
      HH_LIB=$PWD/$lib timeout 300 python scripts/profile_matvec.py $c 3 2>&1 | grep nrhs= | sed "s/^/[$v] /"
    done
  done
done
