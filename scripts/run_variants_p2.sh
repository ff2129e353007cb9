# Time the phase-2 NR=16 variants (scripts/variants_p2.sh) with CUDA events, two rounds.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for r in 1 2; do
  for v in default peel p2s3_x8 p2s3_x8_peel p2s2_w24_x8 p2s3_x6; do
    if [ "$v" = default ]; then lib=paper_2604_09147_b200/libhh.so; else lib=paper_2604_09147_b200/libhh_$v.so; fi
    for c in "3d_exp_proxy 16" "3d_laplace 16"; do
      HH_LIB=$PWD/$lib timeout 300 python scripts/profile_matvec.py $c 3 2>&1 | grep nrhs= | sed "s/^/[$v] /"
    done
  done
done
