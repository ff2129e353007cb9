timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2
for c in 3d_exp_proxy 3d_laplace; do for r in 8 16; do echo "$(timeout 300 python scripts/profile_matvec.py $c $r 3 2>&1 | tail -1)"; done; done
