timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2
HH_PROFILE_BUILD=1 timeout 300 python scripts/profile_matvec.py 3d_laplace 1 3 2>&1 | tail -4
HH_PROFILE_BUILD=1 timeout 900 python scripts/profile_matvec.py 3d_large 1 3 2>&1 | tail -4
