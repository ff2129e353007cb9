for i in 1 2; do
HH_P1_ROWS=100000000 timeout 600 python scripts/profile_matvec.py 3d_large 1 3 2>&1 | tail -1 | sed 's/^/[nosplit] /'
timeout 600 python scripts/profile_matvec.py 3d_large 1 3 2>&1 | tail -1 | sed 's/^/[split] /'
done
