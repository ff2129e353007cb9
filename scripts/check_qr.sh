python scripts/profile_matvec.py 3d_large 1 1 > gpurun_out/plain_q.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,launch__grid_size,launch__shared_mem_per_block_dynamic --clock-control none -k regex:"k_(qr|jacobi|gemm_gen)" --csv --log-file gpurun_out/launches_qr.csv python scripts/profile_matvec.py 3d_large 1 1 > gpurun_out/ncu_q.log 2>&1; echo rc $?
