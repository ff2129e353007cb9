set -x
export HH_PROFILE_BUILD=1
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo smoke rc $?
timeout 600 python bench.py --config 2d_medium --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_2dmed.log 2>&1; echo rc $?
timeout 900 python bench.py --config 3d_laplace --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_3dlap.log 2>&1; echo rc $?
timeout 2400 python bench.py --config 3d_large --steps 10 --warmup 3 > gpurun_out/bench_3dlarge.log 2>&1; echo rc $?
nvidia-smi --query-gpu=memory.used,memory.total --format=csv
