set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo smoke rc $?
timeout 300 python scripts/gpu_debug.py 2d_tiny > gpurun_out/dbg_tiny.log 2>&1; echo dbg rc $?
timeout 300 python scripts/gpu_debug.py 3d_small_exp > gpurun_out/dbg_3dexp.log 2>&1; echo dbg rc $?
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc $?
tail -5 gpurun_out/pytest_gpu.log
