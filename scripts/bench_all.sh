# bench.py on every BASELINE config that is not the default (nrhs=1), one line each
for c in 2d_tiny 2d_medium 3d_laplace sweep; do
  timeout 900 python bench.py --config $c --no-cpu-baseline > gpurun_out/bench_$c.log 2>&1; echo "$c rc $?"
done
timeout 900 python bench.py --config 3d_sphere --no-cpu-baseline > gpurun_out/bench_3d_sphere.log 2>&1; echo "3d_sphere rc $?"
