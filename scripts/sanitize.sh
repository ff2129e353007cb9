# compute-sanitizer on a small end-to-end case (one tool per gpurun call; never on a
# program that faulted).  usage: bash scripts/sanitize.sh memcheck|racecheck|synccheck|initcheck
tool=${1:-memcheck}
timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 \
  python scripts/profile_matvec.py 2d_tiny 2 1 > gpurun_out/sanitize_$tool.log 2>&1
echo "$tool rc $?"
tail -5 gpurun_out/sanitize_$tool.log
