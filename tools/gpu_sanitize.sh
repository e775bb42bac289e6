# usage: bash tools/gpu_sanitize.sh TOOL   (racecheck | synccheck | memcheck); plain run first
TOOL=${1:-racecheck}
timeout 600 python tools/sanitize_kernels.py > gpurun_out/sanitize_plain.log 2>&1; rc=$?
echo "plain rc $rc"; tail -3 gpurun_out/sanitize_plain.log
if [ $rc -eq 0 ]; then
  timeout 2400 /usr/local/cuda/bin/compute-sanitizer --tool $TOOL --print-limit 50 python tools/sanitize_kernels.py > gpurun_out/sanitize_$TOOL.log 2>&1
  echo "$TOOL rc $?"; tail -8 gpurun_out/sanitize_$TOOL.log
fi
