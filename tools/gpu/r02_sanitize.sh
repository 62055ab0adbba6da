set -x
mkdir -p gpurun_out/san
timeout 900 python tools/sanitize_cases.py > gpurun_out/san/plain.log 2>&1; echo "plain rc=$?"; tail -2 gpurun_out/san/plain.log
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize_cases.py > gpurun_out/san/$tool.log 2>&1; echo "$tool rc=$?"; tail -3 gpurun_out/san/$tool.log
done
