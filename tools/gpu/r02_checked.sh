set -x
timeout 900 python -m pytest tests/test_gpu_checked.py -x -q > gpurun_out/r02_checked.log 2>&1; echo "checked rc=$?"; tail -5 gpurun_out/r02_checked.log
