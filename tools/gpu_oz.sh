cd /root/repo
mkdir -p gpurun_out
timeout 600 python tools/oz_sweep.py > gpurun_out/oz_sweep.log 2>&1; echo "rc=$?" >> gpurun_out/oz_sweep.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/oz_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/oz_tests.log
