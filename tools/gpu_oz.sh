cd /root/repo
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_int8.py -x -q > gpurun_out/oz_t8.log 2>&1; echo "rc=$?" >> gpurun_out/oz_t8.log
