cd /root/repo
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_int8.py -x -q > gpurun_out/oz_t8.log 2>&1; echo "rc=$?" >> gpurun_out/oz_t8.log
timeout 120 python tools/oz_profile_run.py > gpurun_out/ozp.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/oz_launches.csv python tools/oz_profile_run.py >> gpurun_out/ozp.log 2>&1; echo "rc=$?" >> gpurun_out/ozp.log
