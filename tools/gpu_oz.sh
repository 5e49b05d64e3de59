cd /root/repo
mkdir -p gpurun_out
QTB_OZAKI_PIPE=0 timeout 300 python bench.py --config 5 --no-cpu-baseline --steps 5 --warmup 3 --e2e-steps 0 > gpurun_out/oz_bench_c5_seq1.json 2> /dev/null
timeout 120 python tools/oz_profile_run.py > gpurun_out/ozp.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/oz_launches.csv python tools/oz_profile_run.py >> gpurun_out/ozp.log 2>&1; echo "ncu rc=$?"
