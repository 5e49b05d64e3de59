cd /root/repo
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_int8.py -x -q > gpurun_out/oz_t8.log 2>&1; echo "t8 rc=$?"; tail -2 gpurun_out/oz_t8.log
for c in 5; do
timeout 300 python bench.py --config $c --no-cpu-baseline --steps 5 --warmup 3 > gpurun_out/oz_bench_c$c.json 2> gpurun_out/oz_bench_c$c.err; echo "c$c rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/oz_bench_c$c.json')); r=d['roofline']; print(d['ms_per_step'], d['value'], r['achieved'], r['frac'], r['kernel_ms'], r['kernel_times_ms_per_step'], d['e2e']['ms_per_step'], d['clocks'], d['gpu_launches'])"
done
timeout 120 python tools/oz_profile_run.py > gpurun_out/ozp.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/oz_launches.csv python tools/oz_profile_run.py >> gpurun_out/ozp.log 2>&1; echo "ncu rc=$?"
