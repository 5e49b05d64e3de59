cd /root/repo
mkdir -p gpurun_out/sweep
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/sweep/tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/sweep/tests.log
for c in 5 4 2 3 1; do
  timeout 600 python bench.py --config $c > gpurun_out/sweep/bench_cfg$c.json 2> gpurun_out/sweep/bench_cfg$c.err; echo "cfg$c rc=$?"
done
timeout 300 python bench.py --steps 2 --warmup 1 --e2e-steps 1 --no-cpu-baseline > gpurun_out/sweep/plain.json 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/sweep/launches_bench_cfg5.csv python bench.py --steps 2 --warmup 1 --e2e-steps 1 --no-cpu-baseline > gpurun_out/sweep/ncu.log 2>&1; echo "ncu rc=$?"
