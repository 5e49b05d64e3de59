cd /root/repo
mkdir -p gpurun_out
timeout 300 python bench.py --config 5 --no-cpu-baseline --steps 5 --warmup 3 --e2e-steps 1 > gpurun_out/oz_bench_c5.json 2> gpurun_out/oz_bench_c5.err; echo "c5 rc=$?"
timeout 300 python bench.py --config 1 --no-cpu-baseline --steps 5 --warmup 3 --e2e-steps 1 > gpurun_out/oz_bench_c1.json 2> gpurun_out/oz_bench_c1.err; echo "c1 rc=$?"
