cd /root/repo
mkdir -p gpurun_out
for i in 1 2; do
QTB_OZAKI_PIPE=0 timeout 300 python bench.py --config 5 --no-cpu-baseline --steps 5 --warmup 3 --e2e-steps 0 > gpurun_out/oz_bench_c5_seq$i.json 2> /dev/null
timeout 300 python bench.py --config 5 --no-cpu-baseline --steps 5 --warmup 3 --e2e-steps 0 > gpurun_out/oz_bench_c5_pipe$i.json 2> /dev/null
done
