cd /root/repo
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_int8.py -x -q > gpurun_out/oz_t8.log 2>&1; echo "rc=$?" >> gpurun_out/oz_t8.log
timeout 300 python bench.py --config 5 --no-cpu-baseline --steps 5 --warmup 3 --e2e-steps 1 > gpurun_out/oz_bench_c5.json 2> gpurun_out/oz_bench_c5.err; echo "c5 rc=$?" >> gpurun_out/oz_t8.log
QTB_OZAKI_PIPE=0 timeout 300 python bench.py --config 5 --no-cpu-baseline --steps 5 --warmup 3 --e2e-steps 0 > gpurun_out/oz_bench_c5_seq.json 2> gpurun_out/oz_bench_c5_seq.err; echo "c5 seq rc=$?" >> gpurun_out/oz_t8.log
