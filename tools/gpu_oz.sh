cd /root/repo
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "grid2d or chunked" > gpurun_out/oz_t8.log 2>&1; echo "rc=$?" >> gpurun_out/oz_t8.log
timeout 600 python tools/rank_emul.py > gpurun_out/rank_emul.log 2>&1; echo rc=$? >> gpurun_out/rank_emul.log
timeout 300 python bench.py --config 5 --no-cpu-baseline --steps 5 --warmup 3 --e2e-steps 1 --sharded > gpurun_out/oz_bench_c5s.json 2> gpurun_out/oz_bench_c5s.err; echo "c5s rc=$?" >> gpurun_out/oz_t8.log
