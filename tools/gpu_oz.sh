cd /root/repo
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/oz_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/oz_tests.log
timeout 300 python bench.py --config 5 --no-cpu-baseline --steps 5 --warmup 3 --sharded > gpurun_out/oz_bench_c5s.json 2> gpurun_out/oz_bench_c5s.err; echo "c5s rc=$?" >> gpurun_out/oz_tests.log
