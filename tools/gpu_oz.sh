cd /root/repo
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_int8.py -x -q > gpurun_out/oz_t8.log 2>&1; echo "rc=$?" >> gpurun_out/oz_t8.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/oz_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/oz_tests.log
for c in 5; do
  QTB_TRACE=1 timeout 300 python bench.py --config $c --no-cpu-baseline --steps 5 --warmup 3 > gpurun_out/oz_bench_c$c.json 2> gpurun_out/oz_bench_c$c.err; echo "c$c rc=$?" >> gpurun_out/oz_tests.log
done
