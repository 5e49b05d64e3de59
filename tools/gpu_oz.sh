cd /root/repo
mkdir -p gpurun_out
for i in 1 2; do timeout 300 python bench.py --config 3 --no-cpu-baseline --steps 20 --warmup 5 --e2e-steps 0 > gpurun_out/c3_$i.json 2>/dev/null; done
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "transforms or long_tube or shapes" > gpurun_out/c3t.log 2>&1; echo rc=$? >> gpurun_out/c3t.log
