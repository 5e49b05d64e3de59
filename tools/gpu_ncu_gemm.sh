cd /root/repo
mkdir -p gpurun_out
timeout 300 python bench.py --config 5 --no-cpu-baseline --steps 1 --warmup 1 --e2e-steps 0 > gpurun_out/ncu_plain.json 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"oz_gemm2" -c 1 -o gpurun_out/ncu_cfg5_int8gemm_v2 python bench.py --config 5 --no-cpu-baseline --steps 1 --warmup 1 --e2e-steps 0 > gpurun_out/ncu_run.log 2>&1; echo "ncu rc=$?"
