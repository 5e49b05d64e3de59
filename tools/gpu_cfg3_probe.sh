# Config-3 (p = 4096) FFT passes: launch list and one full capture of each pass kernel,
# plus an A/B of frequency-batch sizes on the config-5 step.
cd /root/repo
mkdir -p gpurun_out
timeout 300 python bench.py --config 3 --steps 5 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/c3_plain.json 2>&1; echo "c3 rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 60 --csv \
  --log-file gpurun_out/c3_launches.csv python bench.py --config 3 --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline > gpurun_out/c3_ncu1.log 2>&1; echo "ncu list rc=$?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"tube_fft" -c 2 -o gpurun_out/c3_fft \
  python bench.py --config 3 --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline > gpurun_out/c3_ncu2.log 2>&1; echo "ncu full rc=$?"
ENVS="QTB_X=0;QTB_OZAKI_WS_MB=3072;QTB_OZAKI_WS_MB=1536;QTB_OZAKI_WS_MB=4608" STEPS=10 bash tools/ab.sh > gpurun_out/ab2.log 2>&1
