# Round-2 (session 3) refresh: GPU tests, bench lines of every config, the
# reference arm, launch lists and full captures of the kernels changed this
# session (one-launch small product, warp-specialised tiny K2), into gpurun_out/.
cd /root/repo
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/rf3_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/rf3_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/rf3_smoke.log 2>&1; echo "smoke rc=$?"
for c in 5 4 2 3 1; do
  extra=""; [ $c != 5 ] && extra="--no-cpu-baseline"
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 $extra > gpurun_out/rf3_bench_cfg$c.json 2> gpurun_out/rf3_bench_cfg$c.err
  echo "cfg$c rc=$?"
done
timeout 600 python bench.py --impl reference --config 5 --steps 2 --warmup 1 > gpurun_out/rf3_reference_cfg5.json 2> gpurun_out/rf3_reference_cfg5.err; echo "ref rc=$?"
for c in 1 3; do
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 80 --csv \
    --log-file gpurun_out/rf3_launches_cfg$c.csv python bench.py --config $c --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline > gpurun_out/rf3_ncu_list$c.log 2>&1
  echo "ncu list cfg$c rc=$?"
done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:small_tprod -c 1 -o gpurun_out/rf3_ncu_small \
  python bench.py --config 1 --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline > gpurun_out/rf3_ncu_small.log 2>&1; echo "ncu small rc=$?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"paired_tiny|tube_fft" -c 5 -o gpurun_out/rf3_ncu_cfg3 \
  python bench.py --config 3 --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline > gpurun_out/rf3_ncu_cfg3.log 2>&1; echo "ncu cfg3 rc=$?"
timeout 120 ./tools/microbench/small_trace > gpurun_out/rf3_small_trace.txt 2>&1; echo "trace rc=$?"
