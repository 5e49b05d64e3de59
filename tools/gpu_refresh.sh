# Round-end refresh: GPU tests, bench lines of every config, the reference arm,
# the config-5 launch list and one full capture of the int8 GEMM (into gpurun_out/).
cd /root/repo
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/rf_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/rf_pytest.log
for c in 5 4 2 3 1; do
  extra=""; [ $c != 5 ] && extra="--no-cpu-baseline"
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 $extra > gpurun_out/rf_bench_cfg$c.json 2> gpurun_out/rf_bench_cfg$c.err
  echo "cfg$c rc=$?"
done
timeout 600 python bench.py --impl reference --config 5 --steps 2 --warmup 1 > gpurun_out/rf_reference_cfg5.json 2> gpurun_out/rf_reference_cfg5.err; echo "ref rc=$?"
timeout 600 python bench.py --sharded --multi freq --steps 5 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/rf_bench_cfg5_freq1.json 2> gpurun_out/rf_freq1.err; echo "freq1 rc=$?"
timeout 600 python bench.py --sharded --multi rows --steps 5 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/rf_bench_cfg5_rows1.json 2> gpurun_out/rf_rows1.err; echo "rows1 rc=$?"
python tools/profile_step.py --config 5 --warmup 1 --steps 1 > /dev/null 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/rf_launches_cfg5.csv python tools/profile_step.py --config 5 --warmup 0 --steps 2 > gpurun_out/rf_ncu1.log 2>&1
echo "ncu list rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"oz_gemm2" -c 1 -o gpurun_out/rf_ncu_gemm \
  python tools/profile_step.py --config 5 --warmup 0 --steps 1 > gpurun_out/rf_ncu2.log 2>&1
echo "ncu full rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"oz_residue_b|oz_residue_a|oz_crt|oz_guard|oz_balance|oz_colexp" -c 7 -o gpurun_out/rf_ncu_aux \
  python tools/profile_step.py --config 5 --warmup 0 --steps 1 > gpurun_out/rf_ncu3.log 2>&1
echo "ncu aux rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/rf_smoke.log 2>&1; echo "smoke rc=$?"
timeout 300 python tools/timeline.py > gpurun_out/rf_timeline.log 2>&1; echo "timeline rc=$?"
