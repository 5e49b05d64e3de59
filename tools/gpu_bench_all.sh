# Bench lines of every config (default arm) and the reference arm, into gpurun_out/ba_*.json
cd /root/repo
mkdir -p gpurun_out
for c in 5 4 2 3 1; do
  extra=""; [ $c != 5 ] && extra="--no-cpu-baseline"
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 $extra > gpurun_out/ba_bench_cfg$c.json 2> gpurun_out/ba_bench_cfg$c.err
  echo "cfg$c rc=$?"
done
timeout 600 python bench.py --impl reference --config 5 --steps 2 --warmup 1 > gpurun_out/ba_reference_cfg5.json 2> gpurun_out/ba_reference_cfg5.err; echo "ref rc=$?"
