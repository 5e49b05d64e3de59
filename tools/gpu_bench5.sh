cd /root/repo
mkdir -p gpurun_out
timeout 300 python bench.py --config 5 --no-cpu-baseline --steps 5 --warmup 3 > gpurun_out/oz_bench_c5.json 2> gpurun_out/oz_bench_c5.err; echo "c5 rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/oz_bench_c5.json')); print(d['ms_per_step'], d['value'], {k:(v.get('ms'), v.get('TFLOP_s')) for k,v in d['stages'].items()}, d['e2e']['ms_per_step'], d['clocks'])"
