# A/B of environment variants of the default bench step: ENVS="A=1 B=2;A=0 B=2" bash tools/ab.sh
# (QTB_LIB_PATH=<other build> runs another build of the library; KT=1 also prints per-kernel ms per step)
IFS=';' read -ra VS <<< "$ENVS"
for rep in $(seq 1 ${REPS:-2}); do
  for v in "${VS[@]}"; do
    env $v timeout -s KILL 150 python bench.py --config ${CFG:-5} --steps ${STEPS:-8} --warmup 3 --e2e-steps 0 --no-cpu-baseline 2>/dev/null \
      | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1])
kt = {k: round(v, 2) for k, v in d['roofline'].get('kernel_times_ms_per_step', {}).items()} if '${KT:-0}' == '1' else ''
print('$v', round(d['ms_per_step'],3), d['clocks']['sm_mhz'], kt)"
  done
done
