# A/B of environment variants of the default bench step: ENVS="A=1 B=2;A=0 B=2" bash tools/ab.sh
IFS=';' read -ra VS <<< "$ENVS"
for rep in 1 2; do
  for v in "${VS[@]}"; do
    env $v timeout -s KILL 120 python bench.py --steps ${STEPS:-8} --warmup 3 --e2e-steps 0 --no-cpu-baseline 2>/dev/null \
      | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v', round(d['ms_per_step'],2), d['clocks']['sm_mhz'])"
  done
done
