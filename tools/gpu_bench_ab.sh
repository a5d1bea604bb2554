# A/B of kernel forms inside the sustained bench (power-capped clocks matter)
for rep in 1 2 3; do
for v in "CF_LEAN2=0" "CF_LEAN2=1"; do
  env $v python bench.py --no-cpu-baseline 2>/dev/null | python3 -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v' or 'default', round(d['value']), round(d['fused_iter_us'],1), d['clocks']['sm_mhz'])"
done; done
