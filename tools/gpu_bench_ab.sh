# A/B of kernel forms inside the sustained bench (power-capped clocks matter)
for rep in 1 2 3; do
for v in "CF_DOUBLE_STAGES=3" "CF_DOUBLE_STAGES=4"; do
  env $v python bench.py --no-cpu-baseline 2>/dev/null | python3 -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v' or 'default', round(d['value']), round(d['fused_iter_us'],1), d['clocks']['sm_mhz'])"
done; done
CF_DOUBLE_STAGES=4 timeout 600 python -m pytest tests -m gpu -x -q -k "cg or pcg or deferred or lean" 2>&1 | tail -1
