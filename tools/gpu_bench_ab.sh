# A/B of kernel forms inside the sustained bench (power-capped clocks matter)
for rep in 1 2 3; do
for v in "CF_LEAN_ROWS=8" "CF_LEAN_ROWS=16"; do
  env $v python bench.py --no-cpu-baseline 2>/dev/null | python3 -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v' or 'default', round(d['value']), round(d['fused_iter_us'],1), d['clocks']['sm_mhz'], round(d['roofline']['design_frac'],3), d['roofline']['dram_frac'])"
done; done
CF_LEAN_ROWS=16 timeout 600 python -m pytest tests -m gpu -x -q -k "lean or cg" 2>&1 | tail -1
