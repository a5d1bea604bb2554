# A/B of kernel forms inside the sustained bench (power-capped clocks matter)
for rep in 1 2 3; do
for v in "CF_PAIR_PF=0" "CF_PAIR_PF=1"; do
  env $v python bench.py --no-cpu-baseline 2>/dev/null | python3 -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v' or 'default', round(d['value']), round(d['fused_iter_us'],1), d['clocks']['sm_mhz'])"
done; done
CF_PAIR_PF=1 timeout 600 python -m pytest tests -m gpu -x -q -k "lean or cg" 2>&1 | tail -1
CF_PAIR_PF=1 CF_CG_DIRECT=8 timeout 600 ncu --metrics gpu__time_duration.sum -k regex:cg_dir_lean2 -c 3 python tools/probe_cg.py --n 256 --iters 20 --repeat 1 2>&1 | grep duration
