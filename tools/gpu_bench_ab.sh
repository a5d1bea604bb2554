# A/B of two library builds inside the sustained bench (CF_LIB)
for rep in 1 2 3; do
for v in old new; do
  CF_LIB=tools/variants/$v.so python bench.py --no-cpu-baseline 2>/dev/null | python3 -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v', round(d['value']), round(d['fused_iter_us'],1), d['clocks']['sm_mhz'])"
done; done
CF_LIB=tools/variants/new.so timeout 600 python -m pytest tests -m gpu -x -q -k "cg or pcg or deferred or lean or parity" 2>&1 | tail -1
