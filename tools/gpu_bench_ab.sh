# A/B of kernel forms inside the sustained bench (power-capped clocks matter)
for rep in 1 2 3; do
for v in "CF_CHUNK_REV=0" "CF_CHUNK_REV=1"; do
  env $v python bench.py --no-cpu-baseline 2>/dev/null | python3 -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v' or 'default', round(d['value']), round(d['fused_iter_us'],1), d['clocks']['sm_mhz'])"
done; done
for v in 0 1; do echo -n "rev=$v 512 "; CF_CHUNK_REV=$v python tools/probe_cg.py --n 512 --iters 60 --repeat 2; echo -n "rev=$v 256 "; CF_CHUNK_REV=$v python tools/probe_cg.py --n 256 --iters 300 --repeat 2; done
CF_CHUNK_REV=1 CF_CG_DIRECT=8 timeout 600 ncu --cache-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum -k regex:"cg_dir|cg_update" -c 8 python tools/probe_cg.py --n 256 --iters 20 --repeat 1 2>&1 | grep -E "cg_dir|cg_update|duration|bytes_read" | paste - - - | awk '{print $2, $(NF-4), $NF}'
CF_CHUNK_REV=0 CF_CG_DIRECT=8 timeout 600 ncu --cache-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum -k regex:"cg_dir|cg_update" -c 8 python tools/probe_cg.py --n 256 --iters 20 --repeat 1 2>&1 | grep -E "cg_dir|cg_update|duration|bytes_read" | paste - - - | awk '{print $2, $(NF-4), $NF}'
