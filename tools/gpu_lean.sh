for rep in 1 2; do
for rows in 4 8 16; do
 echo -n "rows=$rows lean/lean "; CF_LEAN_ROWS=$rows CF_CG_DIR=lean CF_CG_UPD=lean python tools/probe_cg.py --n 256 --iters 300 --repeat 2
 echo -n "rows=$rows lean/tma "; CF_LEAN_ROWS=$rows CF_CG_DIR=lean CF_CG_UPD=tma python tools/probe_cg.py --n 256 --iters 300 --repeat 2
 echo -n "rows=$rows lean/lean "; CF_LEAN_ROWS=$rows CF_CG_DIR=lean CF_CG_UPD=lean python tools/probe_cg.py --n 512 --iters 60 --repeat 2
done; done
CF_LEAN_ROWS=16 CF_CG_DIR=lean CF_CG_UPD=lean timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
