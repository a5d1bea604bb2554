for rep in 1 2; do
for cfg in "8 0" "8 2" "4 0" "4 2"; do set -- $cfg
 echo -n "rows=$1 pf=$2 "; CF_LEAN_ROWS=$1 CF_PAIR_PF=$2 python tools/probe_cg.py --n 256 --iters 300 --repeat 2
done; done
CF_PAIR_PF=2 timeout 900 python -m pytest tests -m gpu -x -q -k "lean or cg or pcg" 2>&1 | tail -1
CF_PAIR_PF=2 CF_CG_DIRECT=8 timeout 600 ncu --set full --clock-control none --import-source on -k regex:cg_dir_lean -s 4 -c 1 -o gpurun_out/dir_pf2 python tools/probe_cg.py --n 256 --iters 20 --repeat 1 > gpurun_out/ncu_full.log 2>&1; echo ncufull=$?
