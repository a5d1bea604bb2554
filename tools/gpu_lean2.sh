for rep in 1 2; do for l in 0 1; do
 echo -n "lean2=$l "; CF_LEAN2=$l python tools/probe_cg.py --n 256 --iters 300 --repeat 2
 echo -n "lean2=$l "; CF_LEAN2=$l python tools/probe_cg.py --n 512 --iters 60 --repeat 2
done; done
CF_LEAN2=1 timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
CF_LEAN2=1 CF_CG_DIRECT=8 timeout 600 ncu --set full --clock-control none -k regex:cg_dir_lean2 -s 4 -c 1 -o gpurun_out/lean2 python tools/probe_cg.py --n 256 --iters 20 --repeat 1 > /dev/null 2>&1; echo ncu=$?
