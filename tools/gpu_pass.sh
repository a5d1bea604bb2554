for f in lean lean16; do CF_PASS_FORM=$f timeout 300 python -m pytest tests -m gpu -x -q -k "single_reduction" 2>&1 | tail -1; done
for i in 1 2; do
echo -n "two  "; python tools/probe_cg.py --n 256 --iters 300 --repeat 2
for f in lean lean16; do
echo -n "$f "; CF_PASS_FORM=$f CF_CG_ALGO=pass python tools/probe_cg.py --n 256 --iters 300 --repeat 2
echo -n "$f 512 "; CF_PASS_FORM=$f CF_CG_ALGO=pass python tools/probe_cg.py --n 512 --iters 60 --repeat 2
done; done
CF_CG_ALGO=pass CF_CG_DIRECT=8 timeout 600 ncu --set full --clock-control none --import-source on -k regex:cg_lpass -s 4 -c 1 -o gpurun_out/lpass_full python tools/probe_cg.py --n 256 --iters 20 --repeat 1 > gpurun_out/ncu_full.log 2>&1; echo ncufull=$?
