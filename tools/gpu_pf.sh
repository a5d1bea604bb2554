for i in 1 2; do
for pf in 0 1; do
 CF_PAIR_PF=$pf python tools/probe_cg.py --n 256 --iters 200 --repeat 3 | sed "s/^/pf=$pf /"
 CF_PAIR_PF=$pf python tools/probe_cg.py --n 512 --iters 50 --repeat 2 | sed "s/^/pf=$pf /"
done; done
CF_PAIR_PF=1 timeout 300 python -m pytest tests -m gpu -x -q -k "cg or pcg" 2>&1 | tail -2
CF_CG_DIRECT=8 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 1 > gpurun_out/ncu.log 2>&1; echo ncu=$?
CF_PAIR_PF=1 CF_CG_DIRECT=8 timeout 600 ncu --set full --clock-control none --import-source on -k regex:cg_dir_pair -s 4 -c 1 -o gpurun_out/dir_pf python tools/probe_cg.py --n 256 --iters 20 --repeat 1 > gpurun_out/ncu_full.log 2>&1; echo ncufull=$?
