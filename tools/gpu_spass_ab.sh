# spass vs two-kernel (us per iteration), correctness on odd boxes
python tools/spass_check.py 64 128 96x80x72 130x66x40 256
echo "== spass 256"; CF_CG_ALGO=spass timeout 120 python tools/probe_cg.py --n 256 --iters 200 --repeat 2
echo "== spass 512"; CF_CG_ALGO=spass timeout 120 python tools/probe_cg.py --n 512 --iters 60 --repeat 2
echo "== two 256"; timeout 120 python tools/probe_cg.py --n 256 --iters 200 --repeat 2
CF_CG_ALGO=spass CF_CG_DIRECT=2 timeout 600 ncu --set full --clock-control none --import-source on -k regex:cg_spass -s 4 -c 2 -o gpurun_out/spass_full4 python tools/probe_cg.py --n 256 --iters 10 --repeat 1 > gpurun_out/spass_ncu.log 2>&1; echo ncu=$?
