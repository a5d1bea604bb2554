# spass forms (us per iteration) + correctness on odd boxes
python tools/spass_check.py 48 128 96x80x72 130x66x40 66x34x20 200x30x9
for f in 2 1; do
  echo "== FORM=$f 256"; CF_SPASS_FORM=$f timeout 120 python tools/probe_cg.py --n 256 --iters 200 --repeat 2
  echo "== FORM=$f 512"; CF_SPASS_FORM=$f timeout 120 python tools/probe_cg.py --n 512 --iters 60 --repeat 2
done
CF_CG_DIRECT=2 timeout 600 ncu --set full --clock-control none --import-source on -k regex:cg_spass -s 4 -c 2 -o gpurun_out/spass_f2 python tools/probe_cg.py --n 256 --iters 10 --repeat 1 > gpurun_out/spass_ncu.log 2>&1; echo ncu=$?
