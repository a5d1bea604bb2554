# spass schedules (us per iteration) + correctness on odd boxes
CF_SPASS_SCHED=phase python tools/spass_check.py 48 128 96x80x72 130x66x40 256
for sch in items phase; do
  echo "== SCHED=$sch"; CF_SPASS_SCHED=$sch python tools/probe_cg.py --n 256 --iters 200 --repeat 2; CF_SPASS_SCHED=$sch python tools/probe_cg.py --n 512 --iters 60 --repeat 2
done
CF_SPASS_SCHED=phase CF_CG_DIRECT=2 timeout 600 ncu --set full --clock-control none --import-source on -k regex:cg_spass -s 4 -c 2 -o gpurun_out/spass_phase python tools/probe_cg.py --n 256 --iters 10 --repeat 1 > gpurun_out/spass_ncu.log 2>&1; echo ncu=$?
