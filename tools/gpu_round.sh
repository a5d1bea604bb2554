# Round check on one B200: smoke, GPU tests, bench (both arms), CG launch list,
# the consolidated per-kernel ncu table (two launch lists: step kernels on the
# cavity, CG kernels on a dense right-hand side), full capture of the CG pass.
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?; tail -1 gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu.log
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?
python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref=$?
cat gpurun_out/bench.json gpurun_out/bench_ref.json
CF_CG_DIRECT=8 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 1 --no-extra --no-cpu-baseline > gpurun_out/ncu.log 2>&1; echo ncu=$?
for part in step cg; do
  CF_CG_DIRECT=2 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/table_$part.csv python tools/ncu_table.py 256 $part > gpurun_out/table_$part.log 2>&1; echo table_$part=$?
done
CF_CG_DIRECT=2 timeout 600 ncu --set full --clock-control none --import-source on -k regex:cg_spass -s 4 -c 2 -o gpurun_out/round_cg_full python tools/probe_cg.py --n 256 --iters 10 --repeat 1 > gpurun_out/ncu_full.log 2>&1; echo ncufull=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:advect_tma -s 1 -c 1 -o gpurun_out/round_adv_full python tools/advect_check.py 256 0.5 > gpurun_out/ncu_adv.log 2>&1; echo ncuadv=$?
python tools/slab_projection.py 1 2 4 8 > gpurun_out/slab_projection.txt 2>&1; echo proj=$?
for i in 1 2 3; do python tools/dic_step_probe.py 40; done > gpurun_out/dic_probe.txt 2>&1; echo dic=$?
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --force-slabs --no-cpu-baseline > gpurun_out/bench_slabs.json 2> gpurun_out/bench_slabs.err; echo slabs=$?
python tools/slab_probe.py --n 256 --iters 100 --slabs 1,2,4,8 > gpurun_out/slab_probe.txt 2>&1; echo slabprobe=$?
timeout 1200 python tools/bench_configs.py > gpurun_out/configs.json 2> gpurun_out/configs.err; echo cfg=$?
bash tools/gpu_skew_ncu.sh > gpurun_out/skew_ncu.out 2>&1; echo skewncu=$?
bash tools/gpu_skew_dbg.sh > gpurun_out/skew_dbg.out 2>&1; echo skewdbg=$?
timeout 300 python tools/dic_probe.py 128 256 2>&1 | grep dic > gpurun_out/dic_sizes.txt; echo dicsizes=$?
