# Round check on one B200: smoke, GPU tests, bench (both arms), launch list, full capture, configs.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu.log
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?
python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref=$?
cat gpurun_out/bench.json gpurun_out/bench_ref.json
CF_CG_DIRECT=8 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 1 > gpurun_out/ncu.log 2>&1; echo ncu=$?
CF_CG_DIRECT=8 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"cg_dir_lean|cg_update_tma" -s 6 -c 4 -o gpurun_out/cg_full python tools/probe_cg.py --n 256 --iters 20 --repeat 1 > gpurun_out/ncu_full.log 2>&1; echo ncufull=$?
timeout 1200 python tools/bench_configs.py > gpurun_out/configs.json 2> gpurun_out/configs.err; echo cfg=$?
