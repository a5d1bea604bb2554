# round-1 DIC mailbox evidence: full GPU tests, DIC-PCG timings, ncu launch list + full capture of the sweeps at 128^3
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -1 gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 600 python tools/dic_probe.py 128 256 2>&1 | tee gpurun_out/dic_probe.txt
CF_DIC_LEVELS=1 timeout 600 python tools/dic_probe.py 128 2>&1 | grep dic | sed 's/^/levels: /' | tee -a gpurun_out/dic_probe.txt
CF_CG_DIRECT=8 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:dic_wave -c 20 --csv --log-file gpurun_out/dic_launches.csv python tools/dic_probe.py 128 > gpurun_out/ncu_dic_l.log 2>&1; echo ncu=$?
CF_CG_DIRECT=8 timeout 600 ncu --set full --clock-control none --import-source on -k regex:dic_wave_fwd_p -s 4 -c 1 -o gpurun_out/dic_full128 python tools/dic_probe.py 128 > gpurun_out/ncu_dic.log 2>&1; echo ncufull=$?
