timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu.log
timeout 600 python tools/dic_probe.py 512 2>&1 | grep dic | tee gpurun_out/dic512.log
for i in 1 2; do python tools/dic_step_probe.py 40; done 2>&1 | tee gpurun_out/dic_probe.txt
