# skewed-warp DIC sweeps: parity tests, then DIC-PCG time per iteration for each tile height
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_box.py -x -q -m gpu -k "dic or DIC" 2>&1 | tail -15 > gpurun_out/skew_tests.log
cat gpurun_out/skew_tests.log
for J in 4 8; do
  echo "J=$J"; CF_DIC_J=$J timeout 300 python tools/dic_probe.py 128 256 2>&1 | grep dic
done 2>&1 | tee gpurun_out/skew_probe.log
echo "tiled wavefront"; CF_DIC_SKEW=0 timeout 300 python tools/dic_probe.py 128 256 2>&1 | grep dic | tee -a gpurun_out/skew_probe.log
