set -x
timeout 300 python tools/skew_debug.py 48x48x48 32x4x16 64x4x16 32x8x16 32x4x48 70x9x5 2>&1 | grep -v "^+" | tee gpurun_out/skew_debug.log
for sh in "32 4 256" "64 4 256" "32 8 256" "256 4 256" "32 256 256" "256 256 256"; do
  for sk in 1; do echo "shape $sh skew=$sk"; CF_DIC_SKEW=$sk timeout 300 python tools/dic_shape_probe.py $sh 2>&1 | tail -1; done
done 2>&1 | tee gpurun_out/skew_shapes.log
for J in 2 8; do echo "J=$J"; CF_DIC_J=$J timeout 300 python tools/dic_shape_probe.py 256 256 256 2>&1 | tail -1; done 2>&1 | tee -a gpurun_out/skew_shapes.log
