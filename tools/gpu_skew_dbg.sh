# skewed-warp DIC sweeps: where (if anywhere) they differ from the level schedule, then the
# per-step pace on boxes of 1, 2, 8 tiles in x / y and the whole 256^3 cube
set -x
timeout 300 python tools/skew_debug.py 48x48x48 32x4x16 64x4x16 32x8x16 32x4x48 70x9x5 2>&1 | grep -v "^+" | tee gpurun_out/skew_debug.log
for sh in "32 8 256" "64 8 256" "32 16 256" "256 8 256" "32 256 256" "128 128 256" "256 256 256"; do
  timeout 300 python tools/dic_shape_probe.py $sh 2>&1 | tail -1
done 2>&1 | tee gpurun_out/skew_shapes.log
