for sh in "128 256 256" "256 128 256" "256 256 128" "256 256 256"; do CF_DIC_SKEW=1 timeout 300 python tools/dic_shape_probe.py $sh 2>&1 | tail -1; done 2>&1 | tee gpurun_out/skew_shapes3.log
