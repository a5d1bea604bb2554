timeout 600 python tools/dic_shape_probe.py 2>&1 | grep tiles
for pub in 1000000; do echo "pub=$pub"; NSHAPES=2 CF_DIC_PUBLISH=$pub timeout 600 python tools/dic_shape_probe.py 2>&1 | grep tiles; done
CF_DIC_DEPTH=0 timeout 600 python tools/dic_shape_probe.py 2>&1 | grep tiles | head -3
timeout 600 ncu --set full --clock-control none --import-source on -k regex:dic_wave_fwd_p -s 3 -c 1 -o gpurun_out/dic_full python tools/dic_probe.py 128 > gpurun_out/ncu_dic.log 2>&1; echo ncu=$?
