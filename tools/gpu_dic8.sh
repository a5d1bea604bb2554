for ns in 0 20 50 100 200 500; do echo "spin_ns=$ns"; CF_DIC_SPIN_NS=$ns NSHAPES=10 timeout 300 python tools/dic_shape_probe.py 2>&1 | grep -E "tiles|Error" | sed -n '7p;9,10p'; done
