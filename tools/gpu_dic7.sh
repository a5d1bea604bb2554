timeout 300 python -m pytest tests -m gpu -x -q -k "dic or DIC" 2>&1 | tail -2
for dep in 2 3 4 6; do echo "depth=$dep"; CF_DIC_DEPTH=$dep timeout 300 python tools/dic_shape_probe.py 2>&1 | grep -E "tiles|Error" | sed -n '1p;3p;7p;9,10p'; done
