timeout 300 python -m pytest tests -m gpu -x -q -k "dic or DIC" 2>&1 | tail -1
timeout 300 python tools/dic_shape_probe.py 2>&1 | grep -E "tiles|Error" | sed -n '1p;7p;9,10p'
timeout 300 python tools/dic_probe.py 128 256 2>&1 | grep dic
