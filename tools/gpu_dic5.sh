timeout 600 python -m pytest tests -m gpu -x -q -k "dic or DIC" 2>&1 | tail -1
for dep in 2 4; do echo "depth=$dep"; CF_DIC_DEPTH=$dep timeout 600 python tools/dic_shape_probe.py 2>&1 | grep tiles; done
