for t in 5 6 7; do echo "tile=$t"; CF_DIC_TILE=$t timeout 300 python -m pytest tests -m gpu -x -q -k "dic or DIC" 2>&1 | tail -1; CF_DIC_TILE=$t timeout 300 python tools/dic_probe.py 128 256 2>&1 | grep dic; done
echo "tile=0"; timeout 300 python tools/dic_probe.py 128 256 2>&1 | grep dic
