for dep in 0 2 3 4 6; do
 echo -n "depth=$dep "; CF_DIC_DEPTH=$dep python tools/dic_probe.py 256 2>&1 | grep dic
done
for dep in 0 3 4; do
 echo -n "depth=$dep "; CF_DIC_DEPTH=$dep python tools/dic_probe.py 128 2>&1 | grep dic
done
for dep in 3 4; do CF_DIC_DEPTH=$dep timeout 600 python -m pytest tests -m gpu -x -q -k "dic or DIC" 2>&1 | tail -1; done
