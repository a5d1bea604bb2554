# DIC wavefront: own r/d ring depth decoupled from the one-step edge lead; depth x publish-interval sweep
for dep in 2 8; do CF_DIC_DEPTH=$dep timeout 600 python -m pytest tests -m gpu -x -q -k "dic or DIC" 2>&1 | tail -1; done
for n in 128 256; do
 for dep in 0 2 4 8 12; do for pub in 2 8; do
  echo -n "n=$n depth=$dep pub=$pub "; CF_DIC_DEPTH=$dep CF_DIC_PUBLISH=$pub timeout 300 python tools/dic_probe.py $n 2>&1 | grep dic
 done; done
done
