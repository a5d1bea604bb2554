for rep in 1 2; do for p in 0 1; do
 echo -n "pdl=$p "; CF_PDL=$p python tools/probe_cg.py --n 256 --iters 300 --repeat 2
 echo -n "pdl=$p "; CF_PDL=$p python tools/probe_cg.py --n 512 --iters 60 --repeat 2
 echo -n "pdl=$p "; CF_PDL=$p python tools/probe_cg.py --n 128 --iters 300 --repeat 2
done; done
CF_PDL=1 timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
