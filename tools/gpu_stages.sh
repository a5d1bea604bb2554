for rep in 1 2; do for st in 3 4 6; do
 echo -n "skip_stages=$st "; CF_SKIP_STAGES=$st python tools/probe_cg.py --n 256 --iters 300 --repeat 2
 echo -n "skip_stages=$st "; CF_SKIP_STAGES=$st python tools/probe_cg.py --n 512 --iters 60 --repeat 2
done; done
for st in 4 6; do CF_SKIP_STAGES=$st timeout 600 python -m pytest tests -m gpu -x -q -k "cg or pcg or deferred" 2>&1 | tail -1; done
