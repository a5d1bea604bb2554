for p in 0 1; do
 for n in 64 96 128 144; do echo -n "persist=$p "; CF_PERSIST=$p python tools/probe_cg.py --n $n --iters 300 --repeat 3; done
done
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
