for rep in 1 2 3; do
for d in 4 8 9 13; do for u in 4 9; do
  echo -n "256 d=$d u=$u: "; CF_PAIR_CHUNKS_DIR=$d CF_TMA_CHUNKS_UPD=$u python tools/probe_cg.py --n 256 --iters 300 --repeat 2
done; done; done
for rep in 1 2; do
for d in 9 16 ; do for u in 1 9 16 32 64; do
  echo -n "512 d=$d u=$u: "; CF_PAIR_CHUNKS_DIR=$d CF_TMA_CHUNKS_UPD=$u python tools/probe_cg.py --n 512 --iters 60 --repeat 2
done; done; done
