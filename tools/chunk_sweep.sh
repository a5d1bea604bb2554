#!/bin/bash
# Chunk-count sweep of the two default CG kernels (us per fused iteration).
n=${N:-256}
for c in ${DIRC:-4 5 6 8 9 12 16}; do
  echo -n "dir_chunks=$c: "; CF_PAIR_CHUNKS_DIR=$c python tools/probe_cg.py --n $n --iters 200 --repeat 2
done
for c in ${UPDC:-2 3 4 6 8}; do
  echo -n "upd_chunks=$c: "; CF_TMA_CHUNKS_UPD=$c python tools/probe_cg.py --n $n --iters 200 --repeat 2
done
