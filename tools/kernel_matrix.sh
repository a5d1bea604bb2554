#!/bin/bash
# CG kernel-form matrix (us per iteration) at the given sizes.
for n in ${SIZES:-256 512}; do
  for d in ${DIRS:-pair tma stage}; do for u in ${UPDS:-pair tma}; do
    echo -n "n=$n dir=$d upd=$u: "; CF_CG_DIR=$d CF_CG_UPD=$u python tools/probe_cg.py --n $n --iters 100 --repeat 2
  done; done
done
