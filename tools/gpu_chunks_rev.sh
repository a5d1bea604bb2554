for rep in 1 2; do
for cfg in "13 9" "13 13" "9 9" "18 9" "13 7" "11 9"; do set -- $cfg
  echo -n "dir=$1 upd=$2 "; CF_LEAN_CHUNKS=$1 CF_TMA_CHUNKS_UPD=$2 python tools/probe_cg.py --n 256 --iters 300 --repeat 2
done; done
