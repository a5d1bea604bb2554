for rep in 1 2; do
 echo -n "tma/tma "; python tools/probe_cg.py --n 256 --iters 300 --repeat 2
 echo -n "skip=lean "; CF_CG_UPD_SKIP=lean python tools/probe_cg.py --n 256 --iters 300 --repeat 2
 echo -n "upd=lean "; CF_CG_UPD=lean python tools/probe_cg.py --n 256 --iters 300 --repeat 2
 echo -n "skip=lean 512 "; CF_CG_UPD_SKIP=lean python tools/probe_cg.py --n 512 --iters 60 --repeat 2
 echo -n "tma/tma 512 "; python tools/probe_cg.py --n 512 --iters 60 --repeat 2
done
