# DIC wavefront sweeps on one B200 (replaces round 1's gpu_dic*.sh one-offs).
#   bash tools/gpu_dic_sweep.sh VAR "v1 v2 ..." [probe]
# VAR: an env switch of csrc/cf_dic_wave.cu (CF_DIC_DEPTH, CF_DIC_TILE, CF_DIC_RLOOK,
# CF_DIC_SPIN_NS, CF_DIC_PUBLISH, CF_DIC_LEVELS); probe: shape (tools/dic_shape_probe.py,
# per-diagonal pace over tile counts) or pcg (tools/dic_probe.py 128 256, DIC-PCG us per
# iteration; the default).  Each value first runs the DIC GPU tests (bit-identity vs levels).
var=${1:?VAR}; vals=${2:?values}; probe=${3:-pcg}
for v in $vals; do
  echo "== $var=$v"
  env "$var=$v" timeout 300 python -m pytest tests -m gpu -x -q -k "dic or DIC" 2>&1 | tail -1
  if [ "$probe" = shape ]; then env "$var=$v" timeout 300 python tools/dic_shape_probe.py 2>&1 | grep -E "tiles|Error"
  else env "$var=$v" timeout 300 python tools/dic_probe.py 128 256 2>&1 | grep dic; fi
done
