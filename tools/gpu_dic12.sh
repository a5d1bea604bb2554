for L in 2 4 8; do echo "rlook=$L"; CF_DIC_RLOOK=$L timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "wavefront_matches_levels" 2>&1 | tail -1; CF_DIC_RLOOK=$L timeout 300 python tools/dic_shape_probe.py 2>&1 | grep -E "tiles|Error" | sed -n '1p;7p;9,10p'; done
echo base; timeout 300 python tools/dic_shape_probe.py 2>&1 | grep -E "tiles|Error" | sed -n '1p;7p;9,10p'
