# single-tile pace vs own-data ring depth, then crossings at depth 2 / 8; ncu of the one-tile forward sweep
for dep in 2 4 8 12; do echo "depth=$dep"; NSHAPES=7 CF_DIC_DEPTH=$dep timeout 600 python tools/dic_shape_probe.py 2>&1 | grep tiles; done
cat > /tmp/one.py <<'PY'
import sys; sys.path.insert(0, '.')
import numpy as np, torch, paper_2504_03697_b200 as cf
shp = (16, 8, 256)
b = np.random.default_rng(0).uniform(-1, 1, 16 * 8 * 256); b -= b.mean()
op = cf.StencilOperator(256, 1 / 256, "sym", shape=shp)
for _ in range(2): x, st = cf.pcg(op, torch.as_tensor(b, device="cuda"), precond=cf.dic_from(op), tol=1e-8, max_iter=50)
print(st.iterations)
PY
CF_CG_DIRECT=8 timeout 600 ncu --set full --clock-control none --import-source on -k regex:dic_wave_fwd_p -s 5 -c 1 -o gpurun_out/dic_one python /tmp/one.py > gpurun_out/ncu_dic.log 2>&1; echo ncu=$?
