import sys
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import numpy as np
from test_gpu_scale import problem
from paper_1711_01897_b200.hmatrix import AcaConfig, assemble_hmatrix, hmat_matvec
v, e, spec, sp, bt = problem(12, "p0", "laplace", "slp", 0.0)
h = assemble_hmatrix(spec, sp, sp, bt, AcaConfig(epsilon=1e-5))
x = np.random.default_rng(7).standard_normal(sp.n_dofs)
yd = hmat_matvec(h, x, device=True)
yh = hmat_matvec(h, x, device=False)
# long-double reference over the leaf payloads
rp, cp = bt.rows.permutation, bt.cols.permutation
rn, cn = bt.rows.node_array, bt.cols.node_array
yl = np.zeros(sp.n_dofs, np.longdouble)
worst = (0, None)
for ix, (r, c, _) in enumerate(bt.leaf_array):
    rows = rp[rn[r, 0]: rn[r, 1]]; cols = cp[cn[c, 0]: cn[c, 1]]
    pl = h.payloads[ix]
    xs = x[cols].astype(np.longdouble)
    if hasattr(pl, "u"):
        t = pl.u.astype(np.longdouble) @ (pl.v.T.astype(np.longdouble) @ xs)
        contrib = np.abs(pl.u) @ (np.abs(pl.v.T) @ np.abs(x[cols]))
        if contrib.max() > worst[0]: worst = (contrib.max(), ix, pl.rank, pl.u.shape, pl.v.shape)
    else:
        t = pl.a.astype(np.longdouble) @ xs
    yl[rows] += t
sc = np.abs(yh).max()
print("device vs ld", float(np.abs(yd - yl).max() / sc), "host vs ld", float(np.abs(yh - yl).max() / sc))
print("worst |u||v||x| contribution", worst, "vs |y| max", sc)
