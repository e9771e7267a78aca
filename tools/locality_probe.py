import numpy as np, sys, os
sys.path.insert(0, os.getcwd())
import vifgen
w = vifgen.make_config(3, device="cuda", n=200000)
X = w.X
q = np.clip((X * 65535).astype(np.int64), 0, 65535)
def spread(v):
    v = (v | (v << 8)) & 0x00FF00FF
    v = (v | (v << 4)) & 0x0F0F0F0F
    v = (v | (v << 2)) & 0x33333333
    v = (v | (v << 1)) & 0x55555555
    return v
code = spread(q[:, 0]) | (spread(q[:, 1]) << 1)
order = np.argsort(code, kind="stable")
pos = np.empty(len(order), np.int64); pos[order] = np.arange(len(order))
nb = w.nbr
ii = np.repeat(np.arange(w.n), nb.shape[1]); jj = nb.ravel(); ok = jj >= 0
d = np.abs(pos[ii[ok]] - pos[jj[ok]])
print("n", w.n, "pairs", ok.sum(), "median |dpos|", np.median(d), "p90", np.percentile(d, 90), "p99", np.percentile(d, 99))
# spatial distance parent-child
sd = np.linalg.norm(X[ii[ok]] - X[jj[ok]], axis=1)
print("median spatial dist", np.median(sd), "p90", np.percentile(sd, 90), "mean NN spacing", 1/np.sqrt(w.n))
