"""Union of conditioning sets per Morton cluster (VERDICT r1 'next' 3: does a shared union Gram per
cluster of P points beat the per-point Gram?).  Reads the neighbour sets of a cached workload
(tools/vecchia_probe.py / step_probe.py cache, or generates the config-3 recipe at n points).
For clusters of P consecutive points in the Morton processing order: |T| = |union of S_i|, the 8x8
tiles of one dense union Gram (ceil(|T|/8) choose 2 + diagonal) vs P x the per-point tiles.
  python tools/union_probe.py [n] [config]"""
import json, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1000000
cid = int(sys.argv[2]) if len(sys.argv) > 2 else 3
cache = f"/tmp/vif_probe_c{cid}_{n}.npz"
if os.path.exists(cache):
    z = np.load(cache)
    X, nbr = z["X"], z["nbr"]
else:
    import vifgen
    w = vifgen.make_config(cid, device="cuda", n=n)
    X, nbr = w.X, w.nbr
    np.savez(cache, X=w.X, Z=w.Z, nbr=w.nbr, y=w.y, theta=json.dumps({**w.theta_dict(), "lengthscale": [float(v) for v in w.lengthscale]}))
n, d = X.shape
mv = nbr.shape[1]
Xn = (X - X.min(0)) / (X.max(0) - X.min(0) + 1e-12)
dd = min(d, 3)
bits = 63 // dd
q = np.minimum((Xn[:, :dd] * (1 << bits)).astype(np.uint64), (1 << bits) - 1)
code = np.zeros(n, dtype=np.uint64)
for b in range(bits):
    for k in range(dd):
        code |= ((q[:, k] >> np.uint64(b)) & np.uint64(1)) << np.uint64(b * dd + k)
order = np.argsort(code, kind="stable")
s = mv + 1
rb = -(-s // 8)
rng = np.random.default_rng(1)
out = {"n": n, "d": d, "mv": mv, "config": cid, "clusters": []}
for P in (1, 2, 4, 8, 16, 32, 64):
    starts = rng.integers(0, n - P, 300) // P * P
    sizes = []
    for c0 in starts:
        pts = order[c0:c0 + P]
        T = set(pts.tolist())
        for i in pts:
            T.update(int(j) for j in nbr[i] if j >= 0)
        sizes.append(len(T))
    sizes = np.array(sizes, dtype=np.float64)
    blocks = np.ceil(sizes / 8)
    tu = float(np.mean(blocks * (blocks + 1) / 2))
    tp = P * rb * (rb + 1) / 2
    out["clusters"].append({"P": P, "T_mean": float(sizes.mean()), "P_times_s": P * s, "union_tiles": tu,
                            "per_point_tiles": tp, "ratio": tu / tp})
print(json.dumps(out))
