"""Seeded synthetic input generator shared by the oracle and the CUDA path.

Produces, once per workload and outside every timed region (north_star:
"ordering, inducing points and correlation-distance neighbor sets ... are
produced once during input generation, timed separately, and consumed by both
paths"):

  X    n x d inputs in Vecchia (random) order            (reading c8)
  Z    m x d inducing points: kMeans++ in the ARD-scaled space (c9)
       or a random subset of X (config 1)
  nbr  n x m_v predecessor neighbour sets under the correlation distance d_c
       (exact brute force, reading c6/c7), -1 padded for i < m_v
  y    response: exact dense GP draw + N(0, sigma^2) noise for small n, random
       Fourier features + noise for large n (reading c10')
  theta  covariance parameters

This module holds none of the method's hot-path arithmetic: it never builds
B, D, M or the NLL.  d_c needs whitened features of its own, which it computes
with its own torch code (independent of both oracle/ and the CUDA library).
PRNG: numpy PCG64 seeded by SeedSequence(20250707 + config_id); child streams
in order X, permutation, Z, lambda, y.
"""
from __future__ import annotations

import math
import time
from dataclasses import dataclass, field
from typing import Dict, Optional

import numpy as np

try:
    import torch
except Exception:  # pragma: no cover - torch is in the image
    torch = None

FAMILY_ID = {"matern12": 0, "matern32": 1, "matern52": 2, "gaussian": 3}
SEED_BASE = 20250707

# BASELINE.json "configs" (index + 1 = config id)
CONFIGS: Dict[int, dict] = {
    1: dict(n=2000, d=2, x="uniform", family="matern32", sigma2=1.0, rho=0.1, nugget=0.1, m=50,
            z="subset", mv=10),
    2: dict(n=100_000, d=2, x="uniform", family="matern32", sigma2=1.0, rho=0.05, nugget=0.05, m=200,
            z="kmeans++", mv=20),
    3: dict(n=1_000_000, d=2, x="uniform", family="matern32", sigma2=1.0, rho=0.05, nugget=0.05, m=500,
            z="kmeans++", mv=30),
    4: dict(n=500_000, d=10, x="normal", family="matern52", sigma2=1.0, rho=None, ard=(0.5, 5.0),
            nugget=0.1, m=1000, z="kmeans++", mv=20),
    5: dict(n=4_000_000, d=3, x="uniform", family="matern12", sigma2=1.0, rho=0.1, nugget=0.01, m=1500,
            z="kmeans++", mv=40),
}


@dataclass
class Workload:
    name: str
    X: np.ndarray            # n x d float64, Vecchia order
    Z: np.ndarray            # m x d float64
    nbr: np.ndarray          # n x mv int32
    y: np.ndarray            # n float64
    family: str
    sigma2: float
    lengthscale: np.ndarray  # d float64
    nugget: float
    jitter: float
    timings: Dict[str, float] = field(default_factory=dict)
    latent: Optional[np.ndarray] = None  # latent GP draw of a Laplace workload (y then holds 0/1 labels)

    @property
    def n(self):
        return self.X.shape[0]

    @property
    def d(self):
        return self.X.shape[1]

    @property
    def m(self):
        return self.Z.shape[0]

    @property
    def mv(self):
        return self.nbr.shape[1]

    def theta_dict(self):
        return dict(family=self.family, sigma2=self.sigma2, lengthscale=self.lengthscale.copy(),
                    nugget=self.nugget, jitter=self.jitter)


# ----------------------------------------------------------------------------------------------
# covariance used by the generator only (its own copy: reading c1)
def _cov_from_r(family: str, sigma2: float, r2):
    lib = torch if (torch is not None and isinstance(r2, torch.Tensor)) else np
    r = lib.sqrt(r2)
    if family == "matern12":
        f = lib.exp(-r)
    elif family == "matern32":
        f = (1.0 + math.sqrt(3.0) * r) * lib.exp(-math.sqrt(3.0) * r)
    elif family == "matern52":
        f = (1.0 + math.sqrt(5.0) * r + (5.0 / 3.0) * r2) * lib.exp(-math.sqrt(5.0) * r)
    else:
        f = lib.exp(-r2)
    return sigma2 * f


def _sqdist(A, B):
    """exact pairwise squared distances (no |a|^2+|b|^2-2ab cancellation)"""
    acc = None
    for k in range(A.shape[1]):
        t = A[:, k:k + 1] - B[:, k][None, :]
        t = t * t
        acc = t if acc is None else acc + t
    return acc


def _device(device):
    if device is not None:
        return torch.device(device)
    return torch.device("cuda" if torch.cuda.is_available() else "cpu")


# ----------------------------------------------------------------------------------------------
def kmeanspp(Xs: np.ndarray, m: int, rng: np.random.Generator, iters: int = 10, device=None) -> np.ndarray:
    """kMeans++ (P:501): D^2 seeding, then Lloyd iterations (reading c9), on scaled inputs."""
    n = Xs.shape[0]
    dev = _device(device)
    Xt = torch.from_numpy(Xs).to(dev)
    centers = np.empty((m, Xs.shape[1]))
    first = int(rng.integers(n))
    centers[0] = Xs[first]
    d2 = ((Xt - Xt[first]) ** 2).sum(1)
    for c in range(1, m):
        p = d2.cpu().numpy()
        cs = np.cumsum(p)
        u = rng.random() * cs[-1]
        idx = int(min(np.searchsorted(cs, u, side="right"), n - 1))
        centers[c] = Xs[idx]
        d2 = torch.minimum(d2, ((Xt - Xt[idx]) ** 2).sum(1))
    for _ in range(iters):
        Ct = torch.from_numpy(centers).to(dev)
        lab = torch.empty(n, dtype=torch.int64, device=dev)
        bs = 1 << 16
        for s in range(0, n, bs):
            lab[s:s + bs] = _sqdist(Xt[s:s + bs], Ct).argmin(1)
        lab = lab.cpu().numpy()
        cnt = np.bincount(lab, minlength=m)
        new = np.stack([np.bincount(lab, weights=Xs[:, k], minlength=m) for k in range(Xs.shape[1])], 1)
        keep = cnt > 0
        new[keep] /= cnt[keep, None]
        new[~keep] = centers[~keep]
        if np.array_equal(new, centers):
            break
        centers = new
    return centers


def whitened_features(Xs: np.ndarray, Zs: np.ndarray, family: str, sigma2: float, jitter: float, device=None):
    """u_i = L_m^{-1} k(Z, x_i) for d_c only (generator's own torch implementation)."""
    dev = _device(device)
    m = Zs.shape[0]
    Zt = torch.from_numpy(Zs).to(dev)
    Km = _cov_from_r(family, sigma2, _sqdist(Zt, Zt)) + jitter * torch.eye(m, dtype=torch.float64, device=dev)
    L = torch.linalg.cholesky(Km)
    Xt = torch.from_numpy(Xs).to(dev)
    U = torch.empty((Xs.shape[0], m), dtype=torch.float64, device=dev)
    bs = 1 << 16
    for s in range(0, Xs.shape[0], bs):
        K = _cov_from_r(family, sigma2, _sqdist(Xt[s:s + bs], Zt))
        U[s:s + bs] = torch.linalg.solve_triangular(L, K.T, upper=False).T
    return U


def dc_neighbors(Xs: np.ndarray, Zs: np.ndarray, family: str, sigma2: float, jitter: float, mv: int,
                 device=None, qblock: int = 8192, cblock: int = 65536) -> np.ndarray:
    """m_v nearest predecessors under d_c, exact brute force.

    d_c(i,j) = sqrt(1 - |rho_c(i,j)| / sqrt(rho_c(i,i) rho_c(j,j))), rho_c = Sigma - Sigma_mn^T Sigma_m^-1 Sigma_mn
    (no nugget).  Ranked by (d_c, index) ascending (reading c6).  Degenerate residual
    variance rho_c(j,j) < 1e-7 sigma_1^2 (an inducing point that is also a data point): such a
    candidate gets d_c = 1, and such a query ranks its predecessors by scaled Euclidean distance
    (reading c7).  Rows i <= m_v get all predecessors (reading c5).
    """
    n = Xs.shape[0]
    dev = _device(device)
    out = np.full((n, mv), -1, dtype=np.int32)
    if mv == 0 or n <= 1:
        return out
    Xt = torch.from_numpy(Xs).to(dev)
    m = Zs.shape[0]
    if m > 0:
        U = whitened_features(Xs, Zs, family, sigma2, jitter, device=dev)
        rdiag = sigma2 - (U * U).sum(1)
    else:
        U = None
        rdiag = torch.full((n,), sigma2, dtype=torch.float64, device=dev)
    tau = 1e-7 * sigma2
    degenerate = rdiag < tau
    inv_sd = torch.where(degenerate, torch.zeros_like(rdiag), 1.0 / torch.sqrt(torch.clamp(rdiag, min=tau)))
    for q0 in range(0, n, qblock):
        q1 = min(n, q0 + qblock)
        nq = q1 - q0
        best_v = torch.full((nq, mv), -math.inf, dtype=torch.float64, device=dev)
        best_i = torch.full((nq, mv), -1, dtype=torch.int64, device=dev)
        iq = torch.arange(q0, q1, device=dev)
        for c0 in range(0, q1 - 1, cblock):
            c1 = min(c0 + cblock, q1 - 1)
            score = _cov_from_r(family, sigma2, _sqdist(Xt[q0:q1], Xt[c0:c1]))
            if U is not None:
                score -= U[q0:q1] @ U[c0:c1].T
            score.abs_()
            score *= inv_sd[q0:q1, None]
            score *= inv_sd[None, c0:c1]          # |corr| in [0,1]; degenerate candidates -> 0
            jc = torch.arange(c0, c1, device=dev)
            if c1 > q0:
                score.masked_fill_(jc[None, :] >= iq[:, None], -math.inf)
            cat_v = torch.cat([best_v, score], 1)
            cat_i = torch.cat([best_i, jc[None, :].expand(nq, -1)], 1)
            k = min(mv, cat_v.shape[1])
            v, pos = torch.topk(cat_v, k, dim=1)
            best_v, best_i = v, torch.gather(cat_i, 1, pos)
            del score, cat_v, cat_i
        bv = best_v.cpu().numpy()
        bi = best_i.cpu().numpy()
        for r in range(nq):
            i = q0 + r
            valid = np.isfinite(bv[r]) & (bi[r] >= 0)
            vi, ii = bv[r][valid], bi[r][valid]
            order = np.lexsort((ii, -vi))   # d_c ascending <=> |corr| descending, ties by index
            sel = ii[order][:min(mv, i)]
            out[i, :len(sel)] = sel
    # degenerate queries: scaled-Euclidean nearest predecessors (reading c7)
    dq = torch.nonzero(degenerate).flatten().cpu().numpy()
    for i in dq:
        if i == 0:
            continue
        d2 = ((Xt[:i] - Xt[i]) ** 2).sum(1).cpu().numpy()
        order = np.lexsort((np.arange(i), d2))[:min(mv, i)]
        out[i, :] = -1
        out[i, :len(order)] = order
    return out


def _rff_draw(Xs: np.ndarray, family: str, sigma2: float, rng: np.random.Generator, R: int = 4096, device=None):
    """Approximate zero-mean GP draw by random Fourier features (reading c10').

    Spectral measure of Matern-nu with unit length-scale (inputs pre-scaled): multivariate t with
    2 nu d.o.f.; Gaussian exp(-r^2): N(0, 2 I)."""
    d = Xs.shape[1]
    nu = {"matern12": 0.5, "matern32": 1.5, "matern52": 2.5}.get(family)
    z = rng.standard_normal((R, d))
    if nu is None:
        W = z * math.sqrt(2.0)
    else:
        g = rng.chisquare(2 * nu, size=R)
        W = z * np.sqrt(2 * nu / g)[:, None]
    b = rng.uniform(0, 2 * math.pi, size=R)
    a = rng.standard_normal(R)
    dev = _device(device)
    Xt = torch.from_numpy(Xs).to(dev)
    Wt, bt, at = (torch.from_numpy(v).to(dev) for v in (W, b, a))
    out = torch.empty(Xs.shape[0], dtype=torch.float64, device=dev)
    bs = 1 << 16
    for s in range(0, Xs.shape[0], bs):
        out[s:s + bs] = torch.cos(Xt[s:s + bs] @ Wt.T + bt) @ at
    return (out * math.sqrt(2.0 * sigma2 / R)).cpu().numpy()


def draw_y(Xs: np.ndarray, family: str, sigma2: float, nugget: float, rng: np.random.Generator,
           dense_max: int = 4096, device=None) -> np.ndarray:
    """y = GP draw + N(0, nugget).  Exact dense Cholesky draw for n <= dense_max."""
    n = Xs.shape[0]
    if n <= dense_max:
        K = _cov_from_r(family, sigma2, _sqdist(Xs, Xs)) + 1e-10 * sigma2 * np.eye(n)
        L = np.linalg.cholesky(K)
        b = L @ rng.standard_normal(n)
    else:
        b = _rff_draw(Xs, family, sigma2, rng, device=device)
    return b + math.sqrt(nugget) * rng.standard_normal(n)


def make_workload(n: int, d: int, m: int, mv: int, family: str = "matern32", sigma2: float = 1.0,
                  rho: Optional[float] = 0.1, ard: Optional[tuple] = None, nugget: float = 0.1,
                  x: str = "uniform", z: str = "kmeans++", seed: int = SEED_BASE, device=None,
                  name: str = "custom", neighbors: str = "dc", permute: bool = True,
                  lengthscale: Optional[tuple] = None) -> Workload:
    t0 = time.perf_counter()
    ss = np.random.SeedSequence(seed)
    g_x, g_perm, g_z, g_lam, g_y = (np.random.Generator(np.random.PCG64(s)) for s in ss.spawn(5))
    X = g_x.random((n, d)) if x == "uniform" else g_x.standard_normal((n, d))
    if permute:
        X = X[g_perm.permutation(n)]
    if lengthscale is not None:
        lam = np.asarray(lengthscale, dtype=np.float64)
    elif ard is not None:
        lo, hi = ard
        lam = np.exp(g_lam.uniform(math.log(lo), math.log(hi), size=d))
    else:
        lam = np.full(d, float(rho))
    X = np.ascontiguousarray(X)
    Xs = X / lam
    jitter = 1e-10 * sigma2
    t1 = time.perf_counter()
    if m == 0:
        Z = np.zeros((0, d))
    elif z == "subset":
        Z = X[np.sort(g_z.choice(n, size=m, replace=False))].copy()
    else:
        Z = kmeanspp(Xs, m, g_z, device=device) * lam
    Z = np.ascontiguousarray(Z)
    t2 = time.perf_counter()
    if neighbors == "all":
        nbr = np.full((n, mv), -1, dtype=np.int32)
        for i in range(n):
            k = min(i, mv)
            nbr[i, :k] = np.arange(i - k, i)[::-1] if k else []
    else:
        nbr = dc_neighbors(Xs, Z / lam, family, sigma2, jitter, mv, device=device)
    t3 = time.perf_counter()
    y = draw_y(Xs, family, sigma2, nugget, g_y, device=device)
    t4 = time.perf_counter()
    return Workload(name=name, X=X, Z=Z, nbr=np.ascontiguousarray(nbr, dtype=np.int32), y=y, family=family,
                    sigma2=sigma2, lengthscale=lam, nugget=nugget, jitter=jitter,
                    timings=dict(x=t1 - t0, inducing=t2 - t1, neighbors=t3 - t2, y=t4 - t3))


def make_config(cid: int, device=None, n: Optional[int] = None) -> Workload:
    """BASELINE.json configs[cid-1] (optionally truncated to a smaller n with the same recipe)."""
    c = dict(CONFIGS[cid])
    if n is not None:
        c["n"] = n
    return make_workload(n=c["n"], d=c["d"], m=c["m"], mv=c["mv"], family=c["family"], sigma2=c["sigma2"],
                         rho=c.get("rho"), ard=c.get("ard"), nugget=c["nugget"], x=c["x"], z=c["z"],
                         seed=SEED_BASE + cid, device=device, name=f"config{cid}")


# ----------------------------------------------------------------------------------------------
# prediction inputs (reading p1 in DESIGN.md)
def dc_neighbors_pred(Xs: np.ndarray, Xps: np.ndarray, Zs: np.ndarray, family: str, sigma2: float, jitter: float,
                      mv: int, device=None, qblock: int = 8192, cblock: int = 65536) -> np.ndarray:
    """For each prediction input, the m_v training inputs nearest under d_c, exact brute force,
    ranked by (d_c, index) (reading c6); training candidates with degenerate residual variance get
    d_c = 1 and a degenerate query ranks by scaled Euclidean distance (reading c7).  Coordinates are
    already divided by the length-scales (Xs, Xps, Zs)."""
    n, npred = Xs.shape[0], Xps.shape[0]
    dev = _device(device)
    k = min(mv, n)
    out = np.full((npred, mv), -1, dtype=np.int32)
    if k == 0:
        return out
    Xt = torch.from_numpy(Xs).to(dev)
    Xpt = torch.from_numpy(Xps).to(dev)
    m = Zs.shape[0]
    if m > 0:
        U = whitened_features(Xs, Zs, family, sigma2, jitter, device=dev)
        Up = whitened_features(Xps, Zs, family, sigma2, jitter, device=dev)
        rdiag = sigma2 - (U * U).sum(1)
        rdiag_p = sigma2 - (Up * Up).sum(1)
    else:
        U = Up = None
        rdiag = torch.full((n,), sigma2, dtype=torch.float64, device=dev)
        rdiag_p = torch.full((npred,), sigma2, dtype=torch.float64, device=dev)
    tau = 1e-7 * sigma2
    inv_sd = torch.where(rdiag < tau, torch.zeros_like(rdiag), 1.0 / torch.sqrt(torch.clamp(rdiag, min=tau)))
    degenerate_p = rdiag_p < tau
    inv_sd_p = torch.where(degenerate_p, torch.ones_like(rdiag_p), 1.0 / torch.sqrt(torch.clamp(rdiag_p, min=tau)))
    for q0 in range(0, npred, qblock):
        q1 = min(npred, q0 + qblock)
        nq = q1 - q0
        best_v = torch.full((nq, k), -math.inf, dtype=torch.float64, device=dev)
        best_i = torch.full((nq, k), -1, dtype=torch.int64, device=dev)
        for c0 in range(0, n, cblock):
            c1 = min(c0 + cblock, n)
            score = _cov_from_r(family, sigma2, _sqdist(Xpt[q0:q1], Xt[c0:c1]))
            if U is not None:
                score -= Up[q0:q1] @ U[c0:c1].T
            score.abs_()
            score *= inv_sd_p[q0:q1, None]
            score *= inv_sd[None, c0:c1]
            jc = torch.arange(c0, c1, device=dev)
            cat_v = torch.cat([best_v, score], 1)
            cat_i = torch.cat([best_i, jc[None, :].expand(nq, -1)], 1)
            v, pos = torch.topk(cat_v, k, dim=1)
            best_v, best_i = v, torch.gather(cat_i, 1, pos)
        bv, bi = best_v.cpu().numpy(), best_i.cpu().numpy()
        for r in range(nq):
            order = np.lexsort((bi[r], -bv[r]))
            out[q0 + r, :k] = bi[r][order]
    for pq in torch.nonzero(degenerate_p).flatten().cpu().numpy():
        d2 = ((Xt - Xpt[pq]) ** 2).sum(1).cpu().numpy()
        out[pq, :k] = np.lexsort((np.arange(n), d2))[:k]
    return out


def make_prediction(w: Workload, npred: int, seed: int = SEED_BASE + 100, x: str = "uniform", device=None):
    """Seeded prediction inputs drawn like the training inputs (uniform on the unit cube, or N(0, I)) and
    their d_c neighbour sets among the training points.  Returns (Xp, nbrp)."""
    g = np.random.Generator(np.random.PCG64(np.random.SeedSequence(seed)))
    d = w.X.shape[1]
    Xp = g.random((npred, d)) if x == "uniform" else g.standard_normal((npred, d))
    Xp = np.ascontiguousarray(Xp)
    lam = np.asarray(w.lengthscale, dtype=np.float64)
    nbrp = dc_neighbors_pred(w.X / lam, Xp / lam, w.Z.reshape(-1, d) / lam, w.family, w.sigma2, w.jitter, w.mv,
                             device=device)
    return Xp, np.ascontiguousarray(nbrp, dtype=np.int32)


# ----------------------------------------------------------------------------------------------
# VIF-Laplace inputs
LAPLACE_LENGTHSCALE = (0.15, 0.30, 0.45, 0.60, 0.75)  # d = 5, ARD Gaussian covariance


def make_laplace_workload(n: int, d: int = 5, m: int = 200, mv: int = 30, family: str = "gaussian",
                          sigma2: float = 1.0, lengthscale: Optional[tuple] = None, rho: Optional[float] = None,
                          seed: int = SEED_BASE + 40, device=None, neighbors: str = "dc",
                          z: str = "kmeans++") -> Workload:
    """Binary responses from a latent GP: b = zero-mean GP draw (no error term), y_i ~
    Bernoulli(1 / (1 + exp(-b_i))).  Same recipe as make_workload with nugget 0 (the latent process has
    no error variance); the Bernoulli draw uses a sixth child stream.  ``w.y`` holds the labels
    (0.0 / 1.0) and ``w.latent`` the draw b."""
    if lengthscale is None and rho is None:
        lengthscale = LAPLACE_LENGTHSCALE[:d] if d <= len(LAPLACE_LENGTHSCALE) else None
        rho = None if lengthscale is not None else 0.3
    w = make_workload(n=n, d=d, m=m, mv=mv, family=family, sigma2=sigma2, rho=rho, nugget=0.0, z=z, seed=seed,
                      device=device, name="laplace", neighbors=neighbors, lengthscale=lengthscale)
    rng = np.random.Generator(np.random.PCG64(np.random.SeedSequence(seed).spawn(6)[5]))
    b = w.y
    w.latent = b
    w.y = (rng.random(n) < 1.0 / (1.0 + np.exp(-b))).astype(np.float64)
    return w


def make_probes(n: int, m: int, nprobe: int, seed: int = SEED_BASE + 41):
    """Standard normal draws for the SLQ probe vectors z_i = D_V^{1/2} eps2_i + U eps1_i:
    eps1 (m x ell) and eps2 (n x ell), row-major."""
    rng = np.random.Generator(np.random.PCG64(seed))
    eps1 = np.ascontiguousarray(rng.standard_normal((m, nprobe)))
    eps2 = np.ascontiguousarray(rng.standard_normal((n, nprobe)))
    return eps1, eps2
