"""vif_gram: G = W^T W (A6 / K4, "M") on the integer tensor cores (int8 digit slices, tcgen05 kind::i8,
k_ozaki.cu) and on the FP64 DMMA engine, against an exact reference.

The reference is computed in float128-free exact arithmetic where it matters: each G entry is a plain dot
product; numpy's float64 matmul (pairwise/blocked summation) has error ~ k * 2^-53 * sum|w_a||w_b|, so the
comparison tolerance is derived from that bound (plus the slices' 2^-54 column-relative representation)."""
import numpy as np
import pytest
import torch

import paper_2507_05064_b200 as p

pytestmark = pytest.mark.gpu


def _ref(W):
    return W.T @ W


def _bound(W):
    A = np.abs(W)
    k = W.shape[0]
    # FP64 reference error + slice representation (2^-54 of the column maximum per factor) per term
    cm = A.max(0)
    return 4 * k * 2.0 ** -52 * (A.T @ A) + 4 * k * 2.0 ** -53 * np.outer(cm, cm) + 1e-300


@pytest.mark.parametrize("engine", ["int8", "fp64"])
@pytest.mark.parametrize("n,c", [(1, 1), (7, 3), (100, 64), (1000, 130), (40000, 512), (20000, 333), (70000, 1001)])
def test_gram_matches_reference(engine, n, c):
    rng = np.random.default_rng(n * 7919 + c)
    W = rng.standard_normal((n, c)) * np.exp(rng.uniform(-3, 3, size=c))  # columns of very different scales
    Wt = torch.from_numpy(W).cuda()
    G = p.vif_gram(Wt, engine).cpu().numpy()
    torch.cuda.synchronize()
    R = _ref(W)
    err = np.abs(G - R)
    assert np.all(err <= _bound(W)), (engine, float((err / _bound(W)).max()))


def test_gram_multichunk_and_int32_limit():
    """more rows than one digit-slice chunk (2^20) and than one int32 accumulation (16,384 rows) with every
    entry at the digit extremes: the level sums would overflow int32 if a unit ever spanned more rows"""
    n, c = (1 << 20) + 4099, 72
    W = torch.full((n, c), -1.0, dtype=torch.float64, device="cuda")
    W[::2] = 1.0 - 2.0 ** -40
    G = p.vif_gram(W, "int8").cpu().numpy()
    Wh = W.cpu().numpy()
    R = Wh.T @ Wh
    assert np.allclose(G, R, rtol=1e-13, atol=0)


def test_gram_nonfinite_gives_nan():
    W = torch.randn(5000, 64, dtype=torch.float64, device="cuda")
    W[1234, 5] = float("nan")
    G = p.vif_gram(W, "int8").cpu().numpy()
    assert np.isnan(G).all()


def test_gram_engines_agree_on_factor_rows():
    """the two engines on a W with the structure of the factor's rows (whitened residual rows + y column)"""
    rng = np.random.default_rng(3)
    n, c = 200000, 505
    W = rng.standard_normal((n, c)) * np.linspace(0.01, 3.0, c)
    Wt = torch.from_numpy(W).cuda()
    Gi = p.vif_gram(Wt, "int8").cpu().numpy()
    Gf = p.vif_gram(Wt, "fp64").cpu().numpy()
    assert np.max(np.abs(Gi - Gf)) <= 1e-12 * np.abs(Gf).max()


@pytest.mark.parametrize("cid,n", [(1, None), (4, 20000)])
def test_factor_engines_agree(monkeypatch, cid, n):
    """vif_factor + vif_nll + vif_grad with the integer-slice contractions (default) and with the DMMA ones
    (VIF_UFEAT_FP64=1, VIF_SYRK_FP64=1, VIF_GRAD_FP64=1, read at vif_create): U rows agree to 1e-12 (normwise: the oracle
    parity bound of U; measured 1.1e-13 at config 4's m = 1000) and the NLL terms
    to 1e-12 relative (config 4 recipe: d = 10, m = 1000, ld = 1008)"""
    import sys, os
    sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
    import vifgen
    w = vifgen.make_config(cid, device="cuda", n=n)
    th = p.Theta(**w.theta_dict())
    dev = torch.device("cuda")
    res, U, G = {}, {}, {}
    for eng in ("int8", "fp64"):
        for var in ("VIF_SYRK_FP64", "VIF_UFEAT_FP64", "VIF_GRAD_FP64"):
            if eng == "fp64":
                monkeypatch.setenv(var, "1")
            else:
                monkeypatch.delenv(var, raising=False)
        m = p.VifModel(*(torch.from_numpy(np.ascontiguousarray(a)).to(dev) for a in (w.X, w.Z, w.nbr, w.y)))
        t = m.evaluate(th)
        res[eng] = (t.nll, t.logdet_D, t.logdet_M, t.quad)
        U[eng] = m.U().cpu().numpy()
        G[eng] = np.asarray(m.grad(th)[1])
        m.close()
    for a, b in zip(res["int8"], res["fp64"]):
        assert abs(a - b) <= 1e-12 * max(abs(b), 1.0), (res,)
    du = np.linalg.norm(U["int8"] - U["fp64"], axis=1) / np.maximum(np.linalg.norm(U["fp64"], axis=1), 1e-300)
    assert du.max() <= 1e-12, du.max()
    # the gradient (its Gamma, T and G2 contractions on the integer engines too) to 1e-9 of the largest component
    np.testing.assert_allclose(G["int8"], G["fp64"], rtol=0, atol=1e-9 * np.abs(G["fp64"]).max())


def _exact_gram(W):
    """G = W^T W in exact rational arithmetic: every double is m * 2^e with integer m, so each product and sum is
    an exact Python integer at a common exponent; returns the exactly rounded float64 G"""
    from fractions import Fraction
    n, c = W.shape
    F = [[Fraction(float(v)) for v in row] for row in W]
    G = np.zeros((c, c))
    for a in range(c):
        for b in range(a + 1):
            s = sum(F[k][a] * F[k][b] for k in range(n))
            G[a, b] = G[b, a] = float(s)
    return G


def test_gram_int8_error_within_reading_c18_bound():
    """DESIGN reading c18: per entry |G_int8 - G_exact| <= K * 2^-54 * max|w_a| * max|w_b| + 2^-52 |G_exact|
    (one rounding of each operand to 55 bits of its column maximum, dropped digit levels below 2^-51 of the
    product of the maxima, exact int32 level sums, FP64 combination), checked against an exact rational
    reference on columns spanning 2^-200 .. 2^200 and rows spanning 2^-20 .. 2^20 (a column-relative bound:
    small entries of a column carry the column maximum's absolute precision, like FP64's own dot-product bound)"""
    rng = np.random.default_rng(2507)
    n, c = 257, 24
    W = rng.standard_normal((n, c))
    W *= np.exp2(rng.uniform(-20, 20, size=(n, 1)))
    W *= np.exp2(np.linspace(-200, 200, c))[None, :]
    W[:, 7] = 0.0  # an all-zero column
    G = p.vif_gram(torch.from_numpy(W).cuda(), "int8").cpu().numpy()
    E = _exact_gram(W)
    cm = np.abs(W).max(0)
    bound = n * 2.0 ** -54 * np.outer(cm, cm) + 2.0 ** -52 * np.abs(E)
    err = np.abs(G - E)
    assert np.all(err <= bound), float(np.max(err / np.maximum(bound, 1e-300)))
    assert np.all(G[7] == 0.0) and np.all(G[:, 7] == 0.0)
