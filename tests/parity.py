"""Parity criteria between the CUDA path and the oracle (reading c14; north_star tolerances).

  NLL   |dNLL| / |NLL_ref| <= 1e-8   (term scale used when |NLL_ref| < 1e-3 sum |terms|)
  terms logdet_D, logdet_M, quad relative <= 1e-10 (absolute floor 1e-10 * term scale)
  D     elementwise relative <= 1e-9
  B     per row  max|dB_i| <= 1e-9 * max(max|B_i,ref|, 1e-3)
  U     ||dU||_F / ||U||_F <= 1e-12
"""
import numpy as np

NLL_RTOL = 1e-8
TERM_RTOL = 1e-10
D_RTOL = 1e-9
B_RTOL = 1e-9
U_RTOL = 1e-12


def check_terms(gpu, ref_nll, ref_ld, ref_lm, ref_q):
    scale = abs(ref_ld) + abs(ref_lm) + abs(ref_q)
    den = abs(ref_nll) if abs(ref_nll) >= 1e-3 * scale else scale
    assert abs(gpu.nll - ref_nll) <= NLL_RTOL * den, (gpu.nll, ref_nll)
    for name, g, r in (("logdet_D", gpu.logdet_D, ref_ld), ("logdet_M", gpu.logdet_M, ref_lm),
                       ("quad", gpu.quad, ref_q)):
        assert abs(g - r) <= TERM_RTOL * max(abs(r), 1e-10 * scale, 1e-300), (name, g, r)


def check_D(D, Dref):
    D, Dref = np.asarray(D), np.asarray(Dref)
    rel = np.abs(D - Dref) / np.abs(Dref)
    assert np.all(np.isfinite(D))
    assert rel.max() <= D_RTOL, ("D", rel.max(), int(rel.argmax()))


def check_B(B, Bref):
    B, Bref = np.asarray(B), np.asarray(Bref)
    if B.shape[1] == 0:
        return
    err = np.abs(B - Bref).max(1)
    scale = np.maximum(np.abs(Bref).max(1), 1e-3)
    worst = (err / scale).max()
    assert worst <= B_RTOL, ("B", worst, int((err / scale).argmax()))


def check_U(U, Uref):
    U, Uref = np.asarray(U), np.asarray(Uref)
    if U.size == 0:
        return
    rel = np.linalg.norm(U - Uref) / np.linalg.norm(Uref)
    assert rel <= U_RTOL, ("U", rel)
