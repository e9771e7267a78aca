"""Thin Python binding of libvif.so (include/vif.h): argument marshalling only.

Every step of the VIF factor + NLL runs in the CUDA kernels of libvif.so; PyTorch only
supplies device memory (the workspace is a torch uint8 tensor), the CUDA stream and, for
world > 1, the process group used to broadcast the 128-byte NCCL id.  There is no CPU
fallback: if libvif.so is missing or CUDA is unavailable the calls raise.

Names mirror the C ABI: vif_workspace_bytes, vif_partition, vif_create, vif_set_data,
vif_factor, vif_nll, vif_copy_U, vif_launch_count, vif_last_error, vif_destroy,
vif_nccl_unique_id.  `VifModel` is a convenience owner of one handle + its workspace.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass
from typing import Optional, Sequence, Union

import numpy as np
import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libvif.so")

FAMILIES = {"matern12": 0, "matern32": 1, "matern52": 2, "gaussian": 3}
STATUS = {0: "VIF_OK", 1: "VIF_ERR_INVALID_ARG", 2: "VIF_ERR_NOT_PD", 3: "VIF_ERR_CUDA", 4: "VIF_ERR_NCCL",
          5: "VIF_ERR_NO_MEMORY", 6: "VIF_ERR_STATE"}


class VifError(RuntimeError):
    def __init__(self, status: int, msg: str, bad_row: int = -1):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status, self.msg, self.bad_row = status, msg, bad_row


class _Dims(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int64), ("d", ctypes.c_int32), ("m", ctypes.c_int32), ("mv", ctypes.c_int32),
                ("rank", ctypes.c_int32), ("world", ctypes.c_int32)]


class _Theta(ctypes.Structure):
    _fields_ = [("family", ctypes.c_int32), ("d", ctypes.c_int32), ("sigma2", ctypes.c_double),
                ("lengthscale", ctypes.POINTER(ctypes.c_double)), ("nugget", ctypes.c_double),
                ("jitter", ctypes.c_double)]


class _LaOpts(ctypes.Structure):
    _fields_ = [("max_newton", ctypes.c_int32), ("newton_tol", ctypes.c_double), ("max_cg", ctypes.c_int32),
                ("cg_tol", ctypes.c_double), ("nprobe", ctypes.c_int32), ("slq_tol", ctypes.c_double)]


class _LaTerms(ctypes.Structure):
    _fields_ = [("nll", ctypes.c_double), ("neg_loglik", ctypes.c_double), ("quad", ctypes.c_double),
                ("logdet", ctypes.c_double), ("logdet_W", ctypes.c_double), ("logdet_P", ctypes.c_double),
                ("newton_iters", ctypes.c_int32), ("cg_iters", ctypes.c_int32), ("slq_iters_max", ctypes.c_int32),
                ("slq_iters_mean", ctypes.c_double)]


class _Terms(ctypes.Structure):
    _fields_ = [("nll", ctypes.c_double), ("logdet_D", ctypes.c_double), ("logdet_M", ctypes.c_double),
                ("quad", ctypes.c_double), ("bad_row", ctypes.c_int64)]


_lib = None


def load_library():
    """Load libvif.so (built in-tree by __graft_entry__.build()); raise loudly if it is missing."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} not built: run `python -c 'import __graft_entry__ as g; g.build()'`")
        lib = ctypes.CDLL(LIB_PATH)
        P, i32, i64, sz = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_size_t
        lib.vif_nccl_unique_id.argtypes = [P]
        lib.vif_workspace_bytes.argtypes = [ctypes.POINTER(_Dims), ctypes.POINTER(sz)]
        lib.vif_partition.argtypes = [ctypes.POINTER(_Dims), ctypes.POINTER(i64), ctypes.POINTER(i64)]
        lib.vif_create.argtypes = [ctypes.POINTER(P), ctypes.POINTER(_Dims), P, sz, P, P, P, P, P, P]
        lib.vif_set_data.argtypes = [P, P, P, P, P, i32]
        lib.vif_factor.argtypes = [P, ctypes.POINTER(_Theta), P, P]
        lib.vif_nll.argtypes = [P, ctypes.POINTER(_Terms)]
        lib.vif_copy_U.argtypes = [P, P]
        lib.vif_launch_count.argtypes = [P, ctypes.POINTER(i64)]
        lib.vif_gram.argtypes = [P, i64, i64, i32, P, i64, i32, P]
        lib.vif_last_error.argtypes = [P]
        lib.vif_last_error.restype = ctypes.c_char_p
        lib.vif_profile.argtypes = [P, i32]
        lib.vif_stage_times.argtypes = [P, P, ctypes.POINTER(i64)]
        lib.vif_stage_name.argtypes = [i32]
        lib.vif_stage_name.restype = ctypes.c_char_p
        lib.vif_destroy.argtypes = [P]
        lib.vif_destroy.restype = None
        lib.vif_grad_workspace_bytes.argtypes = [ctypes.POINTER(_Dims), ctypes.POINTER(sz)]
        lib.vif_grad.argtypes = [P, ctypes.POINTER(_Theta), P, sz, P, ctypes.POINTER(_Terms)]
        lib.vif_predict_workspace_bytes.argtypes = [ctypes.POINTER(_Dims), i64, ctypes.POINTER(sz)]
        lib.vif_predict.argtypes = [P, ctypes.POINTER(_Theta), i64, P, P, P, sz, P, P, P, P]
        lib.vif_neighbors.argtypes = [P, ctypes.POINTER(_Theta), i32, P]
        lib.vif_stage_data.argtypes = [P, P, P, P, P]
        lib.vif_owned_rows.argtypes = [P, ctypes.POINTER(i64), ctypes.POINTER(i64), ctypes.POINTER(i32),
                                       ctypes.POINTER(i64)]
        lib.vif_la_workspace_bytes.argtypes = [ctypes.POINTER(_Dims), i32, i32, ctypes.POINTER(sz)]
        lib.vif_la_prepare.argtypes = [P, ctypes.POINTER(_Theta), i32, i32, P, sz]
        lib.vif_la_apply.argtypes = [P, P, i32, i32, P, P, P]
        lib.vif_la_nll.argtypes = [P, P, P, ctypes.POINTER(_LaOpts), P, P, P, ctypes.POINTER(_LaTerms)]
        for f in ("vif_nccl_unique_id", "vif_workspace_bytes", "vif_partition", "vif_create", "vif_set_data",
                  "vif_factor", "vif_nll", "vif_copy_U", "vif_launch_count", "vif_profile", "vif_stage_times",
                  "vif_gram", "vif_grad_workspace_bytes", "vif_grad", "vif_predict_workspace_bytes", "vif_predict",
                  "vif_neighbors", "vif_stage_data", "vif_owned_rows", "vif_la_workspace_bytes", "vif_la_prepare", "vif_la_apply",
                  "vif_la_nll"):
            getattr(lib, f).restype = ctypes.c_int
        _lib = lib
    return _lib


EXPORTED = ("vif_nccl_unique_id", "vif_workspace_bytes", "vif_partition", "vif_create", "vif_set_data",
            "vif_factor", "vif_nll", "vif_copy_U", "vif_launch_count", "vif_profile", "vif_stage_times",
            "vif_stage_name", "vif_last_error", "vif_destroy", "vif_grad_workspace_bytes", "vif_grad",
            "vif_predict_workspace_bytes", "vif_predict", "vif_neighbors", "vif_stage_data",
            "vif_la_workspace_bytes", "vif_la_prepare", "vif_la_apply", "vif_la_nll", "vif_owned_rows", "vif_gram")
LA_OPS = {"sigma": 0, "A": 1, "binv": 2, "btinv": 3, "fitc_solve": 4, "sigma_inv": 5, "A1": 6}
NUM_STAGES = 8


def _check(st: int, handle=None, bad_row: int = -1):
    if st != 0:
        msg = load_library().vif_last_error(handle).decode(errors="replace")
        raise VifError(st, msg, bad_row)


def _dims(n, d, m, mv, rank=0, world=1) -> _Dims:
    return _Dims(int(n), int(d), int(m), int(mv), int(rank), int(world))


def vif_workspace_bytes(n: int, d: int, m: int, mv: int, rank: int = 0, world: int = 1) -> int:
    out = ctypes.c_size_t(0)
    _check(load_library().vif_workspace_bytes(ctypes.byref(_dims(n, d, m, mv, rank, world)), ctypes.byref(out)))
    return int(out.value)


def vif_partition(n: int, d: int, m: int, mv: int, rank: int = 0, world: int = 1):
    """(rounds, chunk) of the chunk-cyclic row partition (host only)."""
    r, c = ctypes.c_int64(0), ctypes.c_int64(0)
    _check(load_library().vif_partition(ctypes.byref(_dims(n, d, m, mv, rank, world)), ctypes.byref(r),
                                        ctypes.byref(c)))
    return int(r.value), int(c.value)


def owned_rows(n: int, rank: int, world: int, rounds: int, chunk: int) -> np.ndarray:
    """Global rows of `rank` under the chunk-cyclic partition described by vif_partition."""
    parts = []
    for r in range(rounds):
        s = (r * world + rank) * chunk
        e = min(s + chunk, n)
        if s < e:
            parts.append(np.arange(s, e))
    return np.concatenate(parts) if parts else np.zeros(0, dtype=np.int64)


def vif_nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(load_library().vif_nccl_unique_id(buf))
    return buf.raw


def _ptr(t: Optional[torch.Tensor]):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else None


def _as_input(a, dtype, device) -> Optional[torch.Tensor]:
    """Device tensors pass through; pinned host tensors pass through (the library copies them);
    numpy arrays are moved to the device first (plumbing only)."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        a = torch.from_numpy(np.ascontiguousarray(a)).to(device)
    if a.dtype != dtype:
        raise TypeError(f"expected {dtype}, got {a.dtype}")
    if not a.is_contiguous():
        a = a.contiguous()
    if not a.is_cuda and not a.is_pinned():
        a = a.to(device)
    return a


@dataclass
class Theta:
    """theta: family, sigma_1^2, ARD length-scales, nugget sigma^2, jitter eps (reading c3)."""
    family: Union[str, int]
    sigma2: float
    lengthscale: Sequence[float]
    nugget: float
    jitter: float

    def to_c(self):
        ls = np.ascontiguousarray(np.asarray(self.lengthscale, dtype=np.float64))
        fam = FAMILIES[self.family] if isinstance(self.family, str) else int(self.family)
        th = _Theta(fam, len(ls), float(self.sigma2), ls.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                    float(self.nugget), float(self.jitter))
        return th, ls


@dataclass
class Terms:
    nll: float
    logdet_D: float
    logdet_M: float
    quad: float
    bad_row: int


def vif_create(n, d, m, mv, workspace: torch.Tensor, X=None, Z=None, nbr=None, y=None, *, rank=0, world=1,
               nccl_id: Optional[bytes] = None, stream: Optional[torch.cuda.Stream] = None) -> ctypes.c_void_p:
    lib = load_library()
    h = ctypes.c_void_p()
    s = (stream or torch.cuda.current_stream(workspace.device)).cuda_stream
    idbuf = ctypes.create_string_buffer(nccl_id, 128) if nccl_id is not None else None
    st = lib.vif_create(ctypes.byref(h), ctypes.byref(_dims(n, d, m, mv, rank, world)),
                        ctypes.c_void_p(workspace.data_ptr()), workspace.numel(), _ptr(X), _ptr(Z), _ptr(nbr),
                        _ptr(y), idbuf, ctypes.c_void_p(s))
    _check(st, None)
    return h


def vif_set_data(h, X=None, Z=None, nbr=None, y=None, validate: bool = False):
    _check(load_library().vif_set_data(h, _ptr(X), _ptr(Z), _ptr(nbr), _ptr(y), int(validate)), h)


def vif_stage_data(h, X, Z, nbr, y):
    """Stage the next evaluation's inputs into the second slot (copies overlap the current evaluation)."""
    _check(load_library().vif_stage_data(h, _ptr(X), _ptr(Z), _ptr(nbr), _ptr(y)), h)


def vif_factor(h, theta: Theta, B_out: Optional[torch.Tensor] = None, D_out: Optional[torch.Tensor] = None):
    th, keep = theta.to_c()
    _check(load_library().vif_factor(h, ctypes.byref(th), _ptr(B_out), _ptr(D_out)), h)


def vif_nll(h) -> Terms:
    t = _Terms()
    st = load_library().vif_nll(h, ctypes.byref(t))
    _check(st, h, t.bad_row)
    return Terms(t.nll, t.logdet_D, t.logdet_M, t.quad, t.bad_row)


def vif_grad_workspace_bytes(n: int, d: int, m: int, mv: int, rank: int = 0, world: int = 1) -> int:
    b = ctypes.c_size_t(0)
    _check(load_library().vif_grad_workspace_bytes(ctypes.byref(_dims(n, d, m, mv, rank, world)), ctypes.byref(b)))
    return int(b.value)


def vif_grad(h, theta: Theta, grad_workspace: torch.Tensor):
    """(Terms, dNLL/dtheta) for theta = (sigma_1^2, lambda_1..lambda_d, sigma^2)."""
    th, keep = theta.to_c()
    g = np.zeros(len(keep) + 2)
    t = _Terms()
    st = load_library().vif_grad(h, ctypes.byref(th), ctypes.c_void_p(grad_workspace.data_ptr()),
                                 grad_workspace.numel(), g.ctypes.data_as(ctypes.c_void_p), ctypes.byref(t))
    _check(st, h, t.bad_row)
    return Terms(t.nll, t.logdet_D, t.logdet_M, t.quad, t.bad_row), g


def vif_predict_workspace_bytes(n: int, d: int, m: int, mv: int, npred: int, rank: int = 0, world: int = 1) -> int:
    b = ctypes.c_size_t(0)
    _check(load_library().vif_predict_workspace_bytes(ctypes.byref(_dims(n, d, m, mv, rank, world)), int(npred),
                                                      ctypes.byref(b)))
    return int(b.value)


def vif_predict(h, theta: Theta, Xp: torch.Tensor, nbrp: Optional[torch.Tensor], workspace: torch.Tensor,
                mu: torch.Tensor, var: Optional[torch.Tensor] = None, Dp: Optional[torch.Tensor] = None,
                Bp: Optional[torch.Tensor] = None):
    """Predictive means / variances (Prop. 1; App. C.1) into mu, var (device, np);
    optional D_p and B_p = -A_p."""
    th, keep = theta.to_c()
    st = load_library().vif_predict(h, ctypes.byref(th), int(Xp.shape[0]), _ptr(Xp), _ptr(nbrp),
                                    ctypes.c_void_p(workspace.data_ptr()), workspace.numel(), _ptr(mu), _ptr(var),
                                    _ptr(Dp), _ptr(Bp))
    _check(st, h)


def vif_neighbors(h, theta: Theta, mv: int, out: torch.Tensor):
    """Correlation-distance neighbour sets into out (device, n x mv int32)."""
    th, keep = theta.to_c()
    _check(load_library().vif_neighbors(h, ctypes.byref(th), int(mv), _ptr(out)), h)


@dataclass
class LaOpts:
    """Options of the VIF-Laplace path (readings l3, l4 of DESIGN.md section 13)."""
    max_newton: int = 50
    newton_tol: float = 1e-10
    max_cg: int = 1000
    cg_tol: float = 1e-10
    nprobe: int = 0
    slq_tol: float = 1e-10


@dataclass
class LaTerms:
    nll: float
    neg_loglik: float
    quad: float
    logdet: float
    logdet_W: float
    logdet_P: float
    newton_iters: int
    cg_iters: int
    slq_iters_max: int
    slq_iters_mean: float


def vif_la_workspace_bytes(n, d, m, mv, nprobe, max_cg, rank=0, world=1) -> int:
    b = ctypes.c_size_t(0)
    _check(load_library().vif_la_workspace_bytes(ctypes.byref(_dims(n, d, m, mv, rank, world)), int(nprobe),
                                                 int(max_cg), ctypes.byref(b)))
    return b.value


def vif_la_prepare(h, theta: Theta, nprobe: int, max_cg: int, ws: torch.Tensor):
    th, keep = theta.to_c()
    _check(load_library().vif_la_prepare(h, ctypes.byref(th), int(nprobe), int(max_cg), _ptr(ws), ws.numel()), h)


def vif_la_apply(h, ws: torch.Tensor, op: str, v: torch.Tensor, out: torch.Tensor, winv=None):
    ncol = 1 if v.dim() == 1 else v.shape[1]
    _check(load_library().vif_la_apply(h, _ptr(ws), LA_OPS[op], ncol, _ptr(v), _ptr(winv), _ptr(out)), h)


def vif_la_nll(h, ws: torch.Tensor, y: torch.Tensor, opts: LaOpts, eps1=None, eps2=None, b_mode=None) -> LaTerms:
    o = _LaOpts(opts.max_newton, opts.newton_tol, opts.max_cg, opts.cg_tol, opts.nprobe, opts.slq_tol)
    t = _LaTerms()
    _check(load_library().vif_la_nll(h, _ptr(ws), _ptr(y), ctypes.byref(o), _ptr(eps1), _ptr(eps2), _ptr(b_mode),
                                     ctypes.byref(t)), h)
    return LaTerms(t.nll, t.neg_loglik, t.quad, t.logdet, t.logdet_W, t.logdet_P, t.newton_iters, t.cg_iters,
                   t.slq_iters_max, t.slq_iters_mean)


def vif_owned_rows(h):
    """(first_chunk, chunk, stride, nchunks) of the handle's chunk-cyclic row map."""
    f, c, st, nc = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int32(), ctypes.c_int64()
    _check(load_library().vif_owned_rows(h, ctypes.byref(f), ctypes.byref(c), ctypes.byref(st), ctypes.byref(nc)), h)
    return f.value, c.value, st.value, nc.value


def vif_copy_U(h, out: torch.Tensor):
    _check(load_library().vif_copy_U(h, _ptr(out)), h)


GRAM_ENGINES = {"int8": 0, "fp64": 1}


def vif_gram(W: torch.Tensor, engine: str = "int8", stream: Optional[torch.cuda.Stream] = None) -> torch.Tensor:
    """G = W^T W (lower triangle written; the rest mirrored here) for a CUDA float64 matrix W (nrows x ncols,
    row stride even).  engine: "int8" (tcgen05 integer slices) or "fp64" (DMMA).  Stream-ordered on `stream`
    (default: the current stream)."""
    if not (isinstance(W, torch.Tensor) and W.is_cuda and W.dtype == torch.float64 and W.dim() == 2):
        raise TypeError("W must be a 2-D CUDA float64 tensor")
    if W.stride(1) != 1:
        W = W.contiguous()
    if W.stride(0) % 2:
        W = torch.nn.functional.pad(W, (0, 1))[:, :W.shape[1]]
    n, c = W.shape
    G = torch.zeros((c, c), dtype=torch.float64, device=W.device)
    s = (stream or torch.cuda.current_stream(W.device)).cuda_stream
    _check(load_library().vif_gram(_ptr(W), W.stride(0), n, c, _ptr(G), c, GRAM_ENGINES[engine], s))
    return torch.tril(G) + torch.tril(G, -1).T


def vif_launch_count(h) -> int:
    c = ctypes.c_int64(0)
    _check(load_library().vif_launch_count(h, ctypes.byref(c)), h)
    return int(c.value)


def vif_profile(h, enable: bool = True):
    _check(load_library().vif_profile(h, int(enable)), h)


def vif_stage_times(h):
    """(list of cumulative ms per stage, evaluations accumulated)"""
    arr = (ctypes.c_double * NUM_STAGES)()
    ev = ctypes.c_int64(0)
    _check(load_library().vif_stage_times(h, arr, ctypes.byref(ev)), h)
    return list(arr), int(ev.value)


def vif_stage_name(i: int) -> str:
    return load_library().vif_stage_name(int(i)).decode()


def vif_last_error(h=None) -> str:
    return load_library().vif_last_error(h).decode(errors="replace")


def vif_destroy(h):
    load_library().vif_destroy(h)


class VifModel:
    """One handle + its torch-owned workspace on `device`."""

    def __init__(self, X, Z, nbr, y, *, rank: int = 0, world: int = 1, nccl_id: Optional[bytes] = None,
                 device: Union[str, torch.device] = "cuda", stream: Optional[torch.cuda.Stream] = None):
        if not torch.cuda.is_available():
            raise RuntimeError("VifModel needs a CUDA device (no CPU fallback by design)")
        self.device = torch.device(device)
        X = _as_input(X, torch.float64, self.device)
        Z = _as_input(Z, torch.float64, self.device)
        nbr = _as_input(nbr, torch.int32, self.device)
        y = _as_input(y, torch.float64, self.device)
        self.n, self.d = X.shape
        self.m = Z.shape[0]
        self.mv = nbr.shape[1]
        self.rank, self.world = rank, world
        nbytes = vif_workspace_bytes(self.n, self.d, self.m, self.mv, rank, world)
        self.workspace = torch.empty(nbytes, dtype=torch.uint8, device=self.device)
        self.stream = stream
        self.handle = vif_create(self.n, self.d, self.m, self.mv, self.workspace,
                                 X, Z if self.m > 0 else None, nbr if self.mv > 0 else None, y,
                                 rank=rank, world=world, nccl_id=nccl_id, stream=stream)
        self.rounds, self.chunk = vif_partition(self.n, self.d, self.m, self.mv, rank, world)

    def _inputs(self, X, Z, nbr, y):
        """Marshal new inputs like the constructor does (dtype, contiguity, device or pinned host) and check
        their sizes against the handle's dims; a mismatch raises instead of reading a wrong byte count."""
        X = _as_input(X, torch.float64, self.device)
        Z = _as_input(Z, torch.float64, self.device) if self.m > 0 else None
        nbr = _as_input(nbr, torch.int32, self.device) if self.mv > 0 else None
        y = _as_input(y, torch.float64, self.device)
        for name, t, want in (("X", X, self.n * self.d), ("Z", Z, self.m * self.d), ("nbr", nbr, self.n * self.mv),
                              ("y", y, self.n)):
            if t is not None and t.numel() != want:
                raise ValueError(f"{name} has {t.numel()} elements, the handle needs {want}")
        return X, Z, nbr, y

    def set_data(self, X=None, Z=None, nbr=None, y=None, validate=False):
        X, Z, nbr, y = self._inputs(X, Z, nbr, y)
        vif_set_data(self.handle, X, Z, nbr, y, validate)
        self._staged = (X, Z, nbr, y)  # the copies are asynchronous on the library's stream

    def stage_data(self, X, Z, nbr, y):
        """Inputs of the next evaluation (pinned host or device tensors), copied while this one runs."""
        X, Z, nbr, y = self._inputs(X, Z, nbr, y)
        vif_stage_data(self.handle, X, Z, nbr, y)
        # keep the sources alive until the copy stream has read them (the next staging call at the
        # earliest waits for the slot's previous evaluation, which waited for these copies)
        self._staged_prev, self._staged = getattr(self, "_staged", None), (X, Z, nbr, y)

    def factor(self, theta: Theta, B_out=None, D_out=None):
        vif_factor(self.handle, theta, B_out, D_out)

    def nll(self) -> Terms:
        return vif_nll(self.handle)

    def evaluate(self, theta: Theta, B_out=None, D_out=None) -> Terms:
        self.factor(theta, B_out, D_out)
        return self.nll()

    def grad(self, theta: Theta):
        """NLL terms and dNLL/dtheta, theta = (sigma_1^2, lambda_1..lambda_d, sigma^2); the second
        workspace is allocated on first use and kept."""
        if getattr(self, "grad_workspace", None) is None:
            nbytes = vif_grad_workspace_bytes(self.n, self.d, self.m, self.mv, self.rank, self.world)
            self.grad_workspace = torch.empty(nbytes, dtype=torch.uint8, device=self.device)
        return vif_grad(self.handle, theta, self.grad_workspace)

    def predict(self, theta: Theta, Xp, nbrp, want_var: bool = False, want_D: bool = False, want_B: bool = False):
        """Predictive means at Xp (np x d) with training-neighbour sets nbrp (np x m_v); returns mu (and
        the predictive variances, D_p, B_p = -A_p when asked) as device tensors."""
        Xp = _as_input(Xp, torch.float64, self.device)
        nbrp = _as_input(nbrp, torch.int32, self.device) if self.mv > 0 else None
        npred = Xp.shape[0]
        nbytes = vif_predict_workspace_bytes(self.n, self.d, self.m, self.mv, npred, self.rank, self.world)
        ws = getattr(self, "pred_workspace", None)
        if ws is None or ws.numel() < nbytes:
            ws = self.pred_workspace = torch.empty(nbytes, dtype=torch.uint8, device=self.device)
        mu = torch.empty(npred, dtype=torch.float64, device=self.device)
        var = torch.empty(npred, dtype=torch.float64, device=self.device) if want_var else None
        Dp = torch.empty(npred, dtype=torch.float64, device=self.device) if want_D else None
        Bp = torch.empty((npred, self.mv), dtype=torch.float64, device=self.device) if want_B else None
        vif_predict(self.handle, theta, Xp, nbrp, ws, mu, var, Dp, Bp)
        out = (mu,) + ((var,) if want_var else ()) + ((Dp,) if want_D else ()) + ((Bp,) if want_B else ())
        return out[0] if len(out) == 1 else out

    def neighbors(self, theta: Theta, mv: int) -> torch.Tensor:
        """N(i) under d_c at theta for the handle's X (Vecchia order): device n x mv int32, -1 padded."""
        out = torch.empty((self.n, mv), dtype=torch.int32, device=self.device)
        vif_neighbors(self.handle, theta, mv, out)
        return out

    # ---- VIF-Laplace (Bernoulli-logit latent GP)
    def la_prepare(self, theta: Theta, nprobe: int = 0, max_cg: int = 1000):
        """Latent factor at theta (nugget forced to 0) + transposed structure into the Laplace workspace."""
        nbytes = vif_la_workspace_bytes(self.n, self.d, self.m, self.mv, nprobe, max_cg, self.rank, self.world)
        ws = getattr(self, "la_workspace", None)
        if ws is None or ws.numel() < nbytes:
            ws = self.la_workspace = torch.empty(nbytes, dtype=torch.uint8, device=self.device)
        vif_la_prepare(self.handle, theta, nprobe, max_cg, ws)

    def la_apply(self, op: str, v, winv=None) -> torch.Tensor:
        """Sigma_dagger v ("sigma"), (W^{-1} + Sigma_dagger) v ("A"), B^{-1} v, B^{-T} v, P^{-1} v."""
        v = _as_input(v, torch.float64, self.device)
        winv = _as_input(winv, torch.float64, self.device)
        out = torch.empty_like(v)
        vif_la_apply(self.handle, self.la_workspace, op, v, out, winv)
        return out

    def la_nll(self, y, opts: LaOpts, eps1=None, eps2=None):
        """(LaTerms, mode b~ as a device tensor) for labels y in {0, 1}."""
        y = _as_input(y, torch.float64, self.device)
        eps1 = _as_input(eps1, torch.float64, self.device)
        eps2 = _as_input(eps2, torch.float64, self.device)
        b = torch.empty(self.n, dtype=torch.float64, device=self.device)
        t = vif_la_nll(self.handle, self.la_workspace, y, opts, eps1, eps2, b)
        return t, b

    def U(self) -> torch.Tensor:
        out = torch.empty((self.n, self.m), dtype=torch.float64, device=self.device)
        vif_copy_U(self.handle, out)
        return out

    def owned_rows(self, rank=None) -> np.ndarray:
        return owned_rows(self.n, self.rank if rank is None else rank, self.world, self.rounds, self.chunk)

    def profile(self, enable: bool = True):
        vif_profile(self.handle, enable)

    def stage_times(self):
        ms, ev = vif_stage_times(self.handle)
        return {vif_stage_name(i): v for i, v in enumerate(ms)}, ev

    def launch_count(self) -> int:
        return vif_launch_count(self.handle)

    def close(self):
        if getattr(self, "handle", None) is not None:
            vif_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
