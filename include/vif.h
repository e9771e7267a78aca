/*
 * vif.h -- C ABI of the B200-native VIF factor + Gaussian NLL library (libvif.so).
 *
 * Method: Vecchia-inducing-points full-scale (VIF) approximation, arXiv 2507.05064
 * ("P:NNN" = line of PAPER.md):
 *   whitened inducing features  U = (L_m^{-1} K(Z,X))^T, n x m        P:72-80  (reading c4)
 *   residual Vecchia factor     B (unit lower, B_{i,N(i)} = -A_i), D  P:85-97, Eq. D_A_Vecchia
 *   Woodbury / Sylvester NLL    M_w = I + U^T B^T D^{-1} B U
 *   NLL = n/2 log(2 pi) + 1/2 (sum_i log D_i + logdet M_w) + 1/2 (y^T B^T D^{-1} B y - v^T M_w^{-1} v)
 * The readings of the paper taken where it is silent (c1..c17) are listed in DESIGN.md.
 *
 * Conventions for every call:
 *   - all floating point is IEEE FP64, all matrices row-major, all indices 0-based;
 *   - "device" pointers are CUDA device (or managed) memory of the current device; pointers
 *     documented "device or host" may also be page-locked host memory (copied with
 *     cudaMemcpyAsync(cudaMemcpyDefault)); the library never frees memory it did not allocate;
 *   - the library performs NO cudaMalloc: the caller owns one workspace buffer of
 *     vif_workspace_bytes() bytes (a torch uint8 tensor in the Python binding) for the
 *     handle's lifetime;
 *   - all GPU work is enqueued on the caller's CUDA stream (plus, for world > 1, an internal
 *     communication stream joined by events); only vif_create, vif_set_data(validate=1) and
 *     vif_nll synchronise with the host;
 *   - every call returns a vif_status; nothing aborts or throws across the ABI; the last
 *     error text is available from vif_last_error().
 */
#ifndef VIF_H_
#define VIF_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define VIF_ABI_VERSION 1
#define VIF_MAX_D 16     /* input dimension limit */
#define VIF_MAX_MV 47    /* neighbour limit: conditioning sets of s = m_v + 1 <= 48 points */

typedef enum {
  VIF_OK = 0,
  VIF_ERR_INVALID_ARG = 1, /* bad dims/pointer/parameter, non-finite input, bad neighbour list */
  VIF_ERR_NOT_PD = 2,      /* Cholesky failure of K_m, of a residual block C_{N(i),N(i)}, of M */
  VIF_ERR_CUDA = 3,        /* a CUDA runtime error (text in vif_last_error) */
  VIF_ERR_NCCL = 4,        /* an NCCL error or NCCL unavailable for world > 1 */
  VIF_ERR_NO_MEMORY = 5,   /* workspace smaller than vif_workspace_bytes() */
  VIF_ERR_STATE = 6        /* call order violated (e.g. vif_nll before vif_factor) */
} vif_status;

/* Covariance families, reading c1: k(a,b) = sigma2 * f(r), r = ||(a - b) / lambda|| */
typedef enum {
  VIF_MATERN12 = 0, /* f = exp(-r)                                   nu = 1/2 */
  VIF_MATERN32 = 1, /* f = (1 + sqrt3 r) exp(-sqrt3 r)               nu = 3/2 */
  VIF_MATERN52 = 2, /* f = (1 + sqrt5 r + 5 r^2 / 3) exp(-sqrt5 r)   nu = 5/2 */
  VIF_GAUSSIAN = 3  /* f = exp(-r^2)                                 nu = inf  */
} vif_family;

/* Covariance parameters theta.  Passed by pointer to vif_factor; read before return. */
typedef struct {
  int32_t family;            /* vif_family */
  int32_t d;                 /* must equal vif_dims.d */
  double sigma2;             /* marginal variance sigma_1^2 > 0 */
  const double* lengthscale; /* HOST pointer, d entries > 0 (ARD; isotropic = all equal) */
  double nugget;             /* error variance sigma^2 >= 0, added by index identity (reading c2) */
  double jitter;             /* eps >= 0 added to diag K(Z,Z) only (reading c3) */
} vif_theta;

/* Problem dimensions and the caller's place in the data-parallel job. */
typedef struct {
  int64_t n;     /* number of points, >= 1 */
  int32_t d;     /* input dimension, 1..VIF_MAX_D */
  int32_t m;     /* inducing points, >= 0 (m = 0: classical Vecchia) */
  int32_t mv;    /* neighbours per point, 0..VIF_MAX_MV (m_v = 0: FITC) */
  int32_t rank;  /* this process's rank, 0 <= rank < world */
  int32_t world; /* number of GPUs the rows are sharded over (one process per GPU) */
} vif_dims;

/* Result of vif_nll: identical on every rank. */
typedef struct {
  double nll;      /* L_dagger(theta; y) */
  double logdet_D; /* sum_i log D_i */
  double logdet_M; /* log det M_w = log det M - log det Sigma_m  (reading c4) */
  double quad;     /* y^T Sigma_dagger^{-1} y */
  int64_t bad_row; /* on VIF_ERR_NOT_PD: first failing point index, -1 for K_m / M */
} vif_terms;

/* Fills out128 with a fresh ncclUniqueId (128 bytes).  Call on rank 0 only and broadcast the
 * bytes (torch.distributed) before vif_create on every rank.  Needs libnccl.so.2 at run time. */
int vif_nccl_unique_id(void* out128);

/* Bytes of device workspace a handle with these dims needs (computed on the host, no GPU). */
int vif_workspace_bytes(const vif_dims* dims, size_t* bytes);

/* Rows owned by `rank` under the chunk-cyclic partition (host only, no GPU): the union over
 * rounds r of [(r*world + rank)*chunk, (r*world + rank + 1)*chunk) intersected with [0, n).
 * Writes *rounds and *chunk; the caller derives the rows. */
int vif_partition(const vif_dims* dims, int64_t* rounds, int64_t* chunk);
/* The same map for a created handle (SURVEY 8(b) vif_owned_rows): this rank owns the row chunks
 * first_chunk, first_chunk + stride, ... (< nchunks), chunk c = rows [c*chunk, (c+1)*chunk) & [0, n).
 * An emulated multi-rank handle owns every chunk (first 0, stride 1).  Any output may be NULL. */
int vif_owned_rows(void* handle, int64_t* first_chunk, int64_t* chunk, int32_t* stride, int64_t* nchunks);

/* Create a handle.  `workspace` (device, >= vif_workspace_bytes) is owned by the caller and must
 * outlive the handle.  X (n x d, Vecchia order), Z (m x d), nbr (n x mv int32: nbr[i][k] < i, no
 * duplicates, -1 only as trailing padding; reading c5) and y (n) are device or host pointers,
 * copied into the workspace (the caller may free them afterwards); they may be NULL and supplied
 * later with vif_set_data.  `cuda_stream` is a cudaStream_t (NULL = legacy default stream).
 * `nccl_id` is the 128-byte id from vif_nccl_unique_id when world > 1; with world > 1 and
 * nccl_id == NULL the library EMULATES all `world` ranks inside this one process (the same
 * partition, per-rank ordering and rank-ordered reduction, with the all-gather replaced by the
 * shared buffer and the all-reduce by an in-order sum) -- used to test sharding on one GPU.
 * Errors: INVALID_ARG (dims), NO_MEMORY (workspace too small), NCCL, CUDA. */
int vif_create(void** handle, const vif_dims* dims, void* workspace, size_t ws_bytes, const double* X,
               const double* Z, const int32_t* nbr, const double* y, const void* nccl_id, void* cuda_stream);

/* (Re)load the inputs (same layout/pointer rules as vif_create; NULL leaves a part unchanged).
 * Enqueued on the handle's stream.  validate = 1 also checks finiteness and the neighbour-list
 * rules on the device and synchronises (INVALID_ARG with vif_last_error naming the row).
 * New inputs invalidate a prepared VIF-Laplace workspace (vif_la_* then return VIF_ERR_STATE). */
int vif_set_data(void* handle, const double* X, const double* Z, const int32_t* nbr, const double* y,
                 int32_t validate);

/* Double-buffered input staging for pipelined use: copy X, Z, nbr, y (all required; host pinned or
 * device) into the handle's second input slot on an internal copy stream and sort its processing
 * order there; the next vif_factor / vif_neighbors (and vif_grad / vif_predict through them) swaps the
 * slot in, after the copies.  Returns at once; the current slot is untouched, so a vif_nll of the
 * evaluation already enqueued stays valid, and the copies overlap its compute.  No validation.
 * Errors: INVALID_ARG (missing array), CUDA. */
int vif_stage_data(void* handle, const double* X, const double* Z, const int32_t* nbr, const double* y);

/* Compute the factor at theta: K_m, L_m, L_m^{-1}; U rows (this rank's chunks) and their
 * all-gather; per owned point the residual block, its Cholesky, A_i, D_i and the row
 * w_i = (u_i - sum_k A_ik u_{N(i)_k}) / sqrt(D_i) with r_i appended; the Gram
 * [W r]^T [W r] of the owned rows and its all-reduce.  Asynchronous on the stream.
 * B_out (device, n x mv; stores -A_i in N(i) order, 0 padding; reading c16) and D_out (device, n)
 * are optional caller-owned full-length buffers: each rank writes only its owned rows.
 * Errors: INVALID_ARG (theta), STATE (no data); NOT_PD is reported by vif_nll. */
int vif_factor(void* handle, const vif_theta* theta, double* B_out, double* D_out);

/* Finish the NLL (Cholesky of M_w, z = L_M^{-1} v, quad, log-dets),
 * synchronise the stream and return the terms (same value on every rank).  Multi-rank: the failing
 * row of a residual block is found on the rank that owns it; vif_factor's all-reduce also takes the
 * minimum failing row over the ranks, so every rank returns NOT_PD with the same bad_row.  With a
 * communicator the wait polls ncclCommGetAsyncError and gives up after VIF_NCCL_TIMEOUT_S seconds
 * (environment, default 600): the communicator is aborted and this and every later call on the
 * handle return VIF_ERR_NCCL (a dead or hung peer never blocks the caller forever).
 * Errors: STATE (no vif_factor since create), NOT_PD (terms->bad_row says where), CUDA, NCCL. */
int vif_nll(void* handle, vif_terms* out);

/* Gradient of the NLL (dB, dD of Appendix A) with respect to
 * theta = (sigma_1^2, lambda_1, ..., lambda_d, sigma^2): d + 2 partial derivatives; the jitter is
 * held fixed (an isotropic range rho has dNLL/drho = sum_j dNLL/dlambda_j).
 * vif_grad_workspace_bytes: size of the second, caller-owned device workspace the gradient needs
 * (Q (ld x ld), g rows and R (n x ld each), the per-point state, m x m scratch;
 * ld = roundup(roundup(m,8)+1, 8)).
 * vif_grad runs vif_factor + vif_nll at theta (the factor's rows also write the per-point state:
 * L, A_i, D_i), then the adjoint rows of every point, R = their scatter over the conditioning sets,
 * T = R L_m^{-1} and G2 = R^T U once, and per parameter Phi = L_m^{-1} dK_m L_m^{-T},
 * <T, dK(X,Z)> - <G2, Phi_low> and one pass over the points (dK_S, dA_i, dD_i in adjoint form;
 * DESIGN.md section 10), and synchronises.  grad: host, d + 2 doubles, identical on every rank.
 * terms (optional): as vif_nll.  Multi-rank: each rank sums its own points' terms and one all-reduce
 * of the d + 2 partial sums follows; an emulated handle sums its virtual ranks in order.
 * Every m_v <= VIF_MAX_MV (s > 32: a shared-memory Cholesky in the state pass).
 * Errors: INVALID_ARG (theta), NO_MEMORY
 * (grad workspace too small), NOT_PD (as vif_nll), CUDA. */
int vif_grad_workspace_bytes(const vif_dims* dims, size_t* bytes);
int vif_grad(void* handle, const vif_theta* theta, void* grad_workspace, size_t grad_ws_bytes, double* grad,
             vif_terms* terms);

/* Predictive distribution of the response at np prediction inputs (Proposition 1, and the
 * equivalent variance expression of Appendix C.1), reading p1: each prediction point
 * conditions on m_v training points (B_p = I, B_po = -A_p), so with the whitened row
 * e_p = u_p - A_p U_N(p) of the prediction point,
 *   mu_p  = u_p . z + A_p (y_N(p) - U_N(p) z),          z = M_w^{-1} G_Wr,
 *   var_p = D_p + e_p^T M_w^{-1} e_p,                    u_p = L_m^{-1} k(Z, x_p),
 *   A_p = C_{p,N} C_{N,N}^{-1},  D_p = C_pp - A_p C_{N,p}   (residual covariance C as in vif_factor,
 *   C_pp = sigma_1^2 + sigma^2 - |u_p|^2: the response; the latent b_p has var_p - sigma^2).
 * vif_predict validates the prediction inputs (finite Xp; nbrp rows of distinct indices in [0, n),
 * -1 only trailing: INVALID_ARG naming the row), runs vif_factor + vif_nll at theta, then the
 * prediction features (kx_eval + triangular
 * GEMM), the per-point Vecchia rows of the prediction points against the training rows (the factor's
 * kernel), e_p M_w^{-1} e_p by one triangular GEMM with L_M^{-1}, and mu / var; synchronises.
 * Xp: np x d (device or host), nbrp: np x m_v training indices in [0, n), -1 only as trailing pad
 * (host or device); workspace: caller-owned device buffer of vif_predict_workspace_bytes(dims, np).
 * mu (device, np, required); var, Dp (device, np, optional); Bp (device, np x m_v, optional: -A_p).
 * Multi-rank: every rank passes all np inputs and full-length outputs; rank g predicts the contiguous
 * slice [g ceil(np/G), (g+1) ceil(np/G)) and writes only that slice (as vif_factor's B_out / D_out).
 * Errors: INVALID_ARG (np < 1, NULL, invalid Xp / nbrp), NO_MEMORY (workspace), NOT_PD (training factor, or a
 * prediction block: the message names the prediction row), CUDA. */
int vif_predict_workspace_bytes(const vif_dims* dims, int64_t np, size_t* bytes);
int vif_predict(void* handle, const vif_theta* theta, int64_t np, const double* Xp, const int32_t* nbrp,
                void* workspace, size_t ws_bytes, double* mu, double* var, double* Dp, double* Bp);

/* Correlation-distance neighbour sets (the paper's cover tree, Alg. 3-4, returns the same
 * sets): for every point i of the handle's X (Vecchia order) the mv predecessors j < i with the
 * smallest d_c(i,j) = sqrt(1 - |rho_c(i,j)| / sqrt(rho_c(i,i) rho_c(j,j))), rho_c = k - u_i.u_j at theta
 * (no nugget), ranked by (d_c, index); i <= mv: all predecessors; readings c5-c7 (a point
 * whose residual variance is below 1e-7 sigma_1^2 scores d_c = 1 as a candidate and ranks its own
 * predecessors by length-scale-scaled Euclidean distance).  Exact brute force (n^2 m / 2 FMA): the Gram
 * blocks u_i.u_j as exact int8 digit-slice products on the integer tensor cores when m > 0 (DESIGN reading
 * c18; environment VIF_KNN_FP64=1 selects the FP64 DMMA kernel), scores and ranking in FP64.  nbr_out: device, n x mv int32, -1 padded; mv in [1, VIF_MAX_MV] (independent of
 * dims.mv).  Uses the handle's workspace (invalidates a previous vif_factor: call vif_factor again).
 * Multi-rank: every rank evaluates u_i of all n points; rank g searches the query blocks (128 points on
 * the integer engine, 64 on DMMA) kb = g, g + G, ... (counted from the last block) and writes only their rows of the full-length nbr_out;
 * an emulated handle writes all rows.  Errors: INVALID_ARG, NOT_PD (K(Z,Z) + jitter), CUDA. */
int vif_neighbors(void* handle, const vif_theta* theta, int32_t mv, int32_t* nbr_out);

/* ---- VIF-Laplace iterative path (Bernoulli likelihood, logit link; Sect. 2-3) ----
 * Latent b ~ N(0, Sigma_dagger), Sigma_dagger = B^{-1} D B^{-T} + U U^T with B, D the residual Vecchia
 * factor WITHOUT error variance (vif_factor at nugget 0) and U the whitened features;
 * y_i | b_i ~ Bernoulli(1 / (1 + exp(-b_i))).  L^VIFLA = -log p(y|b~) + b~^T Sigma_dagger^{-1} b~ / 2
 * + log det(Sigma_dagger W + I) / 2 at the mode b~, W = diag(pi (1 - pi)).
 *   mode: Newton with each step's solve in the form (pcls2),
 *         (W^{-1} + Sigma_dagger) x = Sigma_dagger (W b + y - pi), b <- W^{-1} x, by preconditioned CG
 *         with the FITC preconditioner P = D_V + U U^T, D_V = diag(sigma_1^2 - |u_i|^2) + W^{-1}
 *         (App. FITC; reading l2: k = m, the VIF's inducing points);
 *   quad: b~^T Sigma_dagger^{-1} b~ exactly through the factor's Woodbury form (reading l5);
 *   log det: SLQ (slq_v2): log det W + (n / ell) sum_i e1^T log(T_i) e1 + log det P, T_i the
 *         Lanczos matrices from the CG coefficients of the solves with z_i = D_V^{1/2} eps2_i + U eps1_i
 *         (readings l6, l7).
 * Vectors are row-major n x ncol by point index (the Vecchia order).  Single rank in this version. */
typedef struct {
  int32_t max_newton; /* Newton steps cap */
  double newton_tol;  /* stop when |psi_t - psi_{t-1}| <= tol |psi_{t-1}|, psi = log p(y|b) - b^T a / 2 */
  int32_t max_cg;     /* CG iterations cap per solve (<= the prepared max_cg) */
  double cg_tol;      /* Newton solves: stop at ||r|| <= cg_tol ||rhs|| */
  int32_t nprobe;     /* ell SLQ probe vectors (0: mode and quadratic term only) */
  double slq_tol;     /* probe solves: stop at ||r|| <= slq_tol ||z_i|| */
} vif_la_opts;

typedef struct {
  double nll;          /* L^VIFLA (NaN without probes) */
  double neg_loglik;   /* -log p(y | b~) */
  double quad;         /* b~^T Sigma_dagger^{-1} b~ */
  double logdet;       /* SLQ estimate of log det(Sigma_dagger W + I) (NaN without probes) */
  double logdet_W;     /* log det W at the mode */
  double logdet_P;     /* log det of the FITC preconditioner at the mode */
  int32_t newton_iters;
  int32_t cg_iters;    /* CG iterations summed over the Newton steps */
  int32_t slq_iters_max;
  double slq_iters_mean;
} vif_la_terms;

enum { VIF_LA_SIGMA = 0, VIF_LA_A = 1, VIF_LA_BINV = 2, VIF_LA_BTINV = 3, VIF_LA_FITC_SOLVE = 4,
       VIF_LA_SIGMA_INV = 5, VIF_LA_A1 = 6 };

/* Size of the caller-owned device workspace for up to nprobe (<= 64) probe columns and max_cg CG
 * iterations per solve (~ (8 nprobe + 12 + m_v) n doubles plus n x ld for the FITC rows). */
int vif_la_workspace_bytes(const vif_dims* dims, int32_t nprobe, int32_t max_cg, size_t* bytes);
/* vif_factor + vif_nll at theta with the nugget forced to 0, then B, D, |u_i|^2 and the transposed
 * neighbour structure (children lists for B^{-T}) into the workspace; synchronises.  Any later
 * vif_factor / vif_grad / vif_predict / vif_neighbors call on the handle invalidates it (VIF_ERR_STATE).
 * Errors: INVALID_ARG (world > 1, nprobe, max_cg), NO_MEMORY, NOT_PD, CUDA. */
int vif_la_prepare(void* handle, const vif_theta* theta, int32_t nprobe, int32_t max_cg, void* workspace,
                   size_t ws_bytes);
/* Operators of the path on ncol (<= max(1, nprobe)) device columns v (n x ncol) -> out:
 * VIF_LA_SIGMA Sigma_dagger v;  VIF_LA_A (W^{-1} + Sigma_dagger) v;  VIF_LA_BINV B^{-1} v;
 * VIF_LA_BTINV B^{-T} v;  VIF_LA_FITC_SOLVE P^{-1} v;  VIF_LA_SIGMA_INV Sigma_dagger^{-1} v and
 * VIF_LA_A1 (W + Sigma_dagger^{-1}) v, the operator of (pcls1), by Woodbury with the latent
 * factor: B^T D^{-1/2} [s - W_U M^{-1} W_U^T s], s = D^{-1/2} B v (sparse products, no solves).
 * winv (device, n): W^{-1}, required by A, A1 and FITC_SOLVE.  The triangular solves are
 * level-scheduled (dependency levels of B / B^T from vif_la_prepare, one grid barrier per level).
 * Synchronises.  Errors: INVALID_ARG, STATE, NOT_PD (M_V), CUDA. */
int vif_la_apply(void* handle, void* workspace, int32_t op, int32_t ncol, const double* v, const double* winv,
                 double* out);
/* Mode, quadratic term and (with opts.nprobe > 0) the SLQ log-determinant and L^VIFLA.  y: device, n
 * labels in {0, 1}; eps1 (device, m x nprobe) and eps2 (device, n x nprobe): standard normal draws of
 * the probe vectors (row-major); b_mode (optional, device or host, n).  Synchronises.
 * Errors: INVALID_ARG, STATE, NOT_PD (non-finite Newton iterate, M_V), CUDA. */
int vif_la_nll(void* handle, void* workspace, const double* y, const vif_la_opts* opts, const double* eps1,
               const double* eps2, double* b_mode, vif_la_terms* out);

/* Debug / parity: copy the whitened features U (n x m, row-major) to `out` (device or host). */
int vif_copy_U(void* handle, double* out);

/* The Gram matrix G = W^T W of a device matrix (A6 / K4, "M": the contraction the factor runs on its
 * rows [W r]), exposed on its own for tests and benchmarks.
 *   W: device, nrows x ncols row-major, leading dimension ldw doubles (even; W 16-byte aligned);
 *   G: device, ncols x ncols row-major, leading dimension ldg: the lower triangle (a >= b) is written (entries
 *      above the diagonal inside diagonal tiles may be written too, with their symmetric values);
 *   engine: 0 = integer tensor cores (int8 digit slices on tcgen05.mma.kind::i8, exact int32 level sums,
 *      k_ozaki.cu; ncols <= 4096), 1 = FP64 DMMA (k_syrk.cu);
 *   stream: cudaStream_t (NULL = legacy default stream); scratch is taken with cudaMallocAsync on it and
 *      released the same way (the device's default memory pool is set to keep freed memory).  Enqueued only: the caller synchronises.  A non-finite entry of W makes G NaN.
 * Errors: VIF_ERR_INVALID_ARG (NULL pointers, ncols < 1, nrows < 0, ldw < ncols or odd, ldg < ncols,
 * engine 0 with ncols > 4096), VIF_ERR_CUDA. */
int vif_gram(const double* W, int64_t ldw, int64_t nrows, int32_t ncols, double* G, int64_t ldg, int32_t engine,
             void* stream);

/* Number of GPU kernel launches the last vif_factor + vif_nll pair enqueued (for bench.py). */
int vif_launch_count(void* handle, int64_t* count);

/* Per-stage device timing (CUDA events recorded on the handle's stream around each stage; adds
 * no synchronisation).  Stages: see vif_stage_name(0 .. VIF_NUM_STAGES-1).  vif_profile(h, 1)
 * enables and zeroes the accumulators; every vif_nll then adds the elapsed milliseconds of each
 * stage of that evaluation; vif_stage_times copies the VIF_NUM_STAGES cumulative sums and the
 * number of evaluations accumulated. */
#define VIF_NUM_STAGES 8
int vif_profile(void* handle, int32_t enable);
int vif_stage_times(void* handle, double* ms_out, int64_t* evaluations);
const char* vif_stage_name(int32_t stage);

/* Text of the last error on this handle (or of the last failed vif_create when handle is NULL). */
const char* vif_last_error(void* handle);

/* Release the handle (and its NCCL communicator).  Never frees the workspace. */
void vif_destroy(void* handle);

#ifdef __cplusplus
}
#endif
#endif /* VIF_H_ */
