// kernels.h -- host-side launchers of the libvif kernels (internal to the library).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"

namespace vif {

struct VecchiaArgs {
  const double* U;
  int64_t ldu;
  int mk;
  int ld;
  const double* X;
  const int32_t* nbr;
  int mv;
  const int64_t* order;
  int64_t npts;
  CovParams p;
  double* W;
  int64_t ldw;
  double* Dpos;
  double* B_out;
  double* D_out;
  DevStatus* st;
  // the point's own row (index i = order[pos]) comes from Uself / Xself when set (prediction:
  // prediction points whose neighbours are training rows of U / X); NULL = U / X
  const double* Uself = nullptr;
  const double* Xself = nullptr;
  // gradient (vif_grad, one rank per process): the factor's rows also write the per-point state of the gradient's
  // first pass (vif_state_doubles layout, by position; the g_i dots are left to launch_grad_gam)
  double* state = nullptr;
  // K4 on the integer tensor cores: column maxima of |W| (bit patterns) accumulated by the W pass into 64
  // interleaved copies of ld entries (copy pos mod 64; zeroed by the caller), or nullptr
  unsigned long long* cmax = nullptr;
};

// per-point gradient state, by position: L (packed lower, SP = 8 RB rows incl. the identity padding),
// A_i, 1/L_jj, g_i . U_aug[S_k], D_i, ok
template <int RB>
__host__ __device__ constexpr int vif_state_doubles() {
  return (RB * 8) * (RB * 8 + 1) / 2 + 3 * (RB * 8) + 2;
}

// K0 / K5
cudaError_t launch_build_km(const double* Z, int m, const CovParams& p, double* Km, cudaStream_t s);
cudaError_t launch_chol_inv(double* A, int m, int lda, double diag_add, double* Linv, int ldi, int lim_inv,
                            int full_inverse, double* Tscr, int* fail, int num_sms, cudaStream_t s);
cudaError_t launch_logd_sum(const double* Dpos, int64_t npts, double* partials, int np, double* out,
                            cudaStream_t s);
cudaError_t launch_finish(const double* G, int ld, int m, int ycol, const double* Dinv, int ldi,
                          const double* logdetD_dev, int64_t n, double* terms, cudaStream_t s);
// K1
cudaError_t launch_u_features(const double* X, const double* Z, const double* y, int64_t n, int64_t pos0,
                              int64_t npos, int64_t chunk, int world, int rank, int m, int mk, const CovParams& p,
                              const double* Linv, double* S, double* Uaug, int ld, cudaStream_t s, int lds = 0);
// K1 on the integer tensor cores (k_ozaki.cu): S = K(X,Z) evaluated straight into int8 digit slices with a
// per-row scale, Linv rows sliced per output column, tcgen05.mma.kind::i8 triangular GEMM; d in {2,3,5,10}
bool ufeat_i8_supported(int d, int mk);
size_t ufeat_i8_ws_bytes(int mk, int64_t cap_rows);
size_t ufeat_i8_aux_bytes(int mk, int64_t cap_rows);
cudaError_t launch_u_features_i8(const double* X, const double* Z, const double* y, int64_t n, int64_t pos0,
                                 int64_t npos, int64_t chunk, int world, int rank, int m, int mk, const CovParams& p,
                                 const double* Linv, double* Uaug, int ld, int8_t* ws, int64_t cap_rows, void* aux,
                                 int sms, cudaStream_t s);
// C (M x N, ldc) = A B^T, A: M x K (lda), B: N x K (ldb; lower triangular when tri: B[j][k] = 0 for k > j),
// on the integer tensor cores (int8 digit slices, per-row scales); rows in chunks of <= cap_rows
size_t gemm_i8_ws_bytes(int K, int64_t cap_rows);
size_t gemm_i8_aux_bytes(int N, int K, int64_t cap_rows);
cudaError_t launch_gemm_tn_i8(const double* A, int64_t lda, int64_t M, const double* B, int64_t ldb, int N, int K,
                              int tri, double* C, int64_t ldc, int8_t* ws, int64_t cap_rows, void* aux, int sms,
                              cudaStream_t s);
// C (M x N, ldc) = A^T B over nrows rows (A: lda, B: ldb) on the integer tensor cores; rows in chunks whose
// slices of A and B fit ws_bytes; Gpart: gemm_tt_i8_part_doubles(M, N, gemm_tt_i8_chunk(M, N, ws_bytes))
size_t gemm_tt_i8_aux_bytes(int M, int N);
size_t gemm_tt_i8_part_doubles(int M, int N, int64_t chunk_rows);
int64_t gemm_tt_i8_chunk(int M, int N, size_t ws_bytes);
cudaError_t launch_gemm_tt_i8(const double* A, int64_t lda, int M, const double* B, int64_t ldb, int N, int64_t nrows,
                              double* C, int64_t ldc, int8_t* ws, size_t ws_bytes, double* Gpart, void* aux, int sms,
                              cudaStream_t s);
// K2 + K3
cudaError_t launch_vecchia(const VecchiaArgs& a, cudaStream_t s);
// K4
int syrk_ntiles(int ncols);
int syrk_nsplit(int ncols, int64_t nrows, int num_sms);
size_t syrk_part_doubles(int ncols, int nsplit);
cudaError_t launch_syrk(const double* W, int64_t ldw, int64_t nrows, int ncols, int nsplit, double* Gpart,
                        double* G, int ldg, cudaStream_t s);
cudaError_t launch_syrk_part(const double* W, int64_t ldw, int64_t nrows, int ncols, int nsplit, double* Gpart,
                             cudaStream_t s);
// C (M x N, ldc) = A^T B over nrows rows (A: lda, B: ldb) on the SYRK's TMA engine, all tiles, nsplit row splits
int gemm_tt_nsplit(int M, int N, int64_t nrows, int num_sms);
size_t gemm_tt_part_doubles(int M, int N, int nsplit);
cudaError_t launch_gemm_tt(const double* A, int64_t lda, int M, const double* B, int64_t ldb, int N, int64_t nrows,
                           int nsplit, double* part, double* C, int64_t ldc, cudaStream_t s);
// K4 on the integer tensor cores (k_ozaki.cu): int8 digit slices of W, tcgen05.mma.kind::i8, exact int32
// level sums; rows processed in chunks of <= cap_rows (ws: syrk_i8_ws_bytes, Gpart: syrk_i8_part_doubles,
// aux: syrk_i8_aux_bytes)
bool syrk_i8_supported(int ncols);
size_t syrk_i8_ws_bytes(int ncols, int64_t cap_rows);
size_t syrk_i8_part_doubles(int ncols, int64_t cap_rows);
size_t syrk_i8_aux_bytes(int ncols);
cudaError_t launch_syrk_i8(const double* W, int64_t ldw, int64_t nrows, int ncols, int8_t* ws, int64_t cap_rows,
                           double* Gpart, void* aux, double* G, int ldg, int sms, cudaStream_t s,
                           const unsigned long long* cmax64 = nullptr);
// sums the partials of nlaunch consecutive launch_syrk_part calls (same ncols, nsplit) into G
cudaError_t launch_syrk_reduce(const double* Gpart, int ncols, int nsplit, int nlaunch, double* G, int ldg,
                               cudaStream_t s);
// gradient (k_grad.cu)
struct GradPointArgs {
  const double* U;
  const double* dU;   // NULL for the nugget (dU = 0)
  const double* Gam;  // g_i rows by processing position (npts x ld)
  int64_t ldu;
  int mk;
  int ld;
  const double* X;
  const int32_t* nbr;
  int mv;
  const int64_t* order;
  int64_t npts;
  CovParams p;
  double* part;  // (d + 2) x grad_point_nparts(npts) block partials
  double* state; // npts x grad_state_doubles(mv): per-point state of the first pass
  // adjoint form (k_grad.cu): rho, sig (npts x mk) and mu, Dm, beta~ (npts x grad_adj_doubles())
  double* rho = nullptr;
  double* sig = nullptr;
  double* adj = nullptr;
};
int64_t grad_point_nparts(int64_t npts);
// all d + 2 parameters' point terms in one pass (no dU); a.part: (d + 2) x grad_point_nparts(npts) doubles
cudaError_t launch_grad_points_adj_all(const GradPointArgs& a, double* out, cudaStream_t s);
size_t grad_state_doubles(int mv);
// the g_i . U_aug[S_k] slots of a state written by the factor (VecchiaArgs::state)
cudaError_t launch_grad_gam(const GradPointArgs& a, cudaStream_t s);
cudaError_t launch_grad_state(const GradPointArgs& a, cudaStream_t s);
size_t grad_adj_doubles();
cudaError_t launch_grad_adjoint(const GradPointArgs& a, cudaStream_t s);
cudaError_t launch_gchild(const int32_t* nbr, int mv, const int64_t* order, int64_t npts, int64_t n, int* cnt,
                          int* cursor, int* ptr, int* ent, cudaStream_t s);
cudaError_t launch_gR(const int* ptr, const int* ent, const int64_t* order, const int64_t* jorder, int64_t n, int mk,
                      int mv,
                      const double* state, const double* adj, const double* rho, const double* sig, double* R,
                      unsigned long long* next, cudaStream_t s);
int gTdK_blocks();
cudaError_t launch_gTdK(const double* X, const double* Z, int64_t n, int m, int mk, const CovParams& p,
                        const double* T, double* part, double* out, cudaStream_t s);
cudaError_t launch_grev_linv(const double* Linv, int mk, double* Bp, cudaStream_t s);
cudaError_t launch_gfinal(double* out, const double* tdk, int q, const double* G2, const double* Phil, int mk,
                          cudaStream_t s);
cudaError_t launch_dkm(const double* Z, int m, int mk, int pidx, const CovParams& p, double* out, cudaStream_t s);
cudaError_t launch_phi_low(const double* Phi, int mk, double* out, cudaStream_t s);
cudaError_t launch_grad_q(const double* LinvM, int ldi, const double* G, int ldg, int ycol, int m, int ld,
                          double* zh, double* z, double* Q2, cudaStream_t s);
cudaError_t launch_gemm_tn(const double* A, int64_t lda, int64_t nrows, const double* B, int64_t ldb, int N, int K,
                           int tri, double* C, int64_t ldc, double alpha, int accum, cudaStream_t s);
cudaError_t launch_zvec(const double* LinvM, int ldi, const double* G, int ldg, int ycol, int m, double* zh,
                        double* z, cudaStream_t s);
cudaError_t launch_pred_mean(const double* Wp, int ld, int m, int ycol, const double* z, const double* Dpos,
                             const int64_t* order, int64_t np, double* mu, const double* T, int ldt, double* var,
                             cudaStream_t s);
// correlation-distance neighbours (k_knn.cu)
size_t knn_smem_bytes(int mv);
// the same search with the Gram blocks on the integer tensor cores (k_ozaki.cu, reading c18): U rows sliced into
// ws (knn_i8_ws_bytes) with their exponents in erow (n ints); isd / deg from launch_knn_resvar
bool knn_i8_supported(int mv, int64_t n);
size_t knn_i8_ws_bytes(int mk, int64_t n);
cudaError_t launch_knn_i8(const double* U, int64_t ldu, int mk, const double* X, int64_t n, const CovParams& p,
                          const double* isd, const int* deg, int mv, int32_t* out, int8_t* ws, int* erow, int sms,
                          cudaStream_t s, int qoff, int qstride);
cudaError_t launch_knn_resvar(const double* U, int64_t ldu, int m, int64_t n, const CovParams& p, double* isd,
                              int* deg, cudaStream_t s);
cudaError_t launch_knn(const double* U, int64_t ldu, int m, int mk, const double* X, int64_t n, const CovParams& p,
                       double* isd, int* deg, int mv, int32_t* out, cudaStream_t s, int qoff = 0, int qstride = 1);
// VIF-Laplace iterative path (k_laplace.cu)
cudaError_t launch_la_transpose_struct(const int32_t* nbr, int64_t n, int mv, int* cnt, int* cursor, int* tptr,
                                       int* tpos, cudaStream_t s);
cudaError_t launch_la_tvals(const int* tpos, int64_t nnz, int mv, const double* Bc, int* trow, double* tval,
                            cudaStream_t s);
cudaError_t launch_la_levels(const int32_t* nbr, int mv, int64_t n, const int* tptr, const int* trow, int* lev_f,
                             int* lev_b, int* flags, int epoch_f, int epoch_b, int* nlev_dev, cudaStream_t s);
cudaError_t launch_la_reorder(const int* order_f, const int32_t* nbr, const double* Bc, int64_t n, int mv,
                              int32_t* ecol_f, double* eval_f, const int* order_b, const int* tptr, const int* trow,
                              const double* tval, int* cnt, int* eptr_b, int32_t* ecol_b, double* eval_b,
                              cudaStream_t s);
cudaError_t launch_la_bucket(const int* key, int64_t n, int nkeys, int* cnt, int* cursor, int* ptr, int* order,
                             cudaStream_t s);
cudaError_t launch_la_trsv_lvl(bool fwd, const int* order, const int* lptr, int nlev, const int32_t* ecol,
                               const double* eval, const int* eptr, int mv, int ncol, const double* v,
                               const double* scale, double* x, const double* v2, const double* w2, double* out2,
                               cudaStream_t s);
int la_ts_nsplit(int64_t n);
cudaError_t launch_la_tsgemm(const double* U, int64_t ldu, int mk, int64_t n, const double* V, int ncol,
                             const int64_t* vrow, const double* rs, double* part, double* Ct, double alpha,
                             cudaStream_t s);
int la_red_nsplit(int64_t n);
cudaError_t launch_la_reduce(int op, const double* a, const double* b, int64_t n, int ncol, double* part,
                             double* out, cudaStream_t s);
cudaError_t launch_la_newton_prep(const double* y, const double* b, int64_t n, double* W, double* winv, double* v,
                                  double* x0, cudaStream_t s);
cudaError_t launch_la_newton_update(const double* x, const double* v, const double* winv, int64_t n, double* b,
                                    double* a, cudaStream_t s);
cudaError_t launch_la_fitc_rows(const double* U, int64_t ldu, int mk, int ld, int64_t n, const double* unorm2,
                                double sigma2, const double* winv, double* DV, double* dvinv, double* S,
                                cudaStream_t s);
cudaError_t launch_la_rownorm2(const double* U, int64_t ldu, int mk, int64_t n, double* out, cudaStream_t s);
cudaError_t launch_la_rowscale(const double* in, const double* r, int use_sqrt, int64_t n, int ncol, double* out,
                               cudaStream_t s);
cudaError_t launch_la_sub_rowscale(const double* a, const double* b, const double* r, int64_t n, int ncol, double* out,
                                   cudaStream_t s);
cudaError_t launch_la_residual(const double* b, int64_t tot, double* r, cudaStream_t s);
cudaError_t launch_la_cg_alpha(const double* rz, const double* pq, const int* active, int ncol, double* alpha,
                               double* hist_a, cudaStream_t s);
cudaError_t launch_la_cg_xr(const double* alpha, const double* p, const double* q, int64_t n, int ncol, double* x,
                            double* r, cudaStream_t s);
cudaError_t launch_la_cg_beta(const double* rz_new, double* rz, const int* active, int ncol, double* beta,
                              double* hist_b, cudaStream_t s);
cudaError_t launch_la_cg_p(const double* beta, const int* active, const double* z, int64_t n, int ncol, double* p,
                           cudaStream_t s);
cudaError_t launch_la_transpose(const double* in, int rows, int cols, int ldin, double* out, int ldout, cudaStream_t s);
cudaError_t launch_la_logdiag(const double* A, int m, int lda, double* out, cudaStream_t s);
cudaError_t launch_la_slq(const double* hist_a, const double* hist_b, const int* iters, int ncol, int kmax,
                          double* scratch, double* out, cudaStream_t s);
cudaError_t launch_la_gemv(const double* U, int64_t ldu, int64_t n, int mk, const double* c, double alpha, int accum,
                           double* out, cudaStream_t s);
cudaError_t launch_la_bapply_cols(const int32_t* nbr, const double* Bc, int mv, int64_t n, int ncol, const double* D,
                                  const double* v, double* s, cudaStream_t st);
cudaError_t launch_la_woodbury_mid(const double* s, const double* Y, const int* ipos, const double* D, int64_t n,
                                   int ncol, double* z, cudaStream_t st);
cudaError_t launch_la_btapply_cols(const int* tptr, const int* trow, const double* tval, int64_t n, int ncol,
                                   const double* z, const double* winv, const double* v, double* out, cudaStream_t st);
cudaError_t launch_la_invorder(const int64_t* order, int64_t n, int* ipos, cudaStream_t st);
cudaError_t launch_la_bapply(const int32_t* nbr, const double* Bc, int mv, int64_t n, const double* D, const double* b,
                             double* s, cudaStream_t st);
cudaError_t launch_la_finish(const double* fin, const double* slq, int64_t n, int ell, double* out, cudaStream_t s);
// misc
cudaError_t launch_validate(const double* X, int64_t n, int d, const double* Z, int m, const double* y,
                            const int32_t* nbr, int mv, DevStatus* st, cudaStream_t s);
cudaError_t launch_validate_pred(const double* Xp, int64_t np, int d, const int32_t* nbrp, int mv, int64_t ntrain,
                                 DevStatus* st, cudaStream_t s);
size_t order_temp_bytes(int64_t npos);
cudaError_t launch_order(const double* X, int64_t n, int d, int64_t npos, int64_t chunk, int world, int rank,
                         double* bbox, uint64_t* keys, uint64_t* keys_alt, int64_t* vals, int64_t* vals_alt,
                         void* temp, size_t temp_bytes, int64_t** order_out, cudaStream_t s,
                         const int32_t* nbr = nullptr, int mv = 0);
cudaError_t launch_sum_buffers(const double* src, int64_t count, int nbuf, int64_t stride, double* dst,
                               cudaStream_t s);
cudaError_t launch_reset_status(DevStatus* st, cudaStream_t s);

}  // namespace vif
