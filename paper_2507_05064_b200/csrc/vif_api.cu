// vif_api.cu -- the C ABI of include/vif.h: handle, workspace layout, stream orchestration,
// chunk-cyclic row sharding and the two collectives (U all-gather, Gram all-reduce).
//
// One evaluation on rank g of G:
//   A0 K_m, L_m, L_m^{-1}                          launch_build_km + launch_chol_inv   (replicated)
//   A1 U rows of the rank's chunks                 launch_u_features (K1a + K1b)
//   A2 replicate U                                 ncclAllGather per round (in place)
//   A3-A5 per owned point: C_S, chol, A_i, D_i, w_i  launch_vecchia
//   A6 G = [W r]^T [W r] over owned rows, sum log D  launch_syrk + launch_logd_sum
//   A7 sum G and log D over ranks                  ncclAllReduce (one call, (ld^2 + 1) doubles)
//   A8 M_w chol, z, quad, NLL                       launch_chol_inv + launch_finish  (vif_nll)
// NCCL is loaded lazily with dlopen (only for world > 1), so a single-GPU process needs nothing
// beyond the CUDA driver.
#include <dlfcn.h>
#include <math.h>
#include <stdlib.h>
#include <nccl.h>
#include <stdio.h>
#include <string.h>

#include <chrono>
#include <string>
#include <thread>
#include <vector>

#include "../../include/vif.h"
#include "common.cuh"
#include "kernels.h"

using namespace vif;

namespace {

constexpr int kPlanSMs = 148;  // SM count used for host-side workspace planning (B200)
constexpr int kLogdParts = 256;
constexpr int64_t kSingleRounds = 1;  // measured: 2 / 4 / 8 rounds are 2-7% slower (kernels barely co-run)

thread_local std::string g_create_error;

// ---------------------------------------------------------------- NCCL (dlopen)
struct Nccl {
  void* lib = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t*) = nullptr;
  ncclResult_t (*CommAbort)(ncclComm_t) = nullptr;
  bool ok = false;
};

Nccl& nccl() {
  static Nccl n;
  static bool tried = false;
  if (!tried) {
    tried = true;
    n.lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (n.lib) {
      n.GetUniqueId = (decltype(n.GetUniqueId))dlsym(n.lib, "ncclGetUniqueId");
      n.CommInitRank = (decltype(n.CommInitRank))dlsym(n.lib, "ncclCommInitRank");
      n.AllGather = (decltype(n.AllGather))dlsym(n.lib, "ncclAllGather");
      n.AllReduce = (decltype(n.AllReduce))dlsym(n.lib, "ncclAllReduce");
      n.CommDestroy = (decltype(n.CommDestroy))dlsym(n.lib, "ncclCommDestroy");
      n.GroupStart = (decltype(n.GroupStart))dlsym(n.lib, "ncclGroupStart");
      n.GroupEnd = (decltype(n.GroupEnd))dlsym(n.lib, "ncclGroupEnd");
      n.GetErrorString = (decltype(n.GetErrorString))dlsym(n.lib, "ncclGetErrorString");
      n.CommGetAsyncError = (decltype(n.CommGetAsyncError))dlsym(n.lib, "ncclCommGetAsyncError");
      n.CommAbort = (decltype(n.CommAbort))dlsym(n.lib, "ncclCommAbort");
      n.ok = n.GetUniqueId && n.CommInitRank && n.AllGather && n.AllReduce && n.CommDestroy && n.GroupStart &&
             n.GroupEnd && n.GetErrorString && n.CommGetAsyncError && n.CommAbort;
    }
  }
  return n;
}

// ---------------------------------------------------------------- derived dims + layout
struct Plan {
  int64_t n;
  int d, m, mv, rank, world;
  bool emulate;
  int mk, ycol, ld;
  int64_t rounds, chunk, npos, npad;
  int nsplit, nsplit_round;
  bool syrk_i8;    // K4 on the integer tensor cores (k_ozaki.cu); VIF_SYRK_FP64=1 keeps the DMMA SYRK
  bool k1_i8;      // K1 on the integer tensor cores (k_ozaki.cu); VIF_UFEAT_FP64=1 keeps kx_eval + DMMA GEMM
  bool grad_i8;    // the gradient's n x m^2 GEMMs (Gamma, T) likewise; VIF_GRAD_FP64=1 keeps the DMMA GEMMs
  int64_t oz_cap;  // rows per digit-slice chunk
  std::vector<int64_t> n_own;
};

enum Buf {
  B_X, B_Z, B_NBR, B_Y, B_KM, B_LINV, B_U, B_W, B_DPOS, B_ORDER, B_KEYS, B_KEYS2, B_VALS, B_VALS2, B_TEMP,
  B_GPART, B_G, B_GSUM, B_LINVM, B_TSCR, B_PART, B_BBOX, B_TERMS, B_STATUS, B_WS, B_OZAUX, B_OZK1,
  // second input slot (vif_stage_data: inputs of the next evaluation copied while this one runs)
  B_X2, B_Z2, B_NBR2, B_Y2, B_ORDER2,
  // sort scratch of the staging path (its sort runs on the copy stream, beside the main stream's work)
  B_SKEYS, B_SKEYS2, B_SVALS, B_SVALS2, B_STEMP, B_SBBOX, B_COUNT
};

inline Buf slot_buf(Buf b, int sl) {
  if (sl == 0) return b;
  switch (b) {
    case B_X: return B_X2;
    case B_Z: return B_Z2;
    case B_NBR: return B_NBR2;
    case B_Y: return B_Y2;
    case B_ORDER: return B_ORDER2;
    default: return b;
  }
}

struct Layout {
  size_t off[B_COUNT];
  size_t size[B_COUNT];
  size_t total;
};

inline int64_t round_up(int64_t a, int64_t b) { return (a + b - 1) / b * b; }

bool make_plan(const vif_dims* dims, bool emulate, Plan& P, std::string& err) {
  if (!dims) { err = "dims is NULL"; return false; }
  if (dims->n < 1) { err = "n must be >= 1"; return false; }
  if (dims->d < 1 || dims->d > VIF_MAX_D) { err = "d must be in [1, VIF_MAX_D]"; return false; }
  if (dims->m < 0) { err = "m must be >= 0"; return false; }
  if (dims->mv < 0 || dims->mv > VIF_MAX_MV) { err = "mv must be in [0, VIF_MAX_MV]"; return false; }
  if (dims->n > (int64_t)0x7fffffff) { err = "n must fit in int32 (neighbour indices are int32)"; return false; }
  if (dims->world < 1 || dims->rank < 0 || dims->rank >= dims->world) { err = "need 0 <= rank < world"; return false; }
  P.n = dims->n; P.d = dims->d; P.m = dims->m; P.mv = dims->mv; P.rank = dims->rank; P.world = dims->world;
  P.emulate = emulate && dims->world > 1;
  P.mk = (int)round_up(P.m, 8);
  P.ycol = P.mk;
  P.ld = (int)round_up(P.mk + 1, 8);
  // VIF_NCCL_SINGLE=1 (test only): a single-rank handle given an NCCL id runs the multi-GPU schedule
  // (8 rounds, per-round all-gather, all-reduce) on a one-rank communicator, exercising the NCCL
  // plumbing on one GPU without ranks that wait on each other
  static const char* nccl1 = getenv("VIF_NCCL_SINGLE");
  const bool single_nccl = P.world == 1 && nccl1 && nccl1[0] == '1';
  if (P.world == 1 && !single_nccl) {
    // single GPU: R rounds on three streams (K1 of round r+1 and the SYRK of round r-1 run beside
    // the vecchia rows of round r and fill the DMMA pipe while those warps are in their scalar
    // phases); VIF_ROUNDS overrides, 1 = the plain serial schedule
    static const char* env = getenv("VIF_ROUNDS");
    int64_t R = env ? atoll(env) : kSingleRounds;
    if (R < 1) R = 1;
    if (P.n < R * 1024) R = 1;
    P.rounds = R;
    P.chunk = (P.n + R - 1) / R;
  } else {
    P.rounds = 8;
    P.chunk = (P.n + P.rounds * P.world - 1) / (P.rounds * P.world);
    if (P.chunk < 1) P.chunk = 1;
  }
  P.npos = P.rounds * P.chunk;
  P.npad = P.npos * P.world;
  P.n_own.assign(P.world, 0);
  for (int g = 0; g < P.world; ++g)
    for (int64_t r = 0; r < P.rounds; ++r) {
      const int64_t start = (r * P.world + g) * P.chunk;
      const int64_t cnt = P.n - start;
      P.n_own[g] += cnt <= 0 ? 0 : (cnt < P.chunk ? cnt : P.chunk);
    }
  P.nsplit = syrk_nsplit(P.ld, P.npos, kPlanSMs);
  P.nsplit_round = syrk_nsplit(P.ld, P.chunk, kPlanSMs);
  {
    const char* f = getenv("VIF_SYRK_FP64");
    P.syrk_i8 = syrk_i8_supported(P.ld) && !(f && f[0] == '1');
    P.oz_cap = std::min<int64_t>(std::max<int64_t>(P.npos, 1), (int64_t)1 << 20);
    const char* fk = getenv("VIF_UFEAT_FP64");
    P.k1_i8 = P.mk > 0 && ufeat_i8_supported(P.d, P.mk) && !(fk && fk[0] == '1');
    const char* fg = getenv("VIF_GRAD_FP64");
    P.grad_i8 = P.mk > 0 && P.ld <= 4096 && !(fg && fg[0] == '1');
  }
  return true;
}

Layout make_layout(const Plan& P) {
  Layout L{};
  const size_t D8 = sizeof(double);
  const int nrep = P.emulate ? P.world : 1;
  const size_t gsz = ((size_t)P.ld * P.ld + 8) * D8;
  const int64_t m1 = P.m > 0 ? P.m : 1, mk1 = P.mk > 0 ? P.mk : 1;
  L.size[B_X] = (size_t)P.n * P.d * D8;
  L.size[B_Z] = (size_t)m1 * P.d * D8;
  L.size[B_NBR] = (size_t)P.n * (P.mv > 0 ? P.mv : 1) * sizeof(int32_t);
  L.size[B_Y] = (size_t)P.n * D8;
  L.size[B_KM] = (size_t)m1 * m1 * D8;
  L.size[B_LINV] = (size_t)mk1 * mk1 * D8;
  L.size[B_U] = (size_t)P.npad * P.ld * D8;
  // an emulated multi-rank handle keeps every virtual rank's W and D rows (vif_grad reads them back)
  L.size[B_W] = (size_t)nrep * P.npos * P.ld * D8;
  L.size[B_DPOS] = (size_t)nrep * P.npos * D8;
  L.size[B_ORDER] = (size_t)nrep * P.npos * sizeof(int64_t);
  L.size[B_KEYS] = L.size[B_KEYS2] = L.size[B_VALS] = L.size[B_VALS2] = (size_t)P.npos * 8;
  L.size[B_TEMP] = order_temp_bytes(P.npos);
  L.size[B_GPART] = std::max(syrk_part_doubles(P.ld, P.nsplit),
                             (size_t)P.rounds * syrk_part_doubles(P.ld, P.nsplit_round)) * D8;
  if (P.syrk_i8) {
    L.size[B_GPART] = std::max(L.size[B_GPART], syrk_i8_part_doubles(P.ld, P.oz_cap) * D8);
    L.size[B_WS] = syrk_i8_ws_bytes(P.ld, P.oz_cap);
    // + the vecchia W pass' column maxima of |W| (64 interleaved copies, see VecchiaArgs::cmax)
    L.size[B_OZAUX] = (syrk_i8_aux_bytes(P.ld) + 255) / 256 * 256 + (size_t)64 * P.ld * sizeof(unsigned long long);
  }
  if (P.k1_i8) {
    L.size[B_WS] = std::max(L.size[B_WS], ufeat_i8_ws_bytes(P.mk, P.oz_cap));
    L.size[B_OZK1] = ufeat_i8_aux_bytes(P.mk, P.oz_cap);
  }
  if (P.grad_i8) {
    L.size[B_WS] = std::max(L.size[B_WS], gemm_i8_ws_bytes(P.ld, P.oz_cap));
    // G2 = R^T U slices both operands (mk columns each) per row chunk: at least half the chunk of the others
    const int64_t ncp = (P.mk + 127) / 128 * 128, rows = std::min<int64_t>(P.n, P.oz_cap / 2 + 64);
    L.size[B_WS] = std::max(L.size[B_WS], (size_t)7 * 2 * ncp * (size_t)((rows + 63) / 64 * 64));
    L.size[B_OZK1] = std::max(L.size[B_OZK1], gemm_i8_aux_bytes(P.ld, P.ld, P.oz_cap));
  }
  L.size[B_G] = nrep * gsz;
  L.size[B_GSUM] = gsz;
  L.size[B_LINVM] = (size_t)mk1 * mk1 * D8;
  L.size[B_TSCR] = (size_t)mk1 * mk1 * D8;
  L.size[B_PART] = kLogdParts * D8;
  L.size[B_BBOX] = 128 * 6 * D8;
  L.size[B_TERMS] = 8 * D8;
  L.size[B_STATUS] = 256;
  L.size[B_X2] = L.size[B_X];
  L.size[B_Z2] = L.size[B_Z];
  L.size[B_NBR2] = L.size[B_NBR];
  L.size[B_Y2] = L.size[B_Y];
  L.size[B_ORDER2] = L.size[B_ORDER];
  L.size[B_SKEYS] = L.size[B_KEYS];
  L.size[B_SKEYS2] = L.size[B_KEYS2];
  L.size[B_SVALS] = L.size[B_VALS];
  L.size[B_SVALS2] = L.size[B_VALS2];
  L.size[B_STEMP] = L.size[B_TEMP];
  L.size[B_SBBOX] = L.size[B_BBOX];
  size_t off = 0;
  for (int b = 0; b < B_COUNT; ++b) {
    L.off[b] = off;
    off += (L.size[b] + 255) / 256 * 256;
  }
  L.total = off + 256;  // slack for base alignment
  return L;
}

enum Stage { S_KM = 0, S_UFEAT, S_GATHER, S_VECCHIA, S_SYRK, S_REDUCE, S_CHOLM, S_FINISH, S_COUNT };
const char* kStageNames[S_COUNT] = {
    "K0 K_m + chol/inv (cooperative)", "K1 U features (int8 slices on tcgen05; kx_eval + DMMA gemm_tn with VIF_UFEAT_FP64=1)", "A2 U all-gather (NCCL)",
    "K2+K3 vecchia rows (gather + DMMA Gram + chol + W row)", "K4 syrk (int8 digit slices on tcgen05; DMMA with VIF_SYRK_FP64=1)",
    "A6/A7 sum log D + all-reduce", "K5 chol/inv of M (cooperative)", "K5 finish (z, quad, NLL)"};

struct Handle {
  Plan P;
  Layout L;
  char* base = nullptr;
  cudaStream_t stream = nullptr;
  int num_sms = 148;
  ncclComm_t comm = nullptr;
  bool comm_dead = false;                    // aborted after an asynchronous error / timeout
  cudaStream_t cstream = nullptr;            // communication stream (world > 1 with NCCL)
  std::vector<cudaEvent_t> ev_k1, ev_ag;     // per round: K1 done / all-gather done
  // single-GPU rounds: K1 and SYRK streams, round events (vecchia done), K0 / SYRK done
  cudaStream_t s_k1 = nullptr, s_sy = nullptr;
  std::vector<cudaEvent_t> ev_v;
  cudaEvent_t ev_k0 = nullptr, ev_sy = nullptr;
  bool have_data = false, factored = false, finished = false;
  vif_terms cached{};
  int cached_status = VIF_OK;
  std::string err;
  int64_t launches = 0;
  // input slots: `slot` holds the inputs the next evaluation uses; vif_stage_data fills the other one
  // on s_copy (ev_ready), swapped in by the next vif_factor / vif_neighbors; ev_free[k] = last use of k
  int slot = 0, pending = -1;
  cudaStream_t s_copy = nullptr;
  cudaEvent_t ev_ready[2] = {}, ev_free[2] = {};
  // VIF-Laplace state (vif_la_prepare): valid while fgen == la_gen (every vif_factor bumps fgen)
  uint64_t fgen = 0, la_gen = ~0ull;
  const void* la_ws = nullptr;
  int la_epoch = 0, la_nprobe = 0, la_maxcg = 0, la_nlev_f = 0, la_nlev_b = 0;
  double la_sigma2 = 0.0;
  // set by vif_grad around its vif_factor call: the vecchia rows also write the gradient state there
  double* grad_state = nullptr;
  // profiling
  bool prof = false;
  cudaEvent_t ev[S_COUNT][2] = {};
  bool ev_used[S_COUNT] = {};
  double stage_ms[S_COUNT] = {};
  int64_t prof_evals = 0;

  void mark(int stage, int which) {
    if (!prof) return;
    if (!ev[stage][which]) cudaEventCreate(&ev[stage][which]);
    if (which == 0 && ev_used[stage]) return;  // keep the first begin of a multi-part stage
    cudaEventRecord(ev[stage][which], stream);
    if (which == 0) ev_used[stage] = true;
  }

  template <typename T>
  T* buf(Buf b) const { return reinterpret_cast<T*>(base + L.off[slot_buf(b, slot)]); }
  template <typename T>
  T* buf_slot(Buf b, int sl) const { return reinterpret_cast<T*>(base + L.off[slot_buf(b, sl)]); }
  // processing order of (logical) rank g for the current input slot
  const int64_t* ord(int g) const { return buf<int64_t>(B_ORDER) + (size_t)g * P.npos; }
};

int fail(Handle* h, int code, const std::string& msg) {
  if (h) h->err = msg;
  else g_create_error = msg;
  return code;
}

int cuda_fail(Handle* h, cudaError_t e, const char* where) {
  return fail(h, VIF_ERR_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

#define VIF_CUDA(h, call, where)                   \
  do {                                             \
    cudaError_t e_ = (call);                       \
    if (e_ != cudaSuccess) return cuda_fail(h, e_, where); \
  } while (0)

// Wait for the work on `s`.  Without a communicator: cudaStreamSynchronize.  With one (world > 1), a
// peer that died or hung would leave a collective on the stream forever, so the wait polls the stream
// and ncclCommGetAsyncError, and gives up after VIF_NCCL_TIMEOUT_S seconds (default 600): the
// communicator is aborted (its kernels exit, the stream drains) and the call returns VIF_ERR_NCCL;
// the handle's later collective calls fail with VIF_ERR_NCCL too.
int wait_stream(Handle* h, cudaStream_t s) {
  if (!h->comm) {
    if (h->comm_dead) return fail(h, VIF_ERR_NCCL, "the communicator was aborted by an earlier error");
    VIF_CUDA(h, cudaStreamSynchronize(s), "sync");
    return VIF_OK;
  }
  static const char* tenv = getenv("VIF_NCCL_TIMEOUT_S");
  const double limit = tenv ? atof(tenv) : 600.0;
  Nccl& N = nccl();
  const auto t0 = std::chrono::steady_clock::now();
  unsigned spin = 0;
  for (;;) {
    const cudaError_t q = cudaStreamQuery(s);
    if (q == cudaSuccess) return VIF_OK;
    if (q != cudaErrorNotReady) return cuda_fail(h, q, "sync");
    ncclResult_t ar = ncclSuccess;
    N.CommGetAsyncError(h->comm, &ar);
    const double el = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if ((ar != ncclSuccess && ar != ncclInProgress) || el > limit) {
      std::string msg = ar != ncclSuccess && ar != ncclInProgress
                            ? std::string("NCCL asynchronous error: ") + N.GetErrorString(ar)
                            : std::string("NCCL collective did not complete within VIF_NCCL_TIMEOUT_S");
      N.CommAbort(h->comm);
      h->comm = nullptr;
      h->comm_dead = true;
      cudaStreamSynchronize(s);  // the aborted collectives return; the stream drains
      return fail(h, VIF_ERR_NCCL, msg);
    }
    if (++spin > 64) std::this_thread::sleep_for(std::chrono::microseconds(20));
  }
}

#define VIF_WAIT(h, s)                 \
  do {                                 \
    const int w_ = wait_stream(h, s);  \
    if (w_ != VIF_OK) return w_;       \
  } while (0)

bool make_params(const Handle* h, const vif_theta* th, CovParams& p, std::string& err) {
  if (!th) { err = "theta is NULL"; return false; }
  if (th->d != h->P.d) { err = "theta.d != dims.d"; return false; }
  if (th->family < 0 || th->family > 3) { err = "unknown covariance family"; return false; }
  if (!(th->sigma2 > 0.0) || !isfinite(th->sigma2)) { err = "sigma2 must be finite and > 0"; return false; }
  if (!(th->nugget >= 0.0) || !isfinite(th->nugget)) { err = "nugget must be finite and >= 0"; return false; }
  if (!(th->jitter >= 0.0) || !isfinite(th->jitter)) { err = "jitter must be finite and >= 0"; return false; }
  if (!th->lengthscale) { err = "lengthscale is NULL"; return false; }
  memset(&p, 0, sizeof(p));
  for (int k = 0; k < th->d; ++k) {
    const double l = th->lengthscale[k];
    if (!(l > 0.0) || !isfinite(l)) { err = "lengthscales must be finite and > 0"; return false; }
    p.inv_ls[k] = 1.0 / l;
  }
  p.sigma2 = th->sigma2;
  p.nugget = th->nugget;
  p.jitter = th->jitter;
  p.d = th->d;
  p.family = th->family;
  return true;
}

int compute_orders(Handle* h, int sl, cudaStream_t strm, bool staging = false) {
  const Plan& P = h->P;
  const int nrep = P.emulate ? P.world : 1;
  for (int g = 0; g < nrep; ++g) {
    const int rank = P.emulate ? g : P.rank;
    int64_t* sorted = nullptr;
    VIF_CUDA(h, launch_order(h->buf_slot<double>(B_X, sl), P.n, P.d, P.npos, P.chunk, P.world, rank,
                             h->buf<double>(staging ? B_SBBOX : B_BBOX), h->buf<uint64_t>(staging ? B_SKEYS : B_KEYS),
                             h->buf<uint64_t>(staging ? B_SKEYS2 : B_KEYS2), h->buf<int64_t>(staging ? B_SVALS : B_VALS),
                             h->buf<int64_t>(staging ? B_SVALS2 : B_VALS2), h->buf<void>(staging ? B_STEMP : B_TEMP),
                             h->L.size[B_TEMP], &sorted, strm, h->buf_slot<int32_t>(B_NBR, sl), P.mv),
             "order");
    int64_t* dst = h->buf_slot<int64_t>(B_ORDER, sl) + (size_t)g * P.npos;
    VIF_CUDA(h, cudaMemcpyAsync(dst, sorted, P.npos * sizeof(int64_t), cudaMemcpyDeviceToDevice, strm), "order copy");
  }
  return VIF_OK;
}

// make a staged input slot current (the work on the stream waits for its copies)
int apply_pending(Handle* h) {
  if (h->pending < 0) return VIF_OK;
  VIF_CUDA(h, cudaStreamWaitEvent(h->stream, h->ev_ready[h->pending], 0), "event wait");
  h->slot = h->pending;
  h->pending = -1;
  ++h->fgen;  // new inputs: a prepared Laplace workspace no longer matches them
  return VIF_OK;
}

int mark_inputs_used(Handle* h) {
  if (h->ev_free[h->slot]) VIF_CUDA(h, cudaEventRecord(h->ev_free[h->slot], h->stream), "event");
  return VIF_OK;
}

int set_data(Handle* h, const double* X, const double* Z, const int32_t* nbr, const double* y, int validate) {
  const Plan& P = h->P;
  cudaStream_t s = h->stream;
  {
    int r = apply_pending(h);
    if (r != VIF_OK) return r;
  }
  if (X) VIF_CUDA(h, cudaMemcpyAsync(h->buf<double>(B_X), X, P.n * P.d * 8, cudaMemcpyDefault, s), "copy X");
  if (Z && P.m > 0) VIF_CUDA(h, cudaMemcpyAsync(h->buf<double>(B_Z), Z, (size_t)P.m * P.d * 8, cudaMemcpyDefault, s), "copy Z");
  if (nbr && P.mv > 0)
    VIF_CUDA(h, cudaMemcpyAsync(h->buf<int32_t>(B_NBR), nbr, (size_t)P.n * P.mv * 4, cudaMemcpyDefault, s), "copy nbr");
  if (y) VIF_CUDA(h, cudaMemcpyAsync(h->buf<double>(B_Y), y, P.n * 8, cudaMemcpyDefault, s), "copy y");
  if (X) {
    int r = compute_orders(h, h->slot, s);
    if (r != VIF_OK) return r;
  }
  if (X || Z || nbr || y) {
    h->have_data = h->have_data || (X && y && (nbr || P.mv == 0) && (Z || P.m == 0));
    h->factored = h->finished = false;
    ++h->fgen;  // a prepared Laplace workspace (la_check) was built from the old inputs
  }
  if (validate) {
    DevStatus* st = h->buf<DevStatus>(B_STATUS);
    VIF_CUDA(h, launch_reset_status(st, s), "reset status");
    VIF_CUDA(h, launch_validate(h->buf<double>(B_X), P.n, P.d, h->buf<double>(B_Z), P.m, h->buf<double>(B_Y),
                                h->buf<int32_t>(B_NBR), P.mv > 0 ? P.mv : 0, st, s),
             "validate");
    DevStatus hs;
    VIF_CUDA(h, cudaMemcpyAsync(&hs, st, sizeof(hs), cudaMemcpyDeviceToHost, s), "status copy");
    VIF_WAIT(h, s);
    if (hs.bad_input != ~0ULL) {
      char msg[160];
      snprintf(msg, sizeof msg, "invalid input at row %llu (non-finite X/y or neighbour rule: N(i) < i, unique, -1 only trailing)",
               hs.bad_input);
      return fail(h, VIF_ERR_INVALID_ARG, msg);
    }
    if (hs.bad_z) return fail(h, VIF_ERR_INVALID_ARG, "non-finite inducing point");
  }
  return VIF_OK;
}

// ---------------------------------------------------------------- gradient workspace
enum GBuf { G_Q2, G_GAM, G_DU, G_DKM, G_TT, G_PHI, G_PHILOW, G_LINVM, G_MCOPY, G_TSCR, G_ZH, G_Z, G_PART, G_OUT,
            G_STATE, G_RHO, G_SIG, G_ADJ, G_T, G_G2, G_LINVT, G_CCNT, G_CCUR, G_CPTR, G_CENT, G_TSP, G_TDKP, G_TDK,
            G_COUNT };

Layout make_grad_layout(const Plan& P) {
  Layout L{};
  const size_t D8 = sizeof(double);
  const int64_t mk1 = P.mk > 0 ? P.mk : 1;
  L.size[G_Q2] = (size_t)P.ld * P.ld * D8;
  L.size[G_GAM] = (size_t)P.npos * P.ld * D8;
  L.size[G_DU] = (size_t)P.npad * P.ld * D8;
  L.size[G_DKM] = L.size[G_TT] = L.size[G_PHI] = L.size[G_PHILOW] = L.size[G_LINVM] = L.size[G_TSCR] =
      (size_t)mk1 * mk1 * D8;
  L.size[G_MCOPY] = (size_t)P.ld * P.ld * D8;
  L.size[G_ZH] = L.size[G_Z] = (size_t)mk1 * D8;
  L.size[G_PART] = (size_t)(P.d + 2) * grad_point_nparts(P.npos) * D8;
  L.size[G_OUT] = (size_t)(P.d + 2) * (P.emulate ? P.world : 1) * D8;
  L.size[G_STATE] = (size_t)P.npos * grad_state_doubles(P.mv) * D8;
  L.size[G_RHO] = L.size[G_SIG] = (size_t)P.npos * mk1 * D8;
  L.size[G_ADJ] = (size_t)P.npos * grad_adj_doubles() * D8;
  L.size[G_T] = (size_t)P.n * mk1 * D8;
  L.size[G_G2] = L.size[G_LINVT] = (size_t)mk1 * mk1 * D8;
  L.size[G_CCNT] = L.size[G_CCUR] = (size_t)P.n * sizeof(int);
  L.size[G_CPTR] = (size_t)(P.n + 1) * sizeof(int);
  L.size[G_CENT] = (size_t)2 * P.n * (P.mv + 1) * sizeof(int);  // sorted entries + the unsorted fill
  L.size[G_TSP] = gemm_tt_part_doubles((int)mk1, (int)mk1, gemm_tt_nsplit((int)mk1, (int)mk1, P.n, kPlanSMs)) * D8;
  if (P.grad_i8) {
    const size_t ws = make_layout(P).size[B_WS];
    L.size[G_TSP] = std::max(L.size[G_TSP], gemm_tt_i8_part_doubles((int)mk1, (int)mk1,
                                                                    gemm_tt_i8_chunk((int)mk1, (int)mk1, ws)) * D8);
  }
  L.size[G_TDKP] = (size_t)gTdK_blocks() * (P.d + 1) * D8;
  L.size[G_TDK] = (size_t)(P.d + 2) * D8;  // + the R gather's row counter
  size_t off = 0;
  for (int b = 0; b < G_COUNT; ++b) {
    L.off[b] = off;
    off += (L.size[b] + 255) / 256 * 256;
  }
  L.total = off + 256;
  return L;
}

// ---------------------------------------------------------------- prediction workspace
enum PBuf { P_X, P_NBR, P_Y, P_U, P_S, P_W, P_DPOS, P_KEYS, P_KEYS2, P_VALS, P_VALS2, P_TEMP, P_BBOX, P_LINVM,
            P_MCOPY, P_TSCR, P_ZH, P_Z, P_COUNT };

Layout make_pred_layout(const Plan& P, int64_t np) {
  Layout L{};
  const size_t D8 = sizeof(double);
  const int64_t mk1 = P.mk > 0 ? P.mk : 1;
  L.size[P_X] = (size_t)np * P.d * D8;
  L.size[P_NBR] = (size_t)np * (P.mv > 0 ? P.mv : 1) * sizeof(int32_t);
  L.size[P_Y] = (size_t)np * D8;
  L.size[P_U] = (size_t)np * P.ld * D8;
  L.size[P_S] = (size_t)np * mk1 * D8;
  L.size[P_W] = (size_t)np * P.ld * D8;
  L.size[P_DPOS] = (size_t)np * D8;
  L.size[P_KEYS] = L.size[P_KEYS2] = L.size[P_VALS] = L.size[P_VALS2] = (size_t)np * 8;
  L.size[P_TEMP] = order_temp_bytes(np);
  L.size[P_BBOX] = 128 * 6 * D8;
  L.size[P_LINVM] = L.size[P_TSCR] = (size_t)mk1 * mk1 * D8;
  L.size[P_MCOPY] = (size_t)P.ld * P.ld * D8;
  L.size[P_ZH] = L.size[P_Z] = (size_t)mk1 * D8;
  size_t off = 0;
  for (int b = 0; b < P_COUNT; ++b) {
    L.off[b] = off;
    off += (L.size[b] + 255) / 256 * 256;
  }
  L.total = off + 256;
  return L;
}

// ---------------------------------------------------------------- VIF-Laplace workspace
enum LBuf {
  L_B, L_D, L_FLAGS, L_TPTR, L_TPOS, L_CNT, L_CUR, L_TICKET, L_UN2, L_W, L_WINV, L_V, L_BM, L_A, L_DV, L_DVINV,
  L_S, L_GV, L_LVINV, L_LVT, L_MVINV, L_TSCR, L_GPART, L_TSPART, L_CT, L_CT2, L_RPART, L_SC, L_ACTIVE, L_ITERS,
  L_HA, L_HB, L_SLQS, L_X, L_R, L_Z, L_P, L_Q, L_T1, L_T2, L_RHS, L_E1T, L_GM, L_LMINV, L_TROW, L_TVAL, L_LEVF,
  L_LEVB, L_ORDF, L_ORDB, L_LPTRF, L_LPTRB, L_ECF, L_EVF, L_ECB, L_EVB, L_EPB, L_IPOS,
  L_LMINVT, L_T3, L_COUNT
};
// per-column scalar arrays inside L_SC (each kLaCols doubles)
enum LScal { SC_RZ, SC_RZN, SC_PQ, SC_ALPHA, SC_BETA, SC_RR, SC_BN, SC_SLQ, SC_MISC, SC_OUT, SC_COUNT };
constexpr int kLaCols = 64;  // maximum columns (probe vectors) of one block solve

struct LaLayout {
  size_t off[L_COUNT];
  size_t size[L_COUNT];
  size_t total;
};

LaLayout make_la_layout(const Plan& P, int nprobe, int max_cg) {
  LaLayout L{};
  const size_t D8 = sizeof(double);
  const int64_t n = P.n, mv1 = P.mv > 0 ? P.mv : 1, mk1 = P.mk > 0 ? P.mk : 1;
  const int ncol = nprobe > 1 ? nprobe : 1;
  const int kmax = max_cg > 1 ? max_cg : 1;
  const int ns_syrk = syrk_nsplit(P.ld, n, kPlanSMs);
  L.size[L_B] = (size_t)n * mv1 * D8;
  L.size[L_D] = L.size[L_UN2] = L.size[L_W] = L.size[L_WINV] = L.size[L_V] = L.size[L_BM] = L.size[L_A] =
      L.size[L_DV] = L.size[L_DVINV] = (size_t)n * D8;
  L.size[L_FLAGS] = L.size[L_CNT] = L.size[L_CUR] = (size_t)n * sizeof(int);
  L.size[L_TPTR] = (size_t)(n + 1) * sizeof(int);
  L.size[L_TPOS] = L.size[L_TROW] = (size_t)n * mv1 * sizeof(int);
  L.size[L_TVAL] = (size_t)n * mv1 * D8;
  L.size[L_LEVF] = L.size[L_LEVB] = L.size[L_ORDF] = L.size[L_ORDB] = (size_t)n * sizeof(int);
  L.size[L_LPTRF] = L.size[L_LPTRB] = L.size[L_EPB] = (size_t)(n + 1) * sizeof(int);
  L.size[L_IPOS] = (size_t)n * sizeof(int);
  L.size[L_LMINVT] = (size_t)mk1 * mk1 * D8;
  L.size[L_T3] = (size_t)(P.npos > n ? P.npos : n) * ncol * D8;
  L.size[L_ECF] = L.size[L_ECB] = (size_t)n * mv1 * sizeof(int);
  L.size[L_EVF] = L.size[L_EVB] = (size_t)n * mv1 * D8;
  L.size[L_TICKET] = 64;
  L.size[L_S] = (size_t)n * P.ld * D8;
  L.size[L_GV] = (size_t)P.ld * P.ld * D8;
  L.size[L_LVINV] = L.size[L_LVT] = L.size[L_MVINV] = L.size[L_TSCR] = L.size[L_LMINV] = (size_t)mk1 * mk1 * D8;
  L.size[L_GM] = (size_t)P.ld * P.ld * D8;
  L.size[L_GPART] = syrk_part_doubles(P.ld, ns_syrk) * D8;
  L.size[L_TSPART] = (size_t)la_ts_nsplit(n) * ncol * mk1 * D8;
  L.size[L_CT] = L.size[L_CT2] = L.size[L_E1T] = (size_t)ncol * mk1 * D8;
  L.size[L_RPART] = (size_t)la_red_nsplit(n > mk1 ? n : mk1) * ncol * D8;
  L.size[L_SC] = (size_t)SC_COUNT * kLaCols * D8;
  L.size[L_ACTIVE] = L.size[L_ITERS] = (size_t)kLaCols * sizeof(int);
  L.size[L_HA] = L.size[L_HB] = (size_t)kmax * ncol * D8;
  L.size[L_SLQS] = (size_t)3 * kmax * ncol * D8;
  L.size[L_X] = L.size[L_R] = L.size[L_Z] = L.size[L_P] = L.size[L_Q] = L.size[L_T1] = L.size[L_T2] =
      L.size[L_RHS] = (size_t)n * ncol * D8;
  size_t off = 0;
  for (int b = 0; b < L_COUNT; ++b) {
    L.off[b] = off;
    off += (L.size[b] + 255) / 256 * 256;
  }
  L.total = off + 256;
  return L;
}

#define LA_TRY(call)               \
  do {                             \
    int r_ = (call);               \
    if (r_ != VIF_OK) return r_;   \
  } while (0)

// VIF-Laplace helpers: buffers of a prepared workspace and the operators of the iterative path
struct LaCtx {
  Handle* h;
  LaLayout L;
  char* base;
  cudaStream_t s;
  double* d(LBuf b) const { return reinterpret_cast<double*>(base + L.off[b]); }
  int* i(LBuf b) const { return reinterpret_cast<int*>(base + L.off[b]); }
  double* sc(int k) const { return d(L_SC) + (size_t)k * kLaCols; }
  unsigned long long* ticket() const { return reinterpret_cast<unsigned long long*>(base + L.off[L_TICKET]); }
  int* fitc_fail() const { return reinterpret_cast<int*>(base + L.off[L_TICKET] + 8); }
  const double* U() const { return h->buf<double>(B_U); }
  const int32_t* nbr() const { return h->buf<int32_t>(B_NBR); }
};

LaCtx la_ctx(Handle* h, void* ws) {
  LaCtx c{h, make_la_layout(h->P, h->la_nprobe, h->la_maxcg), nullptr, h->stream};
  c.base = reinterpret_cast<char*>(round_up((int64_t)(uintptr_t)ws, 256));
  return c;
}

// B^{-1} (s o v) -> x [out2 = x + w2 o v2] and B^{-T} u -> y: level-scheduled cooperative kernels

int la_binv(LaCtx& c, int ncol, const double* v, const double* scale, double* x, const double* v2, const double* w2,
            double* out2) {
  Handle* h = c.h;
  const Plan& P = h->P;
  VIF_CUDA(h, launch_la_trsv_lvl(true, c.i(L_ORDF), c.i(L_LPTRF), h->la_nlev_f, c.i(L_ECF), c.d(L_EVF), nullptr,
                                   P.mv, ncol, v, scale, x, v2, w2, out2, c.s),
             "B^-1 (levels)");
  return VIF_OK;
}

int la_btinv(LaCtx& c, int ncol, const double* u, double* y) {
  Handle* h = c.h;
  const Plan& P = h->P;
  VIF_CUDA(h, launch_la_trsv_lvl(false, c.i(L_ORDB), c.i(L_LPTRB), h->la_nlev_b, c.i(L_ECB), c.d(L_EVB),
                                   c.i(L_EPB), P.mv, ncol, u, nullptr, y, nullptr, nullptr, nullptr, c.s),
             "B^-T (levels)");
  return VIF_OK;
}

// out = Sigma_dagger v (+ winv o v): B^{-1} D B^{-T} v + U (U^T v); v, out: n x ncol
int la_sigma(LaCtx& c, int ncol, const double* v, double* out, const double* winv) {
  Handle* h = c.h;
  const Plan& P = h->P;
  if (P.mk > 0)
    VIF_CUDA(h, launch_la_tsgemm(c.U(), P.ld, P.mk, P.n, v, ncol, nullptr, nullptr, c.d(L_TSPART), c.d(L_CT), 1.0,
                                 c.s),
             "U^T v");
  LA_TRY(la_btinv(c, ncol, v, c.d(L_T1)));
  LA_TRY(la_binv(c, ncol, c.d(L_T1), c.d(L_D), winv ? c.d(L_T2) : out, v, winv, winv ? out : nullptr));
  if (P.mk > 0) {
    if (ncol == 1)
      VIF_CUDA(h, launch_la_gemv(c.U(), P.ld, P.n, P.mk, c.d(L_CT), 1.0, 1, out, c.s), "U c");
    else
      VIF_CUDA(h, launch_gemm_tn(c.U(), P.ld, P.n, c.d(L_CT), P.mk, ncol, P.mk, 0, out, ncol, 1.0, 1, c.s), "U C");
  }
  return VIF_OK;
}

// out = Sigma_dagger^{-1} v (+ W v with W = 1/winv): the (pcls1) operator W + Sigma_dagger^{-1},
// Woodbury with the latent factor: B^T D^{-1/2} [s - W_U M^{-1} W_U^T s], s = D^{-1/2} B v
int la_sigma_inv(LaCtx& c, int ncol, const double* v, double* out, const double* winv) {
  Handle* h = c.h;
  const Plan& P = h->P;
  double* sv = c.d(L_T1);
  VIF_CUDA(h, launch_la_bapply_cols(c.nbr(), c.d(L_B), P.mv, P.n, ncol, c.d(L_D), v, sv, c.s), "D^-1/2 B v");
  double* Y = nullptr;
  if (P.mk > 0) {
    VIF_CUDA(h, launch_la_tsgemm(h->buf<double>(B_W), P.ld, P.mk, P.n, sv, ncol, h->ord(0), nullptr, c.d(L_TSPART),
                                 c.d(L_CT), 1.0, c.s),
             "W_U^T s");
    VIF_CUDA(h, launch_gemm_tn(c.d(L_CT), P.mk, ncol, c.d(L_LMINV), P.mk, P.mk, P.mk, 0, c.d(L_CT2), P.mk, 1.0, 0, c.s),
             "L_M^-1 c");
    VIF_CUDA(h, launch_gemm_tn(c.d(L_CT2), P.mk, ncol, c.d(L_LMINVT), P.mk, P.mk, P.mk, 0, c.d(L_CT), P.mk, 1.0, 0,
                               c.s),
             "L_M^-T t");
    Y = c.d(L_T3);
    VIF_CUDA(h, launch_gemm_tn(h->buf<double>(B_W), P.ld, P.n, c.d(L_CT), P.mk, ncol, P.mk, 0, Y, ncol, 1.0, 0, c.s),
             "W_U M^-1 c");
  }
  VIF_CUDA(h, launch_la_woodbury_mid(sv, Y, c.i(L_IPOS), c.d(L_D), P.n, ncol, c.d(L_T2), c.s), "Woodbury");
  VIF_CUDA(h, launch_la_btapply_cols(c.i(L_TPTR), c.i(L_TROW), c.d(L_TVAL), P.n, ncol, c.d(L_T2), winv, v, out, c.s),
           "B^T D^-1/2 r");
  return VIF_OK;
}

// FITC preconditioner at W (App. FITC): D_V, M_V = I + U^T D_V^{-1} U, M_V^{-1}, log det M_V
int la_fitc_build(LaCtx& c, const double* winv) {
  Handle* h = c.h;
  const Plan& P = h->P;
  double* ldmv = c.sc(SC_MISC) + 5;
  VIF_CUDA(h, launch_la_fitc_rows(c.U(), P.ld, P.mk, P.ld, P.n, c.d(L_UN2), h->la_sigma2, winv, c.d(L_DV),
                                  c.d(L_DVINV), c.d(L_S), c.s),
           "FITC rows");
  if (P.mk == 0) {
    VIF_CUDA(h, cudaMemsetAsync(ldmv, 0, sizeof(double), c.s), "memset");
    return VIF_OK;
  }
  const int ns = syrk_nsplit(P.ld, P.n, kPlanSMs);
  VIF_CUDA(h, launch_syrk(c.d(L_S), P.ld, P.n, P.ld, ns, c.d(L_GPART), c.d(L_GV), P.ld, c.s), "FITC syrk");
  VIF_CUDA(h, cudaMemsetAsync(c.d(L_LVINV), 0, c.L.size[L_LVINV], c.s), "memset");
  VIF_CUDA(h, launch_chol_inv(c.d(L_GV), P.m, P.ld, 1.0, c.d(L_LVINV), P.mk, P.mk, 1, c.d(L_TSCR), c.fitc_fail(),
                              h->num_sms, c.s),
           "FITC chol");
  VIF_CUDA(h, launch_la_logdiag(c.d(L_GV), P.m, P.ld, ldmv, c.s), "log det M_V");
  VIF_CUDA(h, launch_la_transpose(c.d(L_LVINV), P.mk, P.mk, P.mk, c.d(L_LVT), P.mk, c.s), "transpose");
  VIF_CUDA(h, launch_gemm_tn(c.d(L_LVT), P.mk, P.mk, c.d(L_LVT), P.mk, P.mk, P.mk, 0, c.d(L_MVINV), P.mk, 1.0, 0, c.s),
           "M_V^-1");
  return VIF_OK;
}

// out = P^{-1} w = D_V^{-1} (w - U M_V^{-1} U^T D_V^{-1} w)
int la_fitc_solve(LaCtx& c, int ncol, const double* w, double* out) {
  Handle* h = c.h;
  const Plan& P = h->P;
  if (P.mk == 0) {
    VIF_CUDA(h, launch_la_rowscale(w, c.d(L_DVINV), 0, P.n, ncol, out, c.s), "D_V^-1 w");
    return VIF_OK;
  }
  VIF_CUDA(h, launch_la_tsgemm(c.U(), P.ld, P.mk, P.n, w, ncol, nullptr, c.d(L_DVINV), c.d(L_TSPART), c.d(L_CT), 1.0,
                               c.s),
           "U^T D_V^-1 w");
  VIF_CUDA(h, launch_gemm_tn(c.d(L_CT), P.mk, ncol, c.d(L_MVINV), P.mk, P.mk, P.mk, 0, c.d(L_CT2), P.mk, 1.0, 0, c.s),
           "M_V^-1 C");
  if (ncol == 1)
    VIF_CUDA(h, launch_la_gemv(c.U(), P.ld, P.n, P.mk, c.d(L_CT2), 1.0, 0, c.d(L_T1), c.s), "U c");
  else
    VIF_CUDA(h, launch_gemm_tn(c.U(), P.ld, P.n, c.d(L_CT2), P.mk, ncol, P.mk, 0, c.d(L_T1), ncol, 1.0, 0, c.s),
             "U C");
  VIF_CUDA(h, launch_la_sub_rowscale(w, c.d(L_T1), c.d(L_DVINV), P.n, ncol, out, c.s), "FITC tail");
  return VIF_OK;
}

int la_coldot(LaCtx& c, const double* a, const double* b, int64_t n, int ncol, double* out) {
  VIF_CUDA(c.h, launch_la_reduce(0, a, b, n, ncol, c.d(L_RPART), out, c.s), "dot");
  return VIF_OK;
}

// Preconditioned CG on (W^{-1} + Sigma_dagger) x = rhs, ncol independent columns (pcls2 P:322;
// Saad 2003 Alg. 9.1), readings l3 (stop at ||r|| <= tol ||rhs||).  x holds x0 when warm.  With
// record, alpha_j / beta_j go to L_HA / L_HB [j][c] for the Lanczos matrices.  iters[c]:
// iterations of column c.
int la_pcg(LaCtx& c, int ncol, const double* rhs, double* x, bool warm, double tol, int max_it, const double* winv,
           bool record, std::vector<int>& iters) {
  Handle* h = c.h;
  const Plan& P = h->P;
  const int64_t tot = P.n * ncol;
  double* R = c.d(L_R);
  double* Z = c.d(L_Z);
  double* Pv = c.d(L_P);
  double* Q = c.d(L_Q);
  if (warm) {
    LA_TRY(la_sigma(c, ncol, x, R, winv));
    VIF_CUDA(h, launch_la_residual(rhs, tot, R, c.s), "residual");
  } else {
    VIF_CUDA(h, cudaMemsetAsync(x, 0, tot * sizeof(double), c.s), "memset x");
    VIF_CUDA(h, cudaMemcpyAsync(R, rhs, tot * sizeof(double), cudaMemcpyDeviceToDevice, c.s), "copy r");
  }
  LA_TRY(la_coldot(c, rhs, rhs, P.n, ncol, c.sc(SC_BN)));
  LA_TRY(la_coldot(c, R, R, P.n, ncol, c.sc(SC_RR)));
  LA_TRY(la_fitc_solve(c, ncol, R, Z));
  LA_TRY(la_coldot(c, R, Z, P.n, ncol, c.sc(SC_RZ)));
  VIF_CUDA(h, cudaMemcpyAsync(Pv, Z, tot * sizeof(double), cudaMemcpyDeviceToDevice, c.s), "copy p");
  std::vector<double> bn(ncol), rr(ncol);
  VIF_CUDA(h, cudaMemcpyAsync(bn.data(), c.sc(SC_BN), ncol * sizeof(double), cudaMemcpyDeviceToHost, c.s), "bn");
  VIF_CUDA(h, cudaMemcpyAsync(rr.data(), c.sc(SC_RR), ncol * sizeof(double), cudaMemcpyDeviceToHost, c.s), "rr");
  VIF_WAIT(h, c.s);
  std::vector<int> active(ncol);
  iters.assign(ncol, 0);
  int nact = 0;
  for (int k = 0; k < ncol; ++k) {
    active[k] = bn[k] > 0.0 && sqrt(rr[k]) > tol * sqrt(bn[k]) && max_it > 0;
    nact += active[k];
  }
  VIF_CUDA(h, cudaMemcpyAsync(c.i(L_ACTIVE), active.data(), ncol * sizeof(int), cudaMemcpyHostToDevice, c.s), "active");
  for (int it = 0; it < max_it && nact > 0; ++it) {
    LA_TRY(la_sigma(c, ncol, Pv, Q, winv));
    LA_TRY(la_coldot(c, Pv, Q, P.n, ncol, c.sc(SC_PQ)));
    VIF_CUDA(h, launch_la_cg_alpha(c.sc(SC_RZ), c.sc(SC_PQ), c.i(L_ACTIVE), ncol, c.sc(SC_ALPHA),
                                   record ? c.d(L_HA) + (size_t)it * ncol : nullptr, c.s),
             "alpha");
    VIF_CUDA(h, launch_la_cg_xr(c.sc(SC_ALPHA), Pv, Q, P.n, ncol, x, R, c.s), "x, r");
    LA_TRY(la_coldot(c, R, R, P.n, ncol, c.sc(SC_RR)));
    VIF_CUDA(h, cudaMemcpyAsync(rr.data(), c.sc(SC_RR), ncol * sizeof(double), cudaMemcpyDeviceToHost, c.s), "rr");
    VIF_WAIT(h, c.s);
    bool changed = false;
    for (int k = 0; k < ncol; ++k) {
      if (!active[k]) continue;
      if (!(sqrt(rr[k]) > tol * sqrt(bn[k])) || it + 1 == max_it) {
        active[k] = 0;
        iters[k] = it + 1;
        --nact;
        changed = true;
      }
    }
    if (nact == 0) break;
    if (changed)
      VIF_CUDA(h, cudaMemcpyAsync(c.i(L_ACTIVE), active.data(), ncol * sizeof(int), cudaMemcpyHostToDevice, c.s),
               "active");
    LA_TRY(la_fitc_solve(c, ncol, R, Z));
    LA_TRY(la_coldot(c, R, Z, P.n, ncol, c.sc(SC_RZN)));
    VIF_CUDA(h, launch_la_cg_beta(c.sc(SC_RZN), c.sc(SC_RZ), c.i(L_ACTIVE), ncol, c.sc(SC_BETA),
                                  record ? c.d(L_HB) + (size_t)it * ncol : nullptr, c.s),
             "beta");
    VIF_CUDA(h, launch_la_cg_p(c.sc(SC_BETA), c.i(L_ACTIVE), Z, P.n, ncol, Pv, c.s), "p");
  }
  return VIF_OK;
}

}  // namespace

// ====================================================================== C ABI
extern "C" {

int vif_nccl_unique_id(void* out128) {
  if (!out128) return fail(nullptr, VIF_ERR_INVALID_ARG, "out128 is NULL");
  Nccl& N = nccl();
  if (!N.ok) return fail(nullptr, VIF_ERR_NCCL, "libnccl.so.2 not loadable");
  ncclUniqueId id;
  ncclResult_t r = N.GetUniqueId(&id);
  if (r != ncclSuccess) return fail(nullptr, VIF_ERR_NCCL, N.GetErrorString(r));
  memcpy(out128, &id, sizeof(id));
  return VIF_OK;
}

int vif_workspace_bytes(const vif_dims* dims, size_t* bytes) {
  Plan P;
  std::string err;
  if (!bytes) return fail(nullptr, VIF_ERR_INVALID_ARG, "bytes is NULL");
  if (!make_plan(dims, true, P, err)) return fail(nullptr, VIF_ERR_INVALID_ARG, err);
  *bytes = make_layout(P).total;
  return VIF_OK;
}

int vif_partition(const vif_dims* dims, int64_t* rounds, int64_t* chunk) {
  Plan P;
  std::string err;
  if (!make_plan(dims, false, P, err)) return fail(nullptr, VIF_ERR_INVALID_ARG, err);
  if (rounds) *rounds = P.rounds;
  if (chunk) *chunk = P.chunk;
  return VIF_OK;
}

int vif_owned_rows(void* handle, int64_t* first_chunk, int64_t* chunk, int32_t* stride, int64_t* nchunks) {
  Handle* h = reinterpret_cast<Handle*>(handle);
  if (!h) return fail(nullptr, VIF_ERR_INVALID_ARG, "handle is NULL");
  const Plan& P = h->P;
  if (first_chunk) *first_chunk = P.emulate ? 0 : P.rank;
  if (chunk) *chunk = P.chunk;
  if (stride) *stride = P.emulate ? 1 : P.world;
  if (nchunks) *nchunks = (P.n + P.chunk - 1) / P.chunk;
  return VIF_OK;
}

int vif_create(void** handle, const vif_dims* dims, void* workspace, size_t ws_bytes, const double* X,
               const double* Z, const int32_t* nbr, const double* y, const void* nccl_id, void* cuda_stream) {
  if (!handle) return fail(nullptr, VIF_ERR_INVALID_ARG, "handle is NULL");
  *handle = nullptr;
  Handle* h = new Handle();
  std::string err;
  if (!make_plan(dims, nccl_id == nullptr, h->P, err)) {
    delete h;
    return fail(nullptr, VIF_ERR_INVALID_ARG, err);
  }
  h->L = make_layout(h->P);
  if (!workspace || ws_bytes < h->L.total) {
    char msg[128];
    snprintf(msg, sizeof msg, "workspace too small: need %zu bytes", h->L.total);
    delete h;
    return fail(nullptr, VIF_ERR_NO_MEMORY, msg);
  }
  h->base = reinterpret_cast<char*>(round_up((int64_t)(uintptr_t)workspace, 256));
  h->stream = reinterpret_cast<cudaStream_t>(cuda_stream);
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&h->num_sms, cudaDevAttrMultiProcessorCount, dev);
  if (e != cudaSuccess) {
    std::string m = std::string("cuda: ") + cudaGetErrorString(e);
    delete h;
    return fail(nullptr, VIF_ERR_CUDA, m);
  }
  // zero the reduction buffers once (their upper triangles are never written)
  e = cudaMemsetAsync(h->base + h->L.off[B_G], 0, h->L.size[B_G], h->stream);
  if (e == cudaSuccess) e = cudaMemsetAsync(h->base + h->L.off[B_GSUM], 0, h->L.size[B_GSUM], h->stream);
  if (e != cudaSuccess) {
    std::string m = std::string("memset: ") + cudaGetErrorString(e);
    delete h;
    return fail(nullptr, VIF_ERR_CUDA, m);
  }
  static const char* nccl1 = getenv("VIF_NCCL_SINGLE");
  const bool single_nccl = h->P.world == 1 && nccl_id && nccl1 && nccl1[0] == '1';
  if ((h->P.world > 1 && !h->P.emulate) || single_nccl) {
    Nccl& N = nccl();
    if (!N.ok) {
      delete h;
      return fail(nullptr, VIF_ERR_NCCL, "libnccl.so.2 not loadable");
    }
    ncclUniqueId id;
    memcpy(&id, nccl_id, sizeof(id));
    ncclResult_t r = N.CommInitRank(&h->comm, h->P.world, id, h->P.rank);
    if (r != ncclSuccess) {
      std::string m = std::string("ncclCommInitRank: ") + N.GetErrorString(r);
      delete h;
      return fail(nullptr, VIF_ERR_NCCL, m);
    }
    // the communication stream at the highest priority: the block scheduler then hands freed SMs to the
    // all-gather kernels first instead of to queued vecchia CTAs (tools/corun_probe.py, CORUN_PRIORITY)
    {
      int lo = 0, hi = 0;
      e = cudaDeviceGetStreamPriorityRange(&lo, &hi);
      if (e == cudaSuccess) e = cudaStreamCreateWithPriority(&h->cstream, cudaStreamNonBlocking, hi);
    }
    h->ev_k1.assign(h->P.rounds, nullptr);
    h->ev_ag.assign(h->P.rounds, nullptr);
    for (int64_t k = 0; k < h->P.rounds && e == cudaSuccess; ++k) {
      e = cudaEventCreateWithFlags(&h->ev_k1[k], cudaEventDisableTiming);
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(&h->ev_ag[k], cudaEventDisableTiming);
    }
    if (e != cudaSuccess) {
      std::string m = std::string("comm stream/events: ") + cudaGetErrorString(e);
      vif_destroy(h);
      return fail(nullptr, VIF_ERR_CUDA, m);
    }
  }
  e = cudaStreamCreateWithFlags(&h->s_copy, cudaStreamNonBlocking);
  for (int k = 0; k < 2 && e == cudaSuccess; ++k) {
    e = cudaEventCreateWithFlags(&h->ev_ready[k], cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&h->ev_free[k], cudaEventDisableTiming);
  }
  if (e != cudaSuccess) {
    std::string m = std::string("copy stream/events: ") + cudaGetErrorString(e);
    vif_destroy(h);
    return fail(nullptr, VIF_ERR_CUDA, m);
  }
  if (h->P.world == 1 && h->P.rounds > 1 && !h->comm) {
    e = cudaStreamCreateWithFlags(&h->s_k1, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&h->s_sy, cudaStreamNonBlocking);
    h->ev_k1.assign(h->P.rounds, nullptr);
    h->ev_v.assign(h->P.rounds, nullptr);
    for (int64_t k = 0; k < h->P.rounds && e == cudaSuccess; ++k) {
      e = cudaEventCreateWithFlags(&h->ev_k1[k], cudaEventDisableTiming);
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(&h->ev_v[k], cudaEventDisableTiming);
    }
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&h->ev_k0, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&h->ev_sy, cudaEventDisableTiming);
    if (e != cudaSuccess) {
      std::string m = std::string("round streams/events: ") + cudaGetErrorString(e);
      vif_destroy(h);
      return fail(nullptr, VIF_ERR_CUDA, m);
    }
  }
  if (X || Z || nbr || y) {
    int r = set_data(h, X, Z, nbr, y, 1);
    if (r != VIF_OK) {
      g_create_error = h->err;
      if (h->comm) nccl().CommDestroy(h->comm);
      delete h;
      return r;
    }
  }
  e = cudaStreamSynchronize(h->stream);
  if (e != cudaSuccess) {
    std::string m = std::string("create sync: ") + cudaGetErrorString(e);
    if (h->comm) nccl().CommDestroy(h->comm);
    delete h;
    return fail(nullptr, VIF_ERR_CUDA, m);
  }
  *handle = h;
  return VIF_OK;
}

int vif_set_data(void* handle, const double* X, const double* Z, const int32_t* nbr, const double* y,
                 int32_t validate) {
  Handle* h = reinterpret_cast<Handle*>(handle);
  if (!h) return fail(nullptr, VIF_ERR_INVALID_ARG, "handle is NULL");
  return set_data(h, X, Z, nbr, y, validate);
}

int vif_stage_data(void* handle, const double* X, const double* Z, const int32_t* nbr, const double* y) {
  Handle* h = reinterpret_cast<Handle*>(handle);
  if (!h) return fail(nullptr, VIF_ERR_INVALID_ARG, "handle is NULL");
  const Plan& P = h->P;
  if (!X || !y || (P.m > 0 && !Z) || (P.mv > 0 && !nbr))
    return fail(h, VIF_ERR_INVALID_ARG, "vif_stage_data: X, Z (m > 0), nbr (m_v > 0) and y are all required");
  const int t = h->pending >= 0 ? h->pending : h->slot ^ 1;  // the slot no queued evaluation reads
  cudaStream_t c = h->s_copy;
  VIF_CUDA(h, cudaStreamWaitEvent(c, h->ev_free[t], 0), "event wait");
  VIF_CUDA(h, cudaMemcpyAsync(h->buf_slot<double>(B_X, t), X, P.n * P.d * 8, cudaMemcpyDefault, c), "copy X");
  if (P.m > 0)
    VIF_CUDA(h, cudaMemcpyAsync(h->buf_slot<double>(B_Z, t), Z, (size_t)P.m * P.d * 8, cudaMemcpyDefault, c),
             "copy Z");
  if (P.mv > 0)
    VIF_CUDA(h, cudaMemcpyAsync(h->buf_slot<int32_t>(B_NBR, t), nbr, (size_t)P.n * P.mv * 4, cudaMemcpyDefault, c),
             "copy nbr");
  VIF_CUDA(h, cudaMemcpyAsync(h->buf_slot<double>(B_Y, t), y, P.n * 8, cudaMemcpyDefault, c), "copy y");
  int r = compute_orders(h, t, c, true);
  if (r != VIF_OK) return r;
  VIF_CUDA(h, cudaEventRecord(h->ev_ready[t], c), "event");
  h->pending = t;
  h->have_data = true;
  return VIF_OK;
}

int vif_factor(void* handle, const vif_theta* theta, double* B_out, double* D_out) {
  Handle* h = reinterpret_cast<Handle*>(handle);
  if (!h) return fail(nullptr, VIF_ERR_INVALID_ARG, "handle is NULL");
  if (!h->have_data) return fail(h, VIF_ERR_STATE, "no data: pass X, Z, nbr, y to vif_create or vif_set_data");
  if (h->comm_dead) return fail(h, VIF_ERR_NCCL, "the communicator was aborted by an earlier error");
  CovParams p;
  std::string err;
  if (!make_params(h, theta, p, err)) return fail(h, VIF_ERR_INVALID_ARG, err);
  const Plan& P = h->P;
  cudaStream_t s = h->stream;
  {
    int r = apply_pending(h);
    if (r != VIF_OK) return r;
  }
  DevStatus* st = h->buf<DevStatus>(B_STATUS);
  int64_t nl = 0;
  ++h->fgen;
  for (int k = 0; k < S_COUNT; ++k) h->ev_used[k] = false;
  VIF_CUDA(h, launch_reset_status(st, s), "reset status");
  ++nl;
  // A0: K_m, L_m, L_m^{-1}
  h->mark(S_KM, 0);
  if (P.m > 0) {
    VIF_CUDA(h, launch_build_km(h->buf<double>(B_Z), P.m, p, h->buf<double>(B_KM), s), "build K_m");
    VIF_CUDA(h, cudaMemsetAsync(h->buf<double>(B_LINV), 0, h->L.size[B_LINV], s), "memset Linv");
    VIF_CUDA(h, launch_chol_inv(h->buf<double>(B_KM), P.m, P.m, 0.0, h->buf<double>(B_LINV), P.mk, P.mk, 1,
                                h->buf<double>(B_TSCR), &st->km_fail, h->num_sms, s),
             "chol K_m");
    nl += 2;
  }
  h->mark(S_KM, 1);
  if (P.world == 1 && P.rounds > 1 && !h->comm) {
    // single GPU, R rounds on three streams:
    //   s_k1: K1(0) K1(1) ... K1(R-1)                       (after K0)
    //   s   : [K1(r)] vecchia(r) for r = 0..R-1              (round r conditions on rounds <= r)
    //   s_sy: [vecchia(r)] SYRK partials of round r          (into their own slice of GPART)
    //   s   : [all SYRK] fixed-order reduction of the R x nsplit partials, sum log D
    // The K1 scratch of round r is the W rows of round r (row stride ld), so it never overlaps the W
    // rows that earlier rounds' vecchia launches are writing.
    const size_t part_round = syrk_part_doubles(P.ld, P.nsplit_round);
    VIF_CUDA(h, cudaEventRecord(h->ev_k0, s), "event");
    VIF_CUDA(h, cudaStreamWaitEvent(h->s_k1, h->ev_k0, 0), "event wait");
    VIF_CUDA(h, cudaStreamWaitEvent(h->s_sy, h->ev_k0, 0), "event wait");
    h->mark(S_UFEAT, 0);
    for (int64_t r = 0; r < P.rounds; ++r) {
      const int64_t cnt = std::min<int64_t>(P.chunk, P.n - r * P.chunk);
      if (cnt > 0) {
        VIF_CUDA(h, launch_u_features(h->buf<double>(B_X), h->buf<double>(B_Z), h->buf<double>(B_Y), P.n,
                                      r * P.chunk, cnt, P.chunk, 1, 0, P.m, P.mk, p, h->buf<double>(B_LINV),
                                      h->buf<double>(B_W), h->buf<double>(B_U), P.ld, h->s_k1, P.ld),
                 "U features");
        nl += P.mk > 0 ? 2 : 1;
      }
      VIF_CUDA(h, cudaEventRecord(h->ev_k1[r], h->s_k1), "event");
    }
    h->mark(S_UFEAT, 1);
    h->mark(S_VECCHIA, 0);
    double* G = h->buf<double>(B_G);
    for (int64_t r = 0; r < P.rounds; ++r) {
      const int64_t off = r * P.chunk;
      const int64_t cnt = std::min<int64_t>(P.chunk, P.n - off);
      VIF_CUDA(h, cudaStreamWaitEvent(s, h->ev_k1[r], 0), "event wait");
      if (cnt > 0) {
        VecchiaArgs a;
        a.U = h->buf<double>(B_U);
        a.ldu = P.ld;
        a.mk = P.mk;
        a.ld = P.ld;
        a.X = h->buf<double>(B_X);
        a.nbr = h->buf<int32_t>(B_NBR);
        a.mv = P.mv;
        a.order = h->ord(0) + off;
        a.npts = cnt;
        a.p = p;
        a.W = h->buf<double>(B_W) + (size_t)off * P.ld;
        a.ldw = P.ld;
        a.Dpos = h->buf<double>(B_DPOS) + off;
        a.B_out = B_out;
        a.D_out = D_out;
        a.st = st;
        a.state = h->grad_state ? h->grad_state + (size_t)off * grad_state_doubles(P.mv) : nullptr;
        VIF_CUDA(h, launch_vecchia(a, s), "vecchia");
        ++nl;
      }
      VIF_CUDA(h, cudaEventRecord(h->ev_v[r], s), "event");
      VIF_CUDA(h, cudaStreamWaitEvent(h->s_sy, h->ev_v[r], 0), "event wait");
      if (cnt > 0) {
        VIF_CUDA(h, launch_syrk_part(h->buf<double>(B_W) + (size_t)off * P.ld, P.ld, cnt, P.ld, P.nsplit_round,
                                     h->buf<double>(B_GPART) + (size_t)r * part_round, h->s_sy),
                 "syrk");
        ++nl;
      } else {
        VIF_CUDA(h, cudaMemsetAsync(h->buf<double>(B_GPART) + (size_t)r * part_round, 0, part_round * 8, h->s_sy),
                 "memset");
      }
    }
    h->mark(S_VECCHIA, 1);
    VIF_CUDA(h, cudaEventRecord(h->ev_sy, h->s_sy), "event");
    VIF_CUDA(h, cudaStreamWaitEvent(s, h->ev_sy, 0), "event wait");
    h->mark(S_SYRK, 0);
    VIF_CUDA(h, launch_syrk_reduce(h->buf<double>(B_GPART), P.ld, P.nsplit_round, (int)P.rounds, G, P.ld, s),
             "syrk reduce");
    h->mark(S_SYRK, 1);
    h->mark(S_REDUCE, 0);
    VIF_CUDA(h, launch_logd_sum(h->buf<double>(B_DPOS), P.n, h->buf<double>(B_PART), kLogdParts,
                                G + (size_t)P.ld * P.ld, s),
             "logd");
    h->mark(S_REDUCE, 1);
    nl += 3;
    h->factored = true;
    h->finished = false;
    h->launches = nl;
    return mark_inputs_used(h);
  }
  // A1-A6 in chunk-cyclic rounds.  Round r of a rank = positions [r*chunk, (r+1)*chunk);
  // vif_set_data groups the processing order by round (Morton order inside a round).  Per rank:
  //   compute stream: K1(round 0..R-1), then for each r: [wait AG(r)] vecchia rows of round r
  //   comm stream:    AG(r) right after K1(r)
  // so the all-gather of round r overlaps K1 of later rounds and the vecchia rows of earlier rounds
  // (the rows of round r only condition on predecessors, i.e. on rounds <= r).
  const int nrep = P.emulate ? P.world : 1;
  const bool nccl_path = h->comm != nullptr;
  const size_t gstride = (size_t)P.ld * P.ld + 8;
  h->mark(S_UFEAT, 0);
  for (int64_t r = 0; r < P.rounds; ++r) {
    for (int g = 0; g < nrep; ++g) {
      const int rank = P.emulate ? g : P.rank;
      if (P.k1_i8) {
        VIF_CUDA(h, launch_u_features_i8(h->buf<double>(B_X), h->buf<double>(B_Z), h->buf<double>(B_Y), P.n,
                                         r * P.chunk, P.chunk, P.chunk, P.world, rank, P.m, P.mk, p,
                                         h->buf<double>(B_LINV), h->buf<double>(B_U), P.ld, h->buf<int8_t>(B_WS),
                                         P.oz_cap, h->buf<char>(B_OZK1), kPlanSMs, s),
                 "U features (int8 slices)");
        nl += 1 + 2 * (int)((P.chunk + P.oz_cap - 1) / P.oz_cap);
      } else {
        VIF_CUDA(h, launch_u_features(h->buf<double>(B_X), h->buf<double>(B_Z), h->buf<double>(B_Y), P.n,
                                      r * P.chunk, P.chunk, P.chunk, P.world, rank, P.m, P.mk, p,
                                      h->buf<double>(B_LINV), h->buf<double>(B_W), h->buf<double>(B_U), P.ld, s),
                 "U features");
        nl += P.mk > 0 ? 2 : 1;
      }
    }
    if (nccl_path) {
      Nccl& N = nccl();
      const size_t cnt = (size_t)P.chunk * P.ld;
      double* recv = h->buf<double>(B_U) + (size_t)r * P.world * cnt;
      VIF_CUDA(h, cudaEventRecord(h->ev_k1[r], s), "event");
      VIF_CUDA(h, cudaStreamWaitEvent(h->cstream, h->ev_k1[r], 0), "event wait");
      ncclResult_t rr = N.AllGather(recv + (size_t)P.rank * cnt, recv, cnt, ncclFloat64, h->comm, h->cstream);
      if (rr != ncclSuccess) return fail(h, VIF_ERR_NCCL, std::string("ncclAllGather: ") + N.GetErrorString(rr));
      VIF_CUDA(h, cudaEventRecord(h->ev_ag[r], h->cstream), "event");
    }
  }
  h->mark(S_UFEAT, 1);
  h->mark(S_GATHER, 0);  // the gathers run on the comm stream, overlapped with the stages below
  h->mark(S_GATHER, 1);
  for (int g = 0; g < nrep; ++g) {
    const int rank = P.emulate ? g : P.rank;
    const int64_t npts = P.n_own[rank];
    double* Wg = h->buf<double>(B_W) + (size_t)g * P.npos * P.ld;
    double* Dg = h->buf<double>(B_DPOS) + (size_t)g * P.npos;
    // K4's column maxima come with the W rows (one handle, one W): no separate pass over W
    unsigned long long* c64 = nullptr;
    if (P.syrk_i8 && nrep == 1) {
      c64 = reinterpret_cast<unsigned long long*>(h->buf<char>(B_OZAUX) + (syrk_i8_aux_bytes(P.ld) + 255) / 256 * 256);
      VIF_CUDA(h, cudaMemsetAsync(c64, 0, (size_t)64 * P.ld * sizeof(unsigned long long), s), "memset cmax");
    }
    h->mark(S_VECCHIA, 0);
    int64_t off = 0;
    for (int64_t r = 0; r < P.rounds; ++r) {
      const int64_t start = (r * P.world + rank) * P.chunk;
      const int64_t cnt = P.n - start <= 0 ? 0 : (P.n - start < P.chunk ? P.n - start : P.chunk);
      if (nccl_path) VIF_CUDA(h, cudaStreamWaitEvent(s, h->ev_ag[r], 0), "event wait");
      if (cnt > 0) {
        VecchiaArgs a;
        a.U = h->buf<double>(B_U);
        a.ldu = P.ld;
        a.mk = P.mk;
        a.ld = P.ld;
        a.X = h->buf<double>(B_X);
        a.nbr = h->buf<int32_t>(B_NBR);
        a.mv = P.mv;
        a.order = h->ord(g) + off;
        a.npts = cnt;
        a.p = p;
        a.W = Wg + (size_t)off * P.ld;
        a.ldw = P.ld;
        a.Dpos = Dg + off;
        a.B_out = B_out;
        a.D_out = D_out;
        a.st = st;
        a.state = h->grad_state ? h->grad_state + (size_t)off * grad_state_doubles(P.mv) : nullptr;
        a.cmax = c64;
        VIF_CUDA(h, launch_vecchia(a, s), "vecchia");
        ++nl;
      }
      off += cnt;
    }
    h->mark(S_VECCHIA, 1);
    double* G = h->buf<double>(B_G) + g * gstride;
    h->mark(S_SYRK, 0);
    if (P.syrk_i8)
      VIF_CUDA(h, launch_syrk_i8(Wg, P.ld, npts, P.ld, h->buf<int8_t>(B_WS), P.oz_cap, h->buf<double>(B_GPART),
                                 h->buf<char>(B_OZAUX), G, P.ld, kPlanSMs, s, c64),
               "syrk (int8 slices)");
    else
      VIF_CUDA(h, launch_syrk(Wg, P.ld, npts, P.ld, P.nsplit, h->buf<double>(B_GPART), G, P.ld, s), "syrk");
    h->mark(S_SYRK, 1);
    h->mark(S_REDUCE, 0);
    VIF_CUDA(h, launch_logd_sum(Dg, npts, h->buf<double>(B_PART), kLogdParts,
                                G + (size_t)P.ld * P.ld, s),
             "logd");
    // DMMA: syrk part + reduce; int8 slices: colmax + per chunk (slice, tcgen05 syrk, reduce); + logd (2)
    nl += P.syrk_i8 ? 3 + 3 * (int)((std::max<int64_t>(npts, 1) + P.oz_cap - 1) / P.oz_cap) : 4;
  }
  // A7
  if (P.emulate) {
    VIF_CUDA(h, launch_sum_buffers(h->buf<double>(B_G), (int64_t)gstride, P.world, (int64_t)gstride,
                                   h->buf<double>(B_GSUM), s),
             "emulated all-reduce");
    ++nl;
  } else if (h->comm) {
    Nccl& N = nccl();
    double* G = h->buf<double>(B_G);
    // the Gram + sum log D, and the failure state: a NOT_PD row is found on the rank that owns it, so
    // the minimum failing row is reduced too -- every rank then returns the same status from vif_nll
    // (and vif_grad never has ranks entering its own all-reduce while another has returned)
    DevStatus* st_dev = h->buf<DevStatus>(B_STATUS);
    ncclResult_t rr = N.GroupStart();
    if (rr == ncclSuccess) rr = N.AllReduce(G, G, (size_t)P.ld * P.ld + 1, ncclFloat64, ncclSum, h->comm, s);
    if (rr == ncclSuccess)
      rr = N.AllReduce(&st_dev->bad_row, &st_dev->bad_row, 1, ncclUint64, ncclMin, h->comm, s);
    {
      const ncclResult_t r2 = N.GroupEnd();
      if (rr == ncclSuccess) rr = r2;
    }
    if (rr != ncclSuccess) return fail(h, VIF_ERR_NCCL, std::string("ncclAllReduce: ") + N.GetErrorString(rr));
  }
  h->mark(S_REDUCE, 1);
  h->factored = true;
  h->finished = false;
  h->launches = nl;
  return mark_inputs_used(h);
}

int vif_nll(void* handle, vif_terms* out) {
  Handle* h = reinterpret_cast<Handle*>(handle);
  if (!h) return fail(nullptr, VIF_ERR_INVALID_ARG, "handle is NULL");
  if (!out) return fail(h, VIF_ERR_INVALID_ARG, "out is NULL");
  if (!h->factored) return fail(h, VIF_ERR_STATE, "vif_nll before vif_factor");
  if (h->finished) {
    *out = h->cached;
    return h->cached_status;
  }
  const Plan& P = h->P;
  cudaStream_t s = h->stream;
  DevStatus* st = h->buf<DevStatus>(B_STATUS);
  double* G = P.emulate ? h->buf<double>(B_GSUM) : h->buf<double>(B_G);
  int64_t nl = 0;
  h->mark(S_CHOLM, 0);
  if (P.m > 0) {
    VIF_CUDA(h, cudaMemsetAsync(h->buf<double>(B_LINVM), 0, h->L.size[B_LINVM], s), "memset LinvM");
    VIF_CUDA(h, launch_chol_inv(G, P.m, P.ld, 1.0, h->buf<double>(B_LINVM), P.mk, P.mk, 0, nullptr, &st->m_fail,
                                h->num_sms, s),
             "chol M");
    ++nl;
  }
  h->mark(S_CHOLM, 1);
  double* terms = h->buf<double>(B_TERMS);
  h->mark(S_FINISH, 0);
  VIF_CUDA(h, launch_finish(G, P.ld, P.m, P.ycol, h->buf<double>(B_LINVM), P.mk, G + (size_t)P.ld * P.ld, P.n, terms, s),
           "finish");
  h->mark(S_FINISH, 1);
  ++nl;
  h->launches += nl;
  double ht[4];
  DevStatus hs;
  VIF_CUDA(h, cudaMemcpyAsync(ht, terms, sizeof(ht), cudaMemcpyDeviceToHost, s), "terms copy");
  VIF_CUDA(h, cudaMemcpyAsync(&hs, st, sizeof(hs), cudaMemcpyDeviceToHost, s), "status copy");
  VIF_WAIT(h, s);
  if (h->prof) {
    for (int k = 0; k < S_COUNT; ++k) {
      if (!h->ev_used[k]) continue;
      float ms = 0.f;
      if (cudaEventElapsedTime(&ms, h->ev[k][0], h->ev[k][1]) == cudaSuccess) h->stage_ms[k] += ms;
    }
    ++h->prof_evals;
  }
  vif_terms t;
  t.nll = ht[0];
  t.logdet_D = ht[1];
  t.logdet_M = ht[2];
  t.quad = ht[3];
  t.bad_row = -1;
  int status = VIF_OK;
  if (hs.km_fail) {
    status = fail(h, VIF_ERR_NOT_PD, "Cholesky of K(Z,Z) + jitter failed");
  } else if (hs.bad_row != ~0ULL) {
    t.bad_row = (int64_t)hs.bad_row;
    char msg[128];
    snprintf(msg, sizeof msg, "residual block of point %lld is not positive definite", (long long)hs.bad_row);
    status = fail(h, VIF_ERR_NOT_PD, msg);
  } else if (hs.m_fail) {
    status = fail(h, VIF_ERR_NOT_PD, "Cholesky of M failed");
  }
  h->finished = true;
  h->cached = t;
  h->cached_status = status;
  *out = t;
  return status;
}

int vif_grad_workspace_bytes(const vif_dims* dims, size_t* bytes) {
  Plan P;
  std::string err;
  if (!bytes) return fail(nullptr, VIF_ERR_INVALID_ARG, "bytes is NULL");
  if (!make_plan(dims, true, P, err)) return fail(nullptr, VIF_ERR_INVALID_ARG, err);
  *bytes = make_grad_layout(P).total;
  return VIF_OK;
}

int vif_grad(void* handle, const vif_theta* theta, void* gws, size_t gws_bytes, double* grad, vif_terms* terms) {
  Handle* h = reinterpret_cast<Handle*>(handle);
  if (!h) return fail(nullptr, VIF_ERR_INVALID_ARG, "handle is NULL");
  if (!grad) return fail(h, VIF_ERR_INVALID_ARG, "grad is NULL");
  const Plan& P = h->P;
  if (P.mv > 47) return fail(h, VIF_ERR_INVALID_ARG, "vif_grad: m_v <= 47 in this version");
  const Layout GL = make_grad_layout(P);
  if (!gws || gws_bytes < GL.total) {
    char msg[128];
    snprintf(msg, sizeof msg, "grad workspace too small: need %zu bytes", GL.total);
    return fail(h, VIF_ERR_NO_MEMORY, msg);
  }
  char* gb = reinterpret_cast<char*>(round_up((int64_t)(uintptr_t)gws, 256));
  auto gbuf = [&](GBuf b) { return reinterpret_cast<double*>(gb + GL.off[b]); };
  CovParams p;
  std::string err;
  if (!make_params(h, theta, p, err)) return fail(h, VIF_ERR_INVALID_ARG, err);
  // one (real) rank per process: the factor's vecchia rows write L, A_i, 1/L_jj, D_i of the
  // state (same rows, same arithmetic as the NLL) and only the g_i dots remain for the state pass;
  // VIF_GRAD_STATE=1 recomputes everything in the state pass instead
  static const char* gs_env = getenv("VIF_GRAD_STATE");
  const bool state_ff = P.mv <= 47 && !P.emulate && !(gs_env && gs_env[0] == '1');
  h->grad_state = state_ff ? gbuf(G_STATE) : nullptr;
  int r = vif_factor(handle, theta, nullptr, nullptr);
  h->grad_state = nullptr;
  if (r != VIF_OK) return r;
  cudaStream_t s = h->stream;
  const int m = P.m, mk = P.mk, ld = P.ld;
  double* G = h->buf<double>(P.emulate ? B_GSUM : B_G);  // the (all-)reduced Gram
  VIF_CUDA(h, cudaMemcpyAsync(gbuf(G_MCOPY), G, (size_t)ld * ld * 8, cudaMemcpyDeviceToDevice, s), "copy G");
  vif_terms t;
  r = vif_nll(handle, &t);
  if (terms) *terms = t;
  if (r != VIF_OK) return r;
  DevStatus* st = h->buf<DevStatus>(B_STATUS);
  // M_w^{-1} = L_M^{-T} L_M^{-1} (full inverse of the Cholesky factor), z, Q2 = 2 Q
  if (m > 0) {
    VIF_CUDA(h, cudaMemsetAsync(gbuf(G_LINVM), 0, GL.size[G_LINVM], s), "memset");
    VIF_CUDA(h, launch_chol_inv(gbuf(G_MCOPY), m, ld, 1.0, gbuf(G_LINVM), mk, mk, 1, gbuf(G_TSCR), &st->m_fail,
                                h->num_sms, s),
             "chol M (full inverse)");
  }
  VIF_CUDA(h, launch_grad_q(gbuf(G_LINVM), mk, G, ld, P.ycol, m, ld, gbuf(G_ZH), gbuf(G_Z), gbuf(G_Q2), s), "Q");
  // Per rank (every virtual rank of an emulated handle): Gamma = W (2Q) for its rows by processing position,
  // the per-point state, the adjoint rows and R, then one pass per parameter.
  const int nrep = P.emulate ? P.world : 1;
  const double* Linv = h->buf<double>(B_LINV);
  const double* U = h->buf<double>(B_U);
  const int nparam = P.d + 2;
  VIF_CUDA(h, cudaMemsetAsync(gbuf(G_DU), 0, GL.size[G_DU], s), "memset R");
  for (int g = 0; g < nrep; ++g) {
    const int rank = P.emulate ? g : P.rank;
    double* W = h->buf<double>(B_W) + (size_t)g * P.npos * ld;
    if (P.grad_i8)
      VIF_CUDA(h, launch_gemm_tn_i8(W, ld, P.npos, gbuf(G_Q2), ld, ld, ld, 0, gbuf(G_GAM), ld, h->buf<int8_t>(B_WS),
                                    P.oz_cap, h->buf<char>(B_OZK1), kPlanSMs, s),
               "Gamma (int8 slices)");
    else
      VIF_CUDA(h, launch_gemm_tn(W, ld, P.npos, gbuf(G_Q2), ld, ld, ld, 0, gbuf(G_GAM), ld, 1.0, 0, s), "Gamma");
    GradPointArgs a;
    a.U = U;
    a.dU = nullptr;
    a.Gam = gbuf(G_GAM);
    a.ldu = ld;
    a.mk = mk;
    a.ld = ld;
    a.X = h->buf<double>(B_X);
    a.nbr = h->buf<int32_t>(B_NBR);
    a.mv = P.mv;
    a.order = h->ord(g);
    a.npts = P.n_own[rank];
    a.p = p;
    a.part = gbuf(G_PART);
    a.state = gbuf(G_STATE);
    a.rho = gbuf(G_RHO);
    a.sig = gbuf(G_SIG);
    a.adj = gbuf(G_ADJ);
    if (state_ff) VIF_CUDA(h, launch_grad_gam(a, s), "gradient state (dots)");
    else VIF_CUDA(h, launch_grad_state(a, s), "gradient state");
    VIF_CUDA(h, launch_grad_adjoint(a, s), "gradient adjoint");
    // no dU at all: the adjoint rows scattered to R (n x m), T = R L_m^{-1}, G2 = R^T U, and per kernel
    // parameter <T, dK(X,Z)> - <G2, Phi_low> (at n = 1M, m = 500 materialising dU per
    // parameter cost two n m^2 GEMMs each; the R path is ~100 ms once plus ~3 ms per parameter)
    if (mk > 0) {
      double* R = gbuf(G_DU);  // n x mk
      VIF_CUDA(h, launch_gchild(a.nbr, P.mv, a.order, a.npts, P.n, reinterpret_cast<int*>(gbuf(G_CCNT)),
                                reinterpret_cast<int*>(gbuf(G_CCUR)), reinterpret_cast<int*>(gbuf(G_CPTR)),
                                reinterpret_cast<int*>(gbuf(G_CENT)), s),
               "children lists");
      static const char* jo_env = getenv("VIF_GRAD_RORDER");  // R rows in the Morton order (1-2% faster); 0: index order
      const int64_t* jorder = (!(jo_env && jo_env[0] == '0') && P.world == 1) ? h->ord(0) : nullptr;
      VIF_CUDA(h, launch_gR(reinterpret_cast<int*>(gbuf(G_CPTR)), reinterpret_cast<int*>(gbuf(G_CENT)), a.order,
                            jorder, P.n, mk, P.mv, a.state, a.adj, a.rho, a.sig, R,
                            reinterpret_cast<unsigned long long*>(gbuf(G_TDK) + P.d + 1), s),
               "R");
      // R has reversed columns, so T = R L_m^{-1} is a triangular product (T with reversed columns)
      if (g == 0) VIF_CUDA(h, launch_grev_linv(Linv, mk, gbuf(G_LINVT), s), "reversed L_m^-1");
      if (P.grad_i8)
        VIF_CUDA(h, launch_gemm_tn_i8(R, mk, P.n, gbuf(G_LINVT), mk, mk, mk, 1, gbuf(G_T), mk, h->buf<int8_t>(B_WS),
                                      P.oz_cap, h->buf<char>(B_OZK1), kPlanSMs, s),
                 "T = R L^-1 (int8 slices)");
      else
        VIF_CUDA(h, launch_gemm_tn(R, mk, P.n, gbuf(G_LINVT), mk, mk, mk, 1, gbuf(G_T), mk, 1.0, 0, s), "T = R L^-1");
      if (P.grad_i8)
        VIF_CUDA(h, launch_gemm_tt_i8(R, mk, mk, U, ld, mk, P.n, gbuf(G_G2), mk, h->buf<int8_t>(B_WS), h->L.size[B_WS],
                                      gbuf(G_TSP), h->buf<char>(B_OZK1), kPlanSMs, s),
                 "G2 = R^T U (int8 slices)");
      else
        VIF_CUDA(h, launch_gemm_tt(R, mk, mk, U, ld, mk, P.n, gemm_tt_nsplit(mk, mk, P.n, kPlanSMs), gbuf(G_TSP),
                                   gbuf(G_G2), mk, s),
                 "G2 = R^T U");
      VIF_CUDA(h, launch_gTdK(h->buf<double>(B_X), h->buf<double>(B_Z), P.n, m, mk, p, gbuf(G_T), gbuf(G_TDKP),
                              gbuf(G_TDK), s),
               "<T, dK>");
    }
    // the point terms of every parameter in one pass (bit-identical to one pass per parameter)
    a.dU = nullptr;
    VIF_CUDA(h, launch_grad_points_adj_all(a, gbuf(G_OUT) + (size_t)g * nparam, s), "gradient points");
    for (int pi = 0; pi < nparam; ++pi) {
      const bool kernel_param = pi <= P.d;
      if (kernel_param && m > 0) {
        VIF_CUDA(h, launch_dkm(h->buf<double>(B_Z), m, mk, pi, p, gbuf(G_DKM), s), "dK_m");
        VIF_CUDA(h, launch_gemm_tn(Linv, mk, mk, gbuf(G_DKM), mk, mk, mk, 0, gbuf(G_TT), mk, 1.0, 0, s), "Linv dK_m");
        VIF_CUDA(h, launch_gemm_tn(Linv, mk, mk, gbuf(G_TT), mk, mk, mk, 0, gbuf(G_PHI), mk, 1.0, 0, s), "Phi");
        VIF_CUDA(h, launch_phi_low(gbuf(G_PHI), mk, gbuf(G_PHILOW), s), "Phi_low");
      }
      if (kernel_param && m > 0)
        VIF_CUDA(h, launch_gfinal(gbuf(G_OUT) + (size_t)g * nparam + pi, gbuf(G_TDK), pi, gbuf(G_G2), gbuf(G_PHILOW),
                                  mk, s),
                 "<T, dK> - <G2, Phi_low>");
    }
  }
  if (nrep > 1) {
    VIF_CUDA(h, launch_sum_buffers(gbuf(G_OUT), nparam, nrep, nparam, gbuf(G_OUT), s), "emulated all-reduce");
  } else if (h->comm) {
    Nccl& N = nccl();
    ncclResult_t rr = N.AllReduce(gbuf(G_OUT), gbuf(G_OUT), (size_t)nparam, ncclFloat64, ncclSum, h->comm, s);
    if (rr != ncclSuccess) return fail(h, VIF_ERR_NCCL, std::string("ncclAllReduce: ") + N.GetErrorString(rr));
  }
  {
    int r2 = mark_inputs_used(h);
    if (r2 != VIF_OK) return r2;
  }
  VIF_CUDA(h, cudaMemcpyAsync(grad, gbuf(G_OUT), (size_t)(P.d + 2) * 8, cudaMemcpyDeviceToHost, s), "grad copy");
  VIF_WAIT(h, s);
  for (int pi = 0; pi < P.d + 2; ++pi)
    if (!isfinite(grad[pi])) return fail(h, VIF_ERR_NOT_PD, "gradient: a residual block or M is not positive definite");
  return VIF_OK;
}

int vif_predict_workspace_bytes(const vif_dims* dims, int64_t np, size_t* bytes) {
  Plan P;
  std::string err;
  if (!bytes) return fail(nullptr, VIF_ERR_INVALID_ARG, "bytes is NULL");
  if (np < 1) return fail(nullptr, VIF_ERR_INVALID_ARG, "np must be >= 1");
  if (!make_plan(dims, true, P, err)) return fail(nullptr, VIF_ERR_INVALID_ARG, err);
  *bytes = make_pred_layout(P, np).total;
  return VIF_OK;
}

int vif_predict(void* handle, const vif_theta* theta, int64_t np, const double* Xp, const int32_t* nbrp, void* ws,
                size_t ws_bytes, double* mu, double* var, double* Dp, double* Bp) {
  Handle* h = reinterpret_cast<Handle*>(handle);
  if (!h) return fail(nullptr, VIF_ERR_INVALID_ARG, "handle is NULL");
  const Plan& P = h->P;
  if (np < 1 || !Xp || !mu || (P.mv > 0 && !nbrp)) return fail(h, VIF_ERR_INVALID_ARG, "vif_predict: bad arguments");
  const Layout PL = make_pred_layout(P, np);
  if (!ws || ws_bytes < PL.total) {
    char msg[128];
    snprintf(msg, sizeof msg, "prediction workspace too small: need %zu bytes", PL.total);
    return fail(h, VIF_ERR_NO_MEMORY, msg);
  }
  char* pb = reinterpret_cast<char*>(round_up((int64_t)(uintptr_t)ws, 256));
  auto pbuf = [&](PBuf b) { return reinterpret_cast<double*>(pb + PL.off[b]); };
  CovParams p;
  std::string err;
  if (!make_params(h, theta, p, err)) return fail(h, VIF_ERR_INVALID_ARG, err);
  cudaStream_t s = h->stream;
  // ranks (NCCL) predict contiguous slices of the prediction points and write only their slice of the
  // outputs; an emulated multi-rank handle (one process) predicts all of them
  const double* Xp0 = Xp;
  {
    const int64_t per = P.emulate ? np : (np + P.world - 1) / P.world;
    const int64_t lo = P.emulate ? 0 : std::min<int64_t>(np, P.rank * per);
    const int64_t hi = std::min<int64_t>(np, lo + per);
    Xp += lo * P.d;
    if (nbrp) nbrp += lo * P.mv;
    mu += lo;
    if (var) var += lo;
    if (Dp) Dp += lo;
    if (Bp) Bp += lo * P.mv;
    np = hi - lo;
  }
  if (np > 0) {
    VIF_CUDA(h, cudaMemcpyAsync(pbuf(P_X), Xp, (size_t)np * P.d * 8, cudaMemcpyDefault, s), "copy Xp");
    if (P.mv > 0)
      VIF_CUDA(h, cudaMemcpyAsync(pbuf(P_NBR), nbrp, (size_t)np * P.mv * 4, cudaMemcpyDefault, s), "copy nbrp");
    // the prediction rows are gathered unchecked by the vecchia kernel: validate them first
    DevStatus* st0 = h->buf<DevStatus>(B_STATUS);
    VIF_CUDA(h, launch_reset_status(st0, s), "reset status");
    VIF_CUDA(h, launch_validate_pred(pbuf(P_X), np, P.d, reinterpret_cast<const int32_t*>(pbuf(P_NBR)),
                                     P.mv > 0 ? P.mv : 0, P.n, st0, s),
             "validate prediction inputs");
    DevStatus hs0;
    VIF_CUDA(h, cudaMemcpyAsync(&hs0, st0, sizeof(hs0), cudaMemcpyDeviceToHost, s), "status copy");
    VIF_WAIT(h, s);
    if (hs0.bad_input != ~0ULL) {
      char msg[192];
      snprintf(msg, sizeof msg,
               "invalid prediction input at row %llu (non-finite Xp, or a neighbour outside [0, n), repeated, or "
               "-1 before a valid entry)",
               hs0.bad_input + (unsigned long long)(Xp - Xp0) / (unsigned long long)P.d);
      return fail(h, VIF_ERR_INVALID_ARG, msg);
    }
  }
  int r = vif_factor(handle, theta, nullptr, nullptr);
  if (r != VIF_OK) return r;
  const int m = P.m, mk = P.mk, ld = P.ld;
  double* G = h->buf<double>(P.emulate ? B_GSUM : B_G);  // the (all-)reduced Gram
  VIF_CUDA(h, cudaMemcpyAsync(pbuf(P_MCOPY), G, (size_t)ld * ld * 8, cudaMemcpyDeviceToDevice, s), "copy G");
  vif_terms t;
  r = vif_nll(handle, &t);
  if (r != VIF_OK) return r;
  if (np == 0) return VIF_OK;
  DevStatus* st = h->buf<DevStatus>(B_STATUS);
  // z = M_w^{-1} G_Wr
  if (m > 0) {
    VIF_CUDA(h, cudaMemsetAsync(pbuf(P_LINVM), 0, PL.size[P_LINVM], s), "memset");
    VIF_CUDA(h, launch_chol_inv(pbuf(P_MCOPY), m, ld, 1.0, pbuf(P_LINVM), mk, mk, 1, pbuf(P_TSCR), &st->m_fail,
                                h->num_sms, s),
             "chol M (full inverse)");
    VIF_CUDA(h, launch_zvec(pbuf(P_LINVM), mk, G, ld, P.ycol, m, pbuf(P_ZH), pbuf(P_Z), s), "z");
  }
  // prediction features u_p (y column 0), Morton processing order of the prediction points
  VIF_CUDA(h, cudaMemsetAsync(pbuf(P_Y), 0, PL.size[P_Y], s), "memset y_p");
  VIF_CUDA(h, launch_u_features(pbuf(P_X), h->buf<double>(B_Z), pbuf(P_Y), np, 0, np, np, 1, 0, m, mk, p,
                                h->buf<double>(B_LINV), pbuf(P_S), pbuf(P_U), ld, s),
           "prediction features");
  int64_t* order = nullptr;
  VIF_CUDA(h, launch_order(pbuf(P_X), np, P.d, np, np, 1, 0, pbuf(P_BBOX), reinterpret_cast<uint64_t*>(pbuf(P_KEYS)),
                           reinterpret_cast<uint64_t*>(pbuf(P_KEYS2)), reinterpret_cast<int64_t*>(pbuf(P_VALS)),
                           reinterpret_cast<int64_t*>(pbuf(P_VALS2)), pbuf(P_TEMP), PL.size[P_TEMP], &order, s),
           "prediction order");
  VIF_CUDA(h, launch_reset_status(st, s), "reset status");
  VecchiaArgs a;
  a.U = h->buf<double>(B_U);
  a.ldu = ld;
  a.mk = mk;
  a.ld = ld;
  a.X = h->buf<double>(B_X);
  a.nbr = reinterpret_cast<const int32_t*>(pbuf(P_NBR));
  a.mv = P.mv;
  a.order = order;
  a.npts = np;
  a.p = p;
  a.W = pbuf(P_W);
  a.ldw = ld;
  a.Dpos = pbuf(P_DPOS);
  a.B_out = Bp;
  a.D_out = Dp;
  a.st = st;
  a.Uself = pbuf(P_U);
  a.Xself = pbuf(P_X);
  VIF_CUDA(h, launch_vecchia(a, s), "prediction rows");
  // T = E L_M^{-T} (rows e_p / sqrt(D_p) = the prediction W rows), so e_p M_w^{-1} e_p = D_p |T_p|^2
  if (var && m > 0)
    VIF_CUDA(h, launch_gemm_tn(pbuf(P_W), ld, np, pbuf(P_LINVM), mk, mk, mk, 1, pbuf(P_S), mk, 1.0, 0, s),
             "W L_M^-T");
  VIF_CUDA(h, launch_pred_mean(pbuf(P_W), ld, m, P.ycol, pbuf(P_Z), pbuf(P_DPOS), order, np, mu,
                               var && m > 0 ? pbuf(P_S) : nullptr, mk, var, s),
           "mean / variance");
  {
    int r2 = mark_inputs_used(h);
    if (r2 != VIF_OK) return r2;
  }
  DevStatus hs;
  VIF_CUDA(h, cudaMemcpyAsync(&hs, st, sizeof(hs), cudaMemcpyDeviceToHost, s), "status copy");
  VIF_WAIT(h, s);
  if (hs.bad_row != ~0ULL) {
    char msg[128];
    snprintf(msg, sizeof msg, "residual block of prediction point %llu is not positive definite", hs.bad_row);
    return fail(h, VIF_ERR_NOT_PD, msg);
  }
  return VIF_OK;
}

int vif_neighbors(void* handle, const vif_theta* theta, int32_t mv, int32_t* nbr_out) {
  Handle* h = reinterpret_cast<Handle*>(handle);
  if (!h) return fail(nullptr, VIF_ERR_INVALID_ARG, "handle is NULL");
  const Plan& P = h->P;
  if (!nbr_out || mv < 1 || mv > VIF_MAX_MV) return fail(h, VIF_ERR_INVALID_ARG, "vif_neighbors: bad arguments");
  if (!h->have_data) return fail(h, VIF_ERR_STATE, "no data");
  CovParams p;
  std::string err;
  if (!make_params(h, theta, p, err)) return fail(h, VIF_ERR_INVALID_ARG, err);
  cudaStream_t s = h->stream;
  ++h->fgen;  // reuses the factor's buffers: a prepared Laplace workspace is stale afterwards
  {
    int r = apply_pending(h);
    if (r != VIF_OK) return r;
  }
  DevStatus* st = h->buf<DevStatus>(B_STATUS);
  h->factored = h->finished = false;
  VIF_CUDA(h, launch_reset_status(st, s), "reset status");
  // u_i for all points (K0 + K1 of the factor, single round)
  if (P.m > 0) {
    VIF_CUDA(h, launch_build_km(h->buf<double>(B_Z), P.m, p, h->buf<double>(B_KM), s), "build K_m");
    VIF_CUDA(h, cudaMemsetAsync(h->buf<double>(B_LINV), 0, h->L.size[B_LINV], s), "memset Linv");
    VIF_CUDA(h, launch_chol_inv(h->buf<double>(B_KM), P.m, P.m, 0.0, h->buf<double>(B_LINV), P.mk, P.mk, 1,
                                h->buf<double>(B_TSCR), &st->km_fail, h->num_sms, s),
             "chol K_m");
    // every rank needs u_i of all n points: in row blocks through the W buffer (npos x ld per rank)
    static const char* cap_env = getenv("VIF_KNN_UROWS");  // test hook: smaller row blocks
    int64_t cap = (int64_t)(h->L.size[B_W] / sizeof(double)) / P.mk;
    if (cap_env && atoll(cap_env) > 0 && atoll(cap_env) < cap) cap = atoll(cap_env);
    for (int64_t r0 = 0; r0 < P.n; r0 += cap) {
      const int64_t rows = std::min<int64_t>(cap, P.n - r0);
      VIF_CUDA(h, launch_u_features(h->buf<double>(B_X), h->buf<double>(B_Z), h->buf<double>(B_Y), P.n, r0, rows, P.n, 1,
                                    0, P.m, P.mk, p, h->buf<double>(B_LINV), h->buf<double>(B_W) - r0 * P.mk,
                                    h->buf<double>(B_U), P.ld, s),
               "U features");
    }
  }
  // residual variances (n doubles) and degeneracy flags (n ints) in the dead W buffer; ranks (NCCL) search
  // the query blocks kb = rank, rank + world, ... (64 points each) and write only those rows
  double* isd = h->buf<double>(P.m > 0 ? B_W : B_U);  // (m = 0: U is unused; W could be only 8 n bytes)
  int* deg = reinterpret_cast<int*>(isd + P.n);
  const bool nccl_ranks = P.world > 1 && !P.emulate;
  int qoff = nccl_ranks ? P.rank : 0, qstride = nccl_ranks ? P.world : 1;
  static const char* shard_env = getenv("VIF_KNN_SHARD");  // test hook "g,G": search rank g's blocks of G
  if (shard_env) {
    int g = 0, G = 1;
    if (sscanf(shard_env, "%d,%d", &g, &G) == 2 && G >= 1 && g >= 0 && g < G) {
      qoff = g;
      qstride = G;
    }
  }
  // the Gram blocks on the integer tensor cores when the slice workspace holds all n rows (reading c18);
  // VIF_KNN_FP64=1: the DMMA kernel
  static const char* kf_env = getenv("VIF_KNN_FP64");
  // the slices go to the digit-slice workspace when it holds n rows (n <= 2^20), else behind isd, deg and erow in
  // the dead W buffer (n x ld doubles: 7 slices of KP bytes fit for m >= 32)
  const size_t wmeta = ((size_t)P.n * (sizeof(double) + 2 * sizeof(int)) + 1023) / 1024 * 1024;
  int8_t* kslices = nullptr;
  static const char* kw_env = getenv("VIF_KNN_WSLICES");  // test hook: the W-buffer placement at any n
  if (h->L.size[B_WS] >= knn_i8_ws_bytes(P.mk, P.n) && !(kw_env && kw_env[0] == '1'))
    kslices = h->buf<int8_t>(B_WS);
  else if (P.m > 0 && h->L.size[B_W] >= wmeta + knn_i8_ws_bytes(P.mk, P.n))
    kslices = reinterpret_cast<int8_t*>(h->buf<char>(B_W) + wmeta);
  const bool knn_i8 = P.m > 0 && !(kf_env && kf_env[0] == '1') && knn_i8_supported(mv, P.n) && kslices &&
                      h->L.size[B_W] >= wmeta;
  if (knn_i8) {
    int* erow = deg + P.n;  // row exponents of the digit slices, after isd and deg in the dead W buffer
    VIF_CUDA(h, launch_knn_resvar(h->buf<double>(B_U), P.ld, P.m, P.n, p, isd, deg, s), "residual variances");
    VIF_CUDA(h, launch_knn_i8(h->buf<double>(B_U), P.ld, P.mk, h->buf<double>(B_X), P.n, p, isd, deg, mv, nbr_out,
                              kslices, erow, h->num_sms, s, qoff, qstride),
             "neighbour search (int8 slices)");
  } else {
    VIF_CUDA(h, launch_knn(h->buf<double>(B_U), P.ld, P.m, P.mk, h->buf<double>(B_X), P.n, p, isd, deg, mv, nbr_out,
                           s, qoff, qstride),
             "neighbour search");
  }
  {
    int r = mark_inputs_used(h);
    if (r != VIF_OK) return r;
  }
  DevStatus hs;
  VIF_CUDA(h, cudaMemcpyAsync(&hs, st, sizeof(hs), cudaMemcpyDeviceToHost, s), "status copy");
  VIF_WAIT(h, s);
  if (hs.km_fail) return fail(h, VIF_ERR_NOT_PD, "Cholesky of K(Z,Z) + jitter failed");
  return VIF_OK;
}

// ---------------------------------------------------------------- VIF-Laplace
int vif_la_workspace_bytes(const vif_dims* dims, int32_t nprobe, int32_t max_cg, size_t* bytes) {
  Plan P;
  std::string err;
  if (!bytes) return fail(nullptr, VIF_ERR_INVALID_ARG, "bytes is NULL");
  if (nprobe < 0 || nprobe > kLaCols) return fail(nullptr, VIF_ERR_INVALID_ARG, "nprobe must be in [0, 64]");
  if (max_cg < 1) return fail(nullptr, VIF_ERR_INVALID_ARG, "max_cg must be >= 1");
  if (!make_plan(dims, true, P, err)) return fail(nullptr, VIF_ERR_INVALID_ARG, err);
  *bytes = make_la_layout(P, nprobe, max_cg).total;
  return VIF_OK;
}

int vif_la_prepare(void* handle, const vif_theta* theta, int32_t nprobe, int32_t max_cg, void* ws, size_t ws_bytes) {
  Handle* h = reinterpret_cast<Handle*>(handle);
  if (!h) return fail(nullptr, VIF_ERR_INVALID_ARG, "handle is NULL");
  const Plan& P = h->P;
  if (P.world != 1) return fail(h, VIF_ERR_INVALID_ARG, "vif_la_prepare: single-rank handles only in this version");
  if (nprobe < 0 || nprobe > kLaCols) return fail(h, VIF_ERR_INVALID_ARG, "nprobe must be in [0, 64]");
  if (max_cg < 1) return fail(h, VIF_ERR_INVALID_ARG, "max_cg must be >= 1");
  if (!theta) return fail(h, VIF_ERR_INVALID_ARG, "theta is NULL");
  const LaLayout LL = make_la_layout(P, nprobe, max_cg);
  if (!ws || ws_bytes < LL.total) {
    char msg[128];
    snprintf(msg, sizeof msg, "Laplace workspace too small: need %zu bytes", LL.total);
    return fail(h, VIF_ERR_NO_MEMORY, msg);
  }
  h->la_gen = ~0ull;
  h->la_nprobe = nprobe;
  h->la_maxcg = max_cg;
  h->la_sigma2 = theta->sigma2;
  LaCtx c = la_ctx(h, ws);
  // the latent process has no error variance: the VIF factor at nugget 0
  vif_theta th0 = *theta;
  th0.nugget = 0.0;
  int r = vif_factor(handle, &th0, P.mv > 0 ? c.d(L_B) : nullptr, c.d(L_D));
  if (r != VIF_OK) return r;
  cudaStream_t s = h->stream;
  // M_w = I + W_U^T W_U of the latent factor: the full L_M^{-1} for the quadratic term b^T Sigma_dagger^{-1} b
  VIF_CUDA(h, cudaMemcpyAsync(c.d(L_GM), h->buf<double>(B_G), c.L.size[L_GM], cudaMemcpyDeviceToDevice, s), "copy G");
  vif_terms t;
  r = vif_nll(handle, &t);
  if (r != VIF_OK) return r;
  VIF_CUDA(h, cudaMemsetAsync(c.base + c.L.off[L_TICKET], 0, c.L.size[L_TICKET], s), "memset ticket");
  if (P.m > 0) {
    VIF_CUDA(h, cudaMemsetAsync(c.d(L_LMINV), 0, c.L.size[L_LMINV], s), "memset");
    VIF_CUDA(h, launch_chol_inv(c.d(L_GM), P.m, P.ld, 1.0, c.d(L_LMINV), P.mk, P.mk, 1, c.d(L_TSCR), c.fitc_fail(),
                                h->num_sms, s),
             "chol M (full inverse)");
    VIF_CUDA(h, launch_la_transpose(c.d(L_LMINV), P.mk, P.mk, P.mk, c.d(L_LMINVT), P.mk, s), "L_M^-T");
  }
  VIF_CUDA(h, launch_la_invorder(h->ord(0), P.n, c.i(L_IPOS), s), "inverse order");
  if (P.mk > 0) VIF_CUDA(h, launch_la_rownorm2(c.U(), P.ld, P.mk, P.n, c.d(L_UN2), s), "||u_i||^2");
  else VIF_CUDA(h, cudaMemsetAsync(c.d(L_UN2), 0, c.L.size[L_UN2], s), "memset");
  VIF_CUDA(h, launch_la_transpose_struct(c.nbr(), P.n, P.mv, c.i(L_CNT), c.i(L_CUR), c.i(L_TPTR), c.i(L_TPOS), s),
           "B^T structure");
  {
    int nnz = 0;
    VIF_CUDA(h, cudaMemcpyAsync(&nnz, c.i(L_TPTR) + P.n, sizeof(int), cudaMemcpyDeviceToHost, s), "nnz");
    VIF_WAIT(h, s);
    VIF_CUDA(h, launch_la_tvals(c.i(L_TPOS), nnz, P.mv > 0 ? P.mv : 1, c.d(L_B), c.i(L_TROW), c.d(L_TVAL), s),
             "B^T values");
  }
  // dependency levels of B (forward) and B^T (backward), rows bucketed by level
  VIF_CUDA(h, cudaMemsetAsync(c.i(L_FLAGS), 0, c.L.size[L_FLAGS], s), "memset flags");
  {
    int* nlev = c.i(L_ACTIVE);  // scratch: two ints
    VIF_CUDA(h, launch_la_levels(c.nbr(), P.mv, P.n, c.i(L_TPTR), c.i(L_TROW), c.i(L_LEVF), c.i(L_LEVB), c.i(L_FLAGS),
                                 1, 2, nlev, s),
             "levels");
    int hl[2];
    VIF_CUDA(h, cudaMemcpyAsync(hl, nlev, sizeof(hl), cudaMemcpyDeviceToHost, s), "levels");
    VIF_WAIT(h, s);
    h->la_nlev_f = hl[0] + 1;
    h->la_nlev_b = hl[1] + 1;
    VIF_CUDA(h, launch_la_bucket(c.i(L_LEVF), P.n, h->la_nlev_f, c.i(L_CNT), c.i(L_CUR), c.i(L_LPTRF), c.i(L_ORDF), s),
             "bucket");
    VIF_CUDA(h, launch_la_bucket(c.i(L_LEVB), P.n, h->la_nlev_b, c.i(L_CNT), c.i(L_CUR), c.i(L_LPTRB), c.i(L_ORDB), s),
             "bucket");
    VIF_CUDA(h, launch_la_reorder(c.i(L_ORDF), c.nbr(), c.d(L_B), P.n, P.mv, c.i(L_ECF), c.d(L_EVF), c.i(L_ORDB),
                                  c.i(L_TPTR), c.i(L_TROW), c.d(L_TVAL), c.i(L_CNT), c.i(L_EPB), c.i(L_ECB), c.d(L_EVB),
                                  s),
             "level-ordered entries");
  }
  VIF_CUDA(h, cudaMemsetAsync(c.i(L_FLAGS), 0, c.L.size[L_FLAGS], s), "memset flags");  // solves start at epoch 1
  int ff = 0;
  VIF_CUDA(h, cudaMemcpyAsync(&ff, c.fitc_fail(), sizeof(int), cudaMemcpyDeviceToHost, s), "status");
  VIF_WAIT(h, s);
  if (ff) return fail(h, VIF_ERR_NOT_PD, "Cholesky of M (latent factor) failed");
  h->la_epoch = 0;
  h->la_ws = ws;
  h->la_gen = h->fgen;
  return VIF_OK;
}

static int la_check(Handle* h, void* ws) {
  if (h->la_gen != h->fgen || h->la_ws != ws)
    return fail(h, VIF_ERR_STATE, "Laplace workspace not prepared for the current factor (call vif_la_prepare)");
  return VIF_OK;
}

int vif_la_apply(void* handle, void* ws, int32_t op, int32_t ncol, const double* v, const double* winv, double* out) {
  Handle* h = reinterpret_cast<Handle*>(handle);
  if (!h) return fail(nullptr, VIF_ERR_INVALID_ARG, "handle is NULL");
  LA_TRY(la_check(h, ws));
  const Plan& P = h->P;
  if (ncol < 1 || ncol > (h->la_nprobe > 1 ? h->la_nprobe : 1) || !v || !out)
    return fail(h, VIF_ERR_INVALID_ARG, "vif_la_apply: bad arguments");
  if ((op == VIF_LA_FITC_SOLVE || op == VIF_LA_A || op == VIF_LA_A1) && !winv)
    return fail(h, VIF_ERR_INVALID_ARG, "vif_la_apply: winv is required for this operator");
  LaCtx c = la_ctx(h, ws);
  switch (op) {
    case VIF_LA_SIGMA: LA_TRY(la_sigma(c, ncol, v, out, nullptr)); break;
    case VIF_LA_A: LA_TRY(la_sigma(c, ncol, v, out, winv)); break;
    case VIF_LA_BINV: LA_TRY(la_binv(c, ncol, v, nullptr, out, nullptr, nullptr, nullptr)); break;
    case VIF_LA_BTINV: LA_TRY(la_btinv(c, ncol, v, out)); break;
    case VIF_LA_FITC_SOLVE:
      LA_TRY(la_fitc_build(c, winv));
      LA_TRY(la_fitc_solve(c, ncol, v, out));
      break;
    case VIF_LA_SIGMA_INV: LA_TRY(la_sigma_inv(c, ncol, v, out, nullptr)); break;
    case VIF_LA_A1: LA_TRY(la_sigma_inv(c, ncol, v, out, winv)); break;
    default: return fail(h, VIF_ERR_INVALID_ARG, "vif_la_apply: unknown operator");
  }
  VIF_WAIT(h, c.s);
  int ff = 0;
  VIF_CUDA(h, cudaMemcpy(&ff, c.fitc_fail(), sizeof(int), cudaMemcpyDeviceToHost), "status");
  if (ff) return fail(h, VIF_ERR_NOT_PD, "FITC: Cholesky of M_V failed");
  return VIF_OK;
}

int vif_la_nll(void* handle, void* ws, const double* y, const vif_la_opts* opts, const double* eps1,
               const double* eps2, double* b_mode, vif_la_terms* out) {
  Handle* h = reinterpret_cast<Handle*>(handle);
  if (!h) return fail(nullptr, VIF_ERR_INVALID_ARG, "handle is NULL");
  LA_TRY(la_check(h, ws));
  const Plan& P = h->P;
  if (!y || !opts || !out) return fail(h, VIF_ERR_INVALID_ARG, "vif_la_nll: NULL argument");
  const int ell = opts->nprobe;
  if (ell < 0 || ell > h->la_nprobe) return fail(h, VIF_ERR_INVALID_ARG, "nprobe exceeds the prepared workspace");
  if (ell > 0 && ((P.m > 0 && !eps1) || !eps2)) return fail(h, VIF_ERR_INVALID_ARG, "probe draws are NULL");
  if (opts->max_newton < 1 || opts->max_cg < 1 || opts->max_cg > h->la_maxcg)
    return fail(h, VIF_ERR_INVALID_ARG, "max_newton >= 1 and 1 <= max_cg <= the prepared max_cg");
  LaCtx c = la_ctx(h, ws);
  cudaStream_t s = c.s;
  const int64_t n = P.n;
  double* fin = c.sc(SC_MISC);  // fin[0..5] as la_finish_kernel, fin[7] = b.a
  double* bm = c.d(L_BM);
  VIF_CUDA(h, cudaMemsetAsync(bm, 0, n * sizeof(double), s), "memset b");
  VIF_CUDA(h, cudaMemsetAsync(c.fitc_fail(), 0, sizeof(int), s), "memset");
  // Newton's method for the mode through (pcls2), readings l3 / l4
  double psi_old = 0.0;
  int it = 0, cg_total = 0;
  std::vector<int> iters;
  for (it = 1; it <= opts->max_newton; ++it) {
    VIF_CUDA(h, launch_la_newton_prep(y, bm, n, c.d(L_W), c.d(L_WINV), c.d(L_V), c.d(L_X), s), "Newton prep");
    LA_TRY(la_sigma(c, 1, c.d(L_V), c.d(L_RHS), nullptr));
    LA_TRY(la_fitc_build(c, c.d(L_WINV)));
    LA_TRY(la_pcg(c, 1, c.d(L_RHS), c.d(L_X), true, opts->cg_tol, opts->max_cg, c.d(L_WINV), false, iters));
    cg_total += iters[0];
    VIF_CUDA(h, launch_la_newton_update(c.d(L_X), c.d(L_V), c.d(L_WINV), n, bm, c.d(L_A), s), "Newton update");
    VIF_CUDA(h, launch_la_reduce(1, y, bm, n, 1, c.d(L_RPART), fin + 0, s), "log p");
    LA_TRY(la_coldot(c, bm, c.d(L_A), n, 1, fin + 7));
    double hv[8];
    VIF_CUDA(h, cudaMemcpyAsync(hv, fin, sizeof(hv), cudaMemcpyDeviceToHost, s), "psi");
    VIF_WAIT(h, s);
    const double psi = hv[0] - 0.5 * hv[7];
    if (!isfinite(psi)) return fail(h, VIF_ERR_NOT_PD, "Laplace: Newton iterate is not finite");
    if (it > 1 && fabs(psi - psi_old) <= opts->newton_tol * fabs(psi_old)) break;
    psi_old = psi;
  }
  if (it > opts->max_newton) it = opts->max_newton;
  // b~^T Sigma_dagger^{-1} b~ = ||D^{-1/2} B b||^2 - ||L_M^{-1} W_U^T D^{-1/2} B b||^2 (Woodbury; l5)
  double* sv = c.d(L_T1);
  VIF_CUDA(h, launch_la_bapply(c.nbr(), c.d(L_B), P.mv, n, c.d(L_D), bm, sv, s), "D^-1/2 B b");
  LA_TRY(la_coldot(c, sv, sv, n, 1, fin + 1));
  if (P.mk > 0) {
    VIF_CUDA(h, launch_la_tsgemm(h->buf<double>(B_W), P.ld, P.mk, n, sv, 1, h->ord(0), nullptr, c.d(L_TSPART),
                                 c.d(L_CT), 1.0, s),
             "W_U^T s");
    VIF_CUDA(h, launch_gemm_tn(c.d(L_CT), P.mk, 1, c.d(L_LMINV), P.mk, P.mk, P.mk, 0, c.d(L_CT2), P.mk, 1.0, 0, s),
             "L_M^-1 c");
    LA_TRY(la_coldot(c, c.d(L_CT2), c.d(L_CT2), P.mk, 1, fin + 2));
  } else {
    VIF_CUDA(h, cudaMemsetAsync(fin + 2, 0, sizeof(double), s), "memset");
  }
  int slq_max = 0;
  double slq_mean = 0.0;
  if (ell > 0) {
    // log det(Sigma_dagger W + I) by SLQ (slq_v2), FITC-preconditioned, z_i = D_V^{1/2} eps2 + U eps1
    VIF_CUDA(h, launch_la_newton_prep(y, bm, n, c.d(L_W), c.d(L_WINV), c.d(L_V), nullptr, s), "W at the mode");
    LA_TRY(la_fitc_build(c, c.d(L_WINV)));
    VIF_CUDA(h, launch_la_reduce(2, c.d(L_W), nullptr, n, 1, c.d(L_RPART), fin + 3, s), "log det W");
    VIF_CUDA(h, launch_la_reduce(2, c.d(L_DV), nullptr, n, 1, c.d(L_RPART), fin + 4, s), "log det D_V");
    VIF_CUDA(h, launch_la_rowscale(eps2, c.d(L_DV), 1, n, ell, c.d(L_RHS), s), "D_V^1/2 eps2");
    if (P.mk > 0) {
      VIF_CUDA(h, cudaMemsetAsync(c.d(L_E1T), 0, (size_t)ell * P.mk * sizeof(double), s), "memset");
      VIF_CUDA(h, launch_la_transpose(eps1, P.m, ell, ell, c.d(L_E1T), P.mk, s), "eps1^T");
      VIF_CUDA(h, launch_gemm_tn(c.U(), P.ld, n, c.d(L_E1T), P.mk, ell, P.mk, 0, c.d(L_RHS), ell, 1.0, 1, s),
               "U eps1");
    }
    LA_TRY(la_pcg(c, ell, c.d(L_RHS), c.d(L_X), false, opts->slq_tol, opts->max_cg, c.d(L_WINV), true, iters));
    for (int k = 0; k < ell; ++k) {
      slq_max = iters[k] > slq_max ? iters[k] : slq_max;
      slq_mean += iters[k] / (double)ell;
    }
    VIF_CUDA(h, cudaMemcpyAsync(c.i(L_ITERS), iters.data(), ell * sizeof(int), cudaMemcpyHostToDevice, s), "iters");
    VIF_CUDA(h, launch_la_slq(c.d(L_HA), c.d(L_HB), c.i(L_ITERS), ell, h->la_maxcg, c.d(L_SLQS), c.sc(SC_SLQ), s),
             "SLQ quadrature");
  } else {
    VIF_CUDA(h, cudaMemsetAsync(fin + 3, 0, 3 * sizeof(double), s), "memset");
  }
  VIF_CUDA(h, launch_la_finish(fin, c.sc(SC_SLQ), n, ell, c.sc(SC_OUT), s), "finish");
  if (b_mode) VIF_CUDA(h, cudaMemcpyAsync(b_mode, bm, n * sizeof(double), cudaMemcpyDefault, s), "b copy");
  double o[6];
  int ff = 0;
  VIF_CUDA(h, cudaMemcpyAsync(o, c.sc(SC_OUT), sizeof(o), cudaMemcpyDeviceToHost, s), "terms");
  VIF_CUDA(h, cudaMemcpyAsync(&ff, c.fitc_fail(), sizeof(int), cudaMemcpyDeviceToHost, s), "status");
  VIF_WAIT(h, s);
  out->nll = ell > 0 ? o[0] : NAN;
  out->neg_loglik = o[1];
  out->quad = o[2];
  out->logdet = ell > 0 ? o[3] : NAN;
  out->logdet_W = ell > 0 ? o[4] : NAN;
  out->logdet_P = ell > 0 ? o[5] : NAN;
  out->newton_iters = it;
  out->cg_iters = cg_total;
  out->slq_iters_max = slq_max;
  out->slq_iters_mean = slq_mean;
  if (ff) return fail(h, VIF_ERR_NOT_PD, "FITC: Cholesky of M_V failed");
  return VIF_OK;
}

int vif_copy_U(void* handle, double* out) {
  Handle* h = reinterpret_cast<Handle*>(handle);
  if (!h || !out) return fail(h, VIF_ERR_INVALID_ARG, "NULL argument");
  if (!h->factored) return fail(h, VIF_ERR_STATE, "vif_copy_U before vif_factor");
  const Plan& P = h->P;
  if (P.m == 0) return VIF_OK;
  VIF_CUDA(h, cudaMemcpy2DAsync(out, (size_t)P.m * 8, h->buf<double>(B_U), (size_t)P.ld * 8, (size_t)P.m * 8, P.n,
                                cudaMemcpyDefault, h->stream),
           "copy U");
  VIF_WAIT(h, h->stream);
  return VIF_OK;
}

int vif_gram(const double* W, int64_t ldw, int64_t nrows, int32_t ncols, double* G, int64_t ldg, int32_t engine,
             void* stream) {
  if (!W || !G || ncols < 1 || nrows < 0 || ldw < ncols || (ldw & 1) || ldg < ncols || engine < 0 || engine > 1 ||
      (engine == 0 && !syrk_i8_supported(ncols)) || (reinterpret_cast<uintptr_t>(W) & 15))
    return fail(nullptr, VIF_ERR_INVALID_ARG, "vif_gram: invalid argument");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  char* scratch = nullptr;
  size_t ws = 0, part = 0, aux = 0;
  int nsplit = 0;
  const int64_t cap = std::min<int64_t>(std::max<int64_t>(nrows, 1), (int64_t)1 << 20);
  if (engine == 0) {
    ws = (syrk_i8_ws_bytes(ncols, cap) + 255) / 256 * 256;
    part = syrk_i8_part_doubles(ncols, cap) * sizeof(double);
    aux = syrk_i8_aux_bytes(ncols);
  } else {
    nsplit = syrk_nsplit(ncols, nrows, kPlanSMs);
    part = syrk_part_doubles(ncols, nsplit) * sizeof(double);
  }
  {
    // keep freed scratch in the device's default pool between calls (no re-mapping of GBs per call)
    int dev = 0;
    cudaMemPool_t pool;
    if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t thr = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
  }
  cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&scratch), ws + part + aux + 256, s);
  if (e != cudaSuccess) return fail(nullptr, VIF_ERR_CUDA, std::string("vif_gram: ") + cudaGetErrorString(e));
  double* gpart = reinterpret_cast<double*>(scratch + ws);
  if (engine == 0)
    e = launch_syrk_i8(W, ldw, nrows, ncols, reinterpret_cast<int8_t*>(scratch), cap, gpart,
                       scratch + ws + (part + 255) / 256 * 256, G, (int)ldg, kPlanSMs, s);
  else
    e = launch_syrk(W, ldw, nrows, ncols, nsplit, gpart, G, (int)ldg, s);
  const cudaError_t e2 = cudaFreeAsync(scratch, s);
  if (e == cudaSuccess) e = e2;
  if (e != cudaSuccess) return fail(nullptr, VIF_ERR_CUDA, std::string("vif_gram: ") + cudaGetErrorString(e));
  return VIF_OK;
}

int vif_launch_count(void* handle, int64_t* count) {
  Handle* h = reinterpret_cast<Handle*>(handle);
  if (!h || !count) return fail(h, VIF_ERR_INVALID_ARG, "NULL argument");
  *count = h->launches;
  return VIF_OK;
}

int vif_profile(void* handle, int32_t enable) {
  Handle* h = reinterpret_cast<Handle*>(handle);
  if (!h) return fail(nullptr, VIF_ERR_INVALID_ARG, "handle is NULL");
  h->prof = enable != 0;
  for (int k = 0; k < S_COUNT; ++k) h->stage_ms[k] = 0.0;
  h->prof_evals = 0;
  return VIF_OK;
}

int vif_stage_times(void* handle, double* ms_out, int64_t* evaluations) {
  Handle* h = reinterpret_cast<Handle*>(handle);
  if (!h || !ms_out) return fail(h, VIF_ERR_INVALID_ARG, "NULL argument");
  for (int k = 0; k < S_COUNT; ++k) ms_out[k] = h->stage_ms[k];
  if (evaluations) *evaluations = h->prof_evals;
  return VIF_OK;
}

const char* vif_stage_name(int32_t stage) { return stage >= 0 && stage < S_COUNT ? kStageNames[stage] : ""; }

const char* vif_last_error(void* handle) {
  Handle* h = reinterpret_cast<Handle*>(handle);
  return h ? h->err.c_str() : g_create_error.c_str();
}

void vif_destroy(void* handle) {
  Handle* h = reinterpret_cast<Handle*>(handle);
  if (!h) return;
  if (h->comm) nccl().CommDestroy(h->comm);
  for (cudaEvent_t ev : h->ev_k1)
    if (ev) cudaEventDestroy(ev);
  for (cudaEvent_t ev : h->ev_ag)
    if (ev) cudaEventDestroy(ev);
  if (h->cstream) cudaStreamDestroy(h->cstream);
  for (cudaEvent_t ev : h->ev_v)
    if (ev) cudaEventDestroy(ev);
  if (h->ev_k0) cudaEventDestroy(h->ev_k0);
  if (h->ev_sy) cudaEventDestroy(h->ev_sy);
  if (h->s_k1) cudaStreamDestroy(h->s_k1);
  for (int k = 0; k < 2; ++k) {
    if (h->ev_ready[k]) cudaEventDestroy(h->ev_ready[k]);
    if (h->ev_free[k]) cudaEventDestroy(h->ev_free[k]);
  }
  if (h->s_copy) cudaStreamDestroy(h->s_copy);
  if (h->s_sy) cudaStreamDestroy(h->s_sy);
  for (int k = 0; k < S_COUNT; ++k)
    for (int j = 0; j < 2; ++j)
      if (h->ev[k][j]) cudaEventDestroy(h->ev[k][j]);
  delete h;
}

}  // extern "C"
