// C-ABI implementation: context, init (upload, Padé-13 expm, quadrature ladder), composition driver.
// See include/dme.h for the contract and DESIGN.md for the design and the paper readings.
#include <nccl.h>
#include <nvtx3/nvToolsExt.h>

#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "aux.h"
#include "cheb.h"
#include "common.cuh"
#include "dme.h"
#include "gemm_nt.h"
#include "lu.h"
#include "ozaki.h"
#include "small.h"

using namespace dme;

// NVTX ranges per flow / phase (SURVEY §5 tracing; the paper profiles per sub-function):
// "dme::T1", "dme::T12", "dme::compress", "dme::init", ... visible in nsys / ncu --nvtx.
// Header-only NVTX3: without an attached tool a range costs a few ns.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

void axpy_cols(double* Y, int64_t ldy, const double* X, int64_t ldx, int64_t rows, int64_t cols,
               double alpha, cudaStream_t st);

namespace {

thread_local std::string g_last_error;

struct DmeError : std::runtime_error {
  dme_status code;
  DmeError(dme_status c, const std::string& m) : std::runtime_error(m), code(c) {}
};
#define DME_REQUIRE(cond, code, msg) \
  do {                               \
    if (!(cond)) throw DmeError(code, msg); \
  } while (0)
#define DME_NCCL(x)                                                                       \
  do {                                                                                    \
    ncclResult_t r_ = (x);                                                                \
    if (r_ != ncclSuccess)                                                                \
      throw DmeError(DME_ERR_NCCL, std::string(#x) + ": " + ncclGetErrorString(r_));      \
  } while (0)

// Padé-13 coefficients b_0..b_13 (Higham 2005, Table 2.2 / eq. 2.3)
const double PADE_B[14] = {64764752532480000.0, 32382376266240000.0, 7771770303897600.0,
                           1187353796428800.0,  129060195264000.0,   10559470521600.0,
                           670442572800.0,      33522128640.0,       1323241920.0,
                           40840800.0,          960960.0,            16380.0,
                           182.0,               1.0};
const double THETA13 = 5.371920351148152;

constexpr int64_t KMAX = SMALL_K_MAX;  // column capacity of every factor buffer
constexpr double GRAM_FLOOR = 1e-14;    // effective tolerance floor of the single-pass Gram compression
constexpr double SPLIT_TOL = 1e-11;     // refined compression: first pass keeps theta > 1e-11 theta_max
// The oracle compresses the whole composite rule once (reading G6); the ladder compresses at every
// rung, so the rungs below the final L_I(h/2), L_I(h) keep 64x finer directions and only the final
// factors are truncated at trunc_tol (their ranks then match a one-shot truncation)
constexpr double LADDER_TOL = 1.0 / 64;
constexpr int LOOKAHEAD_RESERVE = 8;  // SMs the look-ahead stream leaves free (tools/la_ab.sh: 116-140 equal step rate)

// Gauss-Legendre nodes/weights on [0,1] by Newton on P_q (Golub-Welsch-free; own implementation)
void gauss_legendre01(int q, std::vector<double>& c, std::vector<double>& w) {
  c.assign(q, 0.0);
  w.assign(q, 0.0);
  for (int i = 0; i < q; ++i) {
    double x = std::cos(M_PI * (i + 0.75) / (q + 0.5));
    for (int it = 0; it < 100; ++it) {
      double p0 = 1.0, p1 = x;
      for (int k = 2; k <= q; ++k) {
        const double pk = ((2.0 * k - 1.0) * x * p1 - (k - 1.0) * p0) / k;
        p0 = p1;
        p1 = pk;
      }
      const double dp = q * (x * p1 - p0) / (x * x - 1.0);
      const double dx = p1 / dp;
      x -= dx;
      if (std::fabs(dx) < 1e-17) break;
    }
    double p0 = 1.0, p1 = x;
    for (int k = 2; k <= q; ++k) {
      const double pk = ((2.0 * k - 1.0) * x * p1 - (k - 1.0) * p0) / k;
      p0 = p1;
      p1 = pk;
    }
    const double dp = q * (x * p1 - p0) / (x * x - 1.0);
    c[q - 1 - i] = 0.5 * (x + 1.0);
    w[q - 1 - i] = 1.0 / ((1.0 - x * x) * dp * dp);  // = (2/((1-x^2)P'^2)) / 2
  }
}

struct Planner {
  char* base = nullptr;
  size_t off = 0;
  template <class T>
  T* take(size_t count) {
    off = (off + 255) & ~size_t(255);
    T* p = base ? reinterpret_cast<T*>(base + off) : nullptr;
    off += count * sizeof(T);
    return p;
  }
};

}  // namespace

struct dme_ctx {
  int64_t n = 0, ldn = 0, p = 0, m = 0, r0 = 0;
  bool has_S = false, dre = false;
  bool sparse_S = false;   // S given in CSR form: T4 products by spmm_csr (aux.h)
  int64_t S_nnz = 0;
  int *S_rp = nullptr, *S_ci = nullptr;
  double* S_v = nullptr;
  int world = 1, rank = 0;  // logical shards of E's rows (= ranks, or virtual shards) and this rank
  int64_t nloc = 0, row0 = 0, rows_loc = 0;
  // shards computed by this process: real multi-rank: {rank}; options.virtual_world = G on one GPU:
  // all G (each through the same per-shard kernels, staging block, NCCL allgather on a one-rank
  // communicator and unpack as a real G-rank run); rows of E held in memory: [erow0, erow0 + erows)
  bool virt = false;
  int nsh = 1, sh0 = 0;
  int64_t erow0 = 0, erows = 0, img = 0;
  dme_options opt{};
  cudaStream_t st = nullptr;
  double h = 0;
  // persistent device buffers
  double *E_half = nullptr, *E_full = nullptr, *S = nullptr, *Bcol = nullptr, *LQ = nullptr;
  double *Zc12h = nullptr, *Zc12f = nullptr, *Zc2 = nullptr, *Z = nullptr, *Ztmp = nullptr;
  double *G = nullptr, *H = nullptr, *Tm = nullptr, *Vg = nullptr, *Es = nullptr, *LRinv = nullptr, *sstats = nullptr;
  double *norm_dev = nullptr, *red_scratch = nullptr, *stage = nullptr;
  double *Zs = nullptr, *Gs = nullptr, *Us = nullptr, *Ts = nullptr;  // refined compression: Zc U, its Gram, U, tail eigenvectors
  bool refine = true;      // options.compression == DME_COMPRESS_REFINED
  bool no_proj_gram = false;  // DME_NO_PROJ_GRAM: unfused Zs = Zc U + Gram (A/B measurement knob)
  bool no_fused_fin = false;  // DME_NO_FUSED_FIN: the tail pass's FIN kernel instead of the fused check
  double tol_scale = 1.0;  // intermediate quadrature-ladder compressions run at trunc_tol * LADDER_TOL
  double last_st[5] = {0, 0, 0, 0, 0};  // stats of the last small-kernel pass read by the host
  cudaEvent_t ev_zc = nullptr, ev_tm = nullptr;
  double *LA = nullptr;  // look-ahead operand [E_h L_I(h) | E_h Y]  (ldn x KMAX)
  // Gram-congruence pipeline (run_f12f3_body): GB = [L_I(h) | B | E_h L_I(h) | E_h Y] (ldn x KMAX),
  // its Gram Ghat (KMAX^2), double-buffered eigen-compression output Tm / Tm2
  double *GB = nullptr, *Ghat = nullptr, *Tm2 = nullptr;
  int* r_dev = nullptr;
  GemmScratch gs, gs2;   // scratch of the main stream and of the look-ahead stream
  // int8 digit slices for the Ozaki E pass (ozaki.h): rows of E_{h/2} / E_h (local shard, sliced
  // once at init) and the columns of the pass operand (one buffer per stream)
  bool oz = false, oz_ready = false;
  int64_t ozld = 0;
  int8_t *ozEh = nullptr, *ozEf = nullptr, *ozY = nullptr, *ozY2 = nullptr;
  int *exEh = nullptr, *exEf = nullptr, *exY = nullptr, *exY2 = nullptr;
  double *ozpm = nullptr, *ozpm2 = nullptr;  // slicing scratch (row maxima per chunk)
  OzScratch ozs, ozs2;
  // init-time square products on the int8 tensor cores: rasterised tile lists
  bool oz_init = false;
  int2* oz_tiles_up = nullptr;  // upper tile triangle (symmetric products)
  int2* oz_tiles_all = nullptr;
  int ntiles_up = 0, ntiles_all = 0;
  std::vector<int2> h_tiles_up, h_tiles_all;
  cudaStream_t st2 = nullptr;
  HostMap* hmap = nullptr;       // pinned, host-mapped rank record (small.h)
  HostMap* hmap_dev = nullptr;   // its device alias
  int map_seq = 0;
  cudaEvent_t ev_gram = nullptr, ev_ahead = nullptr, ev_ghat = nullptr, ev_cong = nullptr,
              ev_y = nullptr;
  bool lookahead = true;
  // init-only device buffers
  double *Aup = nullptr, *X0 = nullptr, *BT = nullptr, *X2 = nullptr, *X4 = nullptr, *X6 = nullptr;
  double *T1 = nullptr, *U = nullptr, *V = nullptr, *lu_scr = nullptr, *Wa = nullptr, *Wb = nullptr;
  double *Yn = nullptr, *L0d = nullptr, *D0d = nullptr;
  // host state
  int64_t r = 0, qh = 0, qf = 0;
  int32_t rank_cap = 0, qn = 14, subpanels = 1;
  std::vector<double> lrinv_host;
  dme_stats stats{};
  bool poisoned = false;
  bool force_jacobi = false;
  bool symA = false;  // A == A^T exactly (host check): symmetric Padé products
  bool fsal = true;
  // sparse A: Chebyshev exponential actions instead of dense E (cheb.h)
  bool sparse = false;
  bool cheb_e = false;  // dense path, sparse symmetric A: E_{h/2} and L_I by Chebyshev actions
  ChebHost chost;
  ChebOp cop;
  ncclComm_t comm = nullptr;
  // profiling: (start, stop, class, flops, bytes) event records drained at sync points
  bool profile = false;
  struct Rec { cudaEvent_t a, b; int cls; double flops, bytes; };
  std::vector<Rec> pending;
  std::vector<cudaEvent_t> pool;
  cudaEvent_t tl_base = nullptr;  // timeline reference (DME_TIMELINE)
  ~dme_ctx() {
    for (auto& r : pending) { cudaEventDestroy(r.a); cudaEventDestroy(r.b); }
    for (auto e : pool) cudaEventDestroy(e);
    if (comm) ncclCommDestroy(comm);
    if (st2) cudaStreamDestroy(st2);
    if (hmap) cudaFreeHost(hmap);
    if (ev_gram) cudaEventDestroy(ev_gram);
    if (ev_ahead) cudaEventDestroy(ev_ahead);
    for (cudaEvent_t e : {ev_ghat, ev_cong, ev_y, ev_zc, ev_tm})
      if (e) cudaEventDestroy(e);
    if (tl_base) cudaEventDestroy(tl_base);
  }
};

namespace {

void plan_buffers(dme_ctx* c, Planner& P) {
  const int64_t n = c->n, ld = c->ldn;
  const size_t nn = (size_t)n * ld, fk = (size_t)ld * KMAX;
  if (!c->sparse) {  // the rows of E this process holds (a real rank: its own rows only)
    c->E_half = P.take<double>((size_t)std::max<int64_t>(c->erows, 1) * ld);
    c->E_full = P.take<double>((size_t)std::max<int64_t>(c->erows, 1) * ld);
  } else {  // partitioned ELL of A^T (cheb.h); no n x n matrix in sparse mode
    const size_t ell = (size_t)c->chost.w * CHEB_CLUSTER * c->chost.R;
    c->cop.n = c->chost.n; c->cop.R = c->chost.R; c->cop.w = c->chost.w; c->cop.C = c->chost.C;
    c->cop.H = c->chost.H; c->cop.P = c->chost.P;
    c->cop.a = c->chost.a; c->cop.b = c->chost.b; c->cop.norm1 = c->chost.norm1;
    c->cop.sym = c->chost.sym; c->cop.mu = c->chost.mu; c->cop.tnorm = c->chost.tnorm;
    c->cop.global = c->chost.global;
    if (c->cop.global) {  // vectors of the grid-wide action (cheb.h)
      const size_t gv = (size_t)CHEB_CLUSTER * c->chost.R * KMAX;
      c->cop.gv0 = P.take<double>(gv);
      c->cop.gv1 = P.take<double>(gv);
      c->cop.gy = P.take<double>(gv);
    }
    c->cop.val = P.take<double>(ell);
    c->cop.idx = P.take<uint32_t>(ell);
    c->cop.push = P.take<uint32_t>(std::max<size_t>(c->chost.push.size(), 1));
    c->cop.rptr = P.take<uint32_t>(std::max<size_t>(c->chost.rptr.size(), 1));
    c->cop.rent = P.take<uint32_t>(std::max<size_t>(c->chost.rent.size(), 1));
  }
  if (c->has_S && !c->sparse_S) c->S = P.take<double>(nn);
  if (c->sparse_S) {
    c->S_rp = P.take<int>((size_t)n + 1);
    c->S_ci = P.take<int>((size_t)std::max<int64_t>(c->S_nnz, 1));
    c->S_v = P.take<double>((size_t)std::max<int64_t>(c->S_nnz, 1));
  }
  c->Bcol = P.take<double>((size_t)ld * std::max<int64_t>(c->m, 1));
  c->LQ = P.take<double>((size_t)ld * std::max<int64_t>(c->p, 1));
  c->Zc12h = P.take<double>(fk);
  c->Zc12f = P.take<double>(fk);
  c->Zc2 = P.take<double>(fk);
  c->Z = P.take<double>(fk);
  c->Ztmp = P.take<double>(fk);
  c->G = P.take<double>((size_t)KMAX * KMAX);
  c->H = P.take<double>((size_t)KMAX * SMALL_M_MAX);
  c->Tm = P.take<double>((size_t)KMAX * KMAX);
  c->Vg = P.take<double>((size_t)KMAX * KMAX);
  c->Es = P.take<double>(eig_split_scratch_doubles());
  c->LRinv = P.take<double>(SMALL_M_MAX * SMALL_M_MAX);
  c->sstats = P.take<double>(16);
  c->norm_dev = P.take<double>(16);
  c->red_scratch = P.take<double>(1024);
  c->r_dev = P.take<int>(16);
  c->gs.max_grid = 256;
  c->gs.max_tiles = 1 << 16;
  c->gs.partial = P.take<double>(GemmScratch::partial_doubles(c->gs.max_grid));
  c->gs.counters = P.take<int>((size_t)c->gs.max_tiles);
  c->gs.tile_list = P.take<int2>((size_t)c->gs.max_tiles);
  c->gs2.max_grid = 256;
  c->gs2.max_tiles = 1 << 16;
  c->gs2.partial = P.take<double>(GemmScratch::partial_doubles(c->gs2.max_grid));
  c->gs2.counters = P.take<int>((size_t)c->gs2.max_tiles);
  c->LA = P.take<double>(fk);
  c->Zs = P.take<double>(fk);
  c->Gs = P.take<double>((size_t)KMAX * KMAX);
  c->Us = P.take<double>((size_t)KMAX * KMAX);
  c->Ts = P.take<double>((size_t)KMAX * KMAX);
  c->GB = P.take<double>(fk);
  c->Ghat = P.take<double>((size_t)KMAX * KMAX);
  c->Tm2 = P.take<double>((size_t)KMAX * KMAX);
  if (c->oz) {
    c->ozld = oz_ldk(n);
    const int64_t rl = std::max<int64_t>(c->rows_loc, 1);
    // E-digit buffers: the local rows of E for the passes, and during the (replicated) init the
    // digits of both n x n operands of each product: n rows
    const int64_t rb = std::max<int64_t>(c->oz_init ? std::max<int64_t>(rl, n) : rl, (int64_t)c->nsh * c->nloc);
    // (the E passes read the tiled, pre-swizzled image of oz_slice_rows_tiled, one image per shard
    // computed here; the init products the row layout)
    c->img = (oz_tiled_bytes(std::max<int64_t>(c->nloc, 1), n) + 255) / 256 * 256;
    const size_t es = std::max<size_t>((size_t)OZ_S * rb * c->ozld, (size_t)c->nsh * c->img);
    const size_t ys = (size_t)OZ_S * OZ_NMAX * c->ozld;
    c->ozEh = P.take<int8_t>(es);
    c->ozEf = P.take<int8_t>(es);
    c->ozY = P.take<int8_t>(ys);
    c->ozY2 = P.take<int8_t>(ys);
    c->exEh = P.take<int>(rb);
    c->exEf = P.take<int>(rb);
    c->exY = P.take<int>(OZ_NMAX);
    c->exY2 = P.take<int>(OZ_NMAX);
    c->ozpm = P.take<double>(oz_slice_scratch_doubles(std::max<int64_t>(rb, OZ_NMAX), n));
    c->ozpm2 = P.take<double>(oz_slice_scratch_doubles(OZ_NMAX, n));
    if (c->oz_init) {
      c->h_tiles_up = oz_tile_list(n, n, true);
      c->h_tiles_all = oz_tile_list(n, n, false);
      c->ntiles_up = (int)c->h_tiles_up.size();
      c->ntiles_all = (int)c->h_tiles_all.size();
      c->oz_tiles_up = P.take<int2>(c->h_tiles_up.size());
      c->oz_tiles_all = P.take<int2>(c->h_tiles_all.size());
    }
    for (OzScratch* o : {&c->ozs, &c->ozs2}) {
      o->max_tiles = ceil_div(rl, 128);
      o->max_grid = 256;
      o->partial = P.take<double>(OzScratch::partial_doubles(o->max_tiles, o->max_grid));
      o->counters = P.take<int>((size_t)o->max_tiles);
    }
  }
  if (c->world > 1) c->stage = P.take<double>((size_t)c->world * c->nloc * KMAX);  // (virtual too)
  // init-only
  if (!c->sparse) {
    c->Aup = P.take<double>(nn);
    c->X0 = P.take<double>(nn);
    c->BT = P.take<double>(nn);
    c->X2 = P.take<double>(nn);
    c->X4 = P.take<double>(nn);
    c->X6 = P.take<double>(nn);
    c->T1 = P.take<double>(nn);
    c->U = P.take<double>(nn);
    c->V = P.take<double>(nn);
    c->lu_scr = P.take<double>(lu_scratch_doubles(n));
  }
  c->Wa = P.take<double>((size_t)ld * std::max<int64_t>(std::max(c->p, c->m), 1));
  c->Wb = P.take<double>((size_t)ld * std::max<int64_t>(c->p, 1));
  c->Yn = P.take<double>((size_t)ld * std::max<int64_t>(c->p * c->qn, 1));
  c->L0d = P.take<double>((size_t)ld * std::max<int64_t>(c->r0, 1));
  c->D0d = P.take<double>((size_t)std::max<int64_t>(c->r0 * c->r0, 1));
}

void shard_rows(int64_t n, int world, int rank, int64_t* row0, int64_t* rows, int64_t* nloc) {
  int64_t nl = (n + world - 1) / world;
  nl = (nl + 15) / 16 * 16;
  *nloc = nl;
  *row0 = std::min<int64_t>(n, (int64_t)rank * nl);
  *rows = std::min<int64_t>(nl, n - *row0);
}

// Largest Ritz value of a symmetric CSR matrix after `iters` plain Lanczos steps (host; a lower
// estimate of lambda_max: Ritz values lie inside the spectrum, and the extreme one converges first,
// loss of orthogonality only adds ghost copies). Start vector: a fixed pseudo-random one.
double lanczos_lmax(int64_t n, const int64_t* rp, const int32_t* ci, const double* vv, int iters) {
  std::vector<double> q(n), qp(n, 0.0), w(n);
  uint64_t s = 0x9E3779B97F4A7C15ull;
  double nrm = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    s = s * 6364136223846793005ull + 1442695040888963407ull;
    q[i] = (double)(s >> 11) * 0x1.0p-53 - 0.5;
    nrm += q[i] * q[i];
  }
  nrm = std::sqrt(nrm);
  for (auto& x : q) x /= nrm;
  std::vector<double> al, be;
  double beta = 0.0;
  for (int it = 0; it < iters; ++it) {
    for (int64_t i = 0; i < n; ++i) {
      double acc = 0.0;
      for (int64_t e = rp[i]; e < rp[i + 1]; ++e) acc += vv[e] * q[ci[e]];
      w[i] = acc - beta * qp[i];
    }
    double alpha = 0.0;
    for (int64_t i = 0; i < n; ++i) alpha += w[i] * q[i];
    for (int64_t i = 0; i < n; ++i) w[i] -= alpha * q[i];
    double b2 = 0.0;
    for (int64_t i = 0; i < n; ++i) b2 += w[i] * w[i];
    al.push_back(alpha);
    beta = std::sqrt(b2);
    if (!(beta > 1e-300)) break;
    be.push_back(beta);
    for (int64_t i = 0; i < n; ++i) { qp[i] = q[i]; q[i] = w[i] / beta; }
  }
  // largest eigenvalue of the Lanczos tridiagonal by bisection on its Sturm sequence
  const int m = (int)al.size();
  double lo = 1e300, hi = -1e300;
  for (int i = 0; i < m; ++i) {
    const double r = (i > 0 ? std::fabs(be[i - 1]) : 0.0) + (i + 1 < m ? std::fabs(be[i]) : 0.0);
    lo = std::min(lo, al[i] - r);
    hi = std::max(hi, al[i] + r);
  }
  auto count_below = [&](double x) {  // eigenvalues < x
    int cnt = 0;
    double dq = 1.0;
    for (int i = 0; i < m; ++i) {
      dq = (al[i] - x) - (i > 0 ? be[i - 1] * be[i - 1] / dq : 0.0);
      if (dq == 0.0) dq = -1e-300;
      cnt += dq < 0.0;
    }
    return cnt;
  };
  for (int it = 0; it < 200 && hi - lo > 1e-12 * std::max(std::fabs(lo), std::fabs(hi)); ++it) {
    const double mid = 0.5 * (lo + hi);
    if (count_below(mid) < m) lo = mid; else hi = mid;
  }
  return 0.5 * (lo + hi);
}

// Accuracy gate of the Chebyshev exponential action (cheb.h): its truncation error is
// 2^-56 e^{tau b} ||X|| (b = the Gershgorin upper bound of A), so relative to the action's size
// e^{tau lambda_max} it is amplified by e^{tau (b - lambda_max)}. Accept when tau max(b, 0) <= ln 4
// (absolute error <= 4 2^-56 ||X||, the level of the FP64 Padé products) or when the Lanczos
// estimate gives tau (b - lambda_max) <= ln 4 (it underestimates lambda_max: conservative).
bool cheb_accurate(double tau, double b, int64_t n, const int64_t* rp, const int32_t* ci,
                   const double* vv, double* lmax_out) {
  const double lim = std::log(4.0);
  *lmax_out = NAN;
  if (tau * std::max(b, 0.0) <= lim) return true;
  const double lm = lanczos_lmax(n, rp, ci, vv, 40);
  *lmax_out = lm;
  return tau * (b - lm) <= lim;
}

void fill_dims(dme_ctx* c, const dme_problem* pr, const dme_options* o) {
  c->n = pr->n;
  c->ldn = (pr->n + 15) / 16 * 16;
  c->p = pr->p;
  c->m = pr->m;
  c->r0 = pr->r0;
  c->sparse_S = pr->S == nullptr && pr->S_rowptr != nullptr;
  c->has_S = pr->S != nullptr || c->sparse_S;
  c->S_nnz = c->sparse_S ? pr->S_nnz : 0;
  c->opt = *o;
  c->world = o->world_size > 0 ? o->world_size : 1;
  c->rank = o->world_rank;
  c->virt = c->world == 1 && o->virtual_world > 1;
  if (c->virt) c->world = o->virtual_world;
  c->nsh = c->virt ? c->world : 1;
  c->sh0 = c->virt ? 0 : c->rank;
  shard_rows(c->n, c->world, c->sh0, &c->row0, &c->rows_loc, &c->nloc);
  // E rows held: a real rank keeps its own rows only; one process (single or virtual) all of them
  c->erow0 = (c->world > 1 && !c->virt) ? c->row0 : 0;
  c->erows = (c->world > 1 && !c->virt) ? c->rows_loc : c->n;
  c->qn = o->quad_nodes > 0 ? o->quad_nodes : 14;
  c->subpanels = o->quad_subpanels > 0 ? o->quad_subpanels : 1;
  int64_t cap = o->rank_cap > 0 ? o->rank_cap : c->n;
  c->rank_cap = (int32_t)std::min<int64_t>(cap, KMAX);
  c->h = o->h;
  c->fsal = o->no_fsal == 0;
  c->refine = o->compression == DME_COMPRESS_REFINED;
  c->no_proj_gram = std::getenv("DME_NO_PROJ_GRAM") != nullptr;
  c->no_fused_fin = std::getenv("DME_NO_FUSED_FIN") != nullptr;
  c->sparse = pr->A == nullptr && pr->A_rowptr != nullptr;
  if (c->sparse) {
    std::string err;
    const int code = cheb_prepare(pr->n, pr->A_nnz, pr->A_rowptr, pr->A_colind, pr->A_values, c->chost, &err);
    if (code) throw DmeError((dme_status)code, err);
    double lm = 0;
    // (a nonsymmetric A takes the Taylor route of cheb.h, accurate by its backward-error bound)
    DME_REQUIRE(!c->chost.sym ||
                    cheb_accurate(o->h, c->chost.b, pr->n, pr->A_rowptr, pr->A_colind, pr->A_values, &lm),
                DME_ERR_CONFIG,
                "sparse A: the Gershgorin bound of A is too loose for an accurate Chebyshev action "
                "(h (b - lambda_max) > ln 4); pass A dense (Padé-13)");
  }
  // E pass on the int8 tensor cores (exact digit slicing) unless disabled or out of its range
  c->oz = !c->sparse && o->e_pass != DME_EPASS_DMMA && c->n <= OZ_KMAX && c->rows_loc > 0;
  // the Padé products and squarings on the int8 tensor cores too (digits of both operands live
  // in the E-digit buffers until E is sliced; the init is replicated on every rank, local work)
  c->oz_init = c->oz;
}

bool all_finite(const double* x, size_t cnt) {
  for (size_t i = 0; i < cnt; ++i)
    if (!std::isfinite(x[i])) return false;
  return true;
}

void validate(const dme_problem* pr, const dme_options* o, bool dre) {
  DME_REQUIRE(pr && o, DME_ERR_INVALID, "NULL problem or options");
  DME_REQUIRE(pr->n > 0 && (pr->A || pr->A_rowptr), DME_ERR_INVALID,
              "n must be positive and A (dense) or A_rowptr (sparse) non-NULL");
  if (!pr->A) {
    DME_REQUIRE(!pr->M, DME_ERR_CONFIG, "a mass matrix M is not supported with a sparse A");
    DME_REQUIRE(o->world_size <= 1 && o->virtual_world <= 1, DME_ERR_CONFIG,
                "a sparse A runs on one GPU (world_size 1, no virtual shards)");
  }
  DME_REQUIRE(std::isfinite(o->h) && o->h > 0, DME_ERR_INVALID, "h must be positive and finite");
  DME_REQUIRE(pr->p >= 0 && (pr->p == 0 || pr->C), DME_ERR_INVALID, "C must be non-NULL when p > 0");
  DME_REQUIRE(pr->r0 >= 0 && (pr->r0 == 0 || pr->L0), DME_ERR_INVALID, "L0 must be non-NULL when r0 > 0");
  DME_REQUIRE(o->trunc_tol >= 0, DME_ERR_INVALID, "trunc_tol must be >= 0");
  if (dre) {
    DME_REQUIRE(pr->m >= 1 && pr->B && pr->R, DME_ERR_INVALID, "dre_init needs m >= 1, B and R");
  } else {
    DME_REQUIRE(pr->m == 0, DME_ERR_INVALID, "dle_init requires m == 0");
  }
  DME_REQUIRE(pr->m <= SMALL_M_MAX, DME_ERR_DIM, "m exceeds 8");
  const int qn = o->quad_nodes > 0 ? o->quad_nodes : 14;
  DME_REQUIRE(qn <= 64, DME_ERR_DIM, "quad_nodes must be <= 64");
  DME_REQUIRE(pr->p * qn <= KMAX && pr->r0 <= KMAX && pr->p <= KMAX, DME_ERR_DIM,
              "p * quad_nodes and r0 must be <= 224");
  const int sp = o->quad_subpanels > 0 ? o->quad_subpanels : 1;
  DME_REQUIRE((sp & (sp - 1)) == 0, DME_ERR_INVALID, "quad_subpanels must be a power of two");
  DME_REQUIRE(o->world_size <= 1 || o->nccl_uid, DME_ERR_INVALID, "nccl_uid required for world_size > 1");
  DME_REQUIRE(o->virtual_world >= 0 && o->virtual_world <= 64, DME_ERR_INVALID, "virtual_world must be in [0, 64]");
  // input finiteness (host scan; inputs are host arrays)
  const size_t nn = (size_t)pr->n * pr->n;
  (void)nn;  // A and S (n x n) are checked on the device after the upload (init_all)
  DME_REQUIRE(!(pr->M && (pr->S || pr->S_rowptr)), DME_ERR_CONFIG,
              "a mass matrix M together with the bilinear term S is not supported");
  if (!pr->S && pr->S_rowptr) {  // CSR S: structure and values on the host
    const int64_t n = pr->n;
    DME_REQUIRE(pr->S_nnz >= 0 && pr->S_nnz < (int64_t)1 << 31 && (pr->S_nnz == 0 || (pr->S_colind && pr->S_values)),
                DME_ERR_INVALID, "CSR S: bad nnz or NULL arrays");
    DME_REQUIRE(pr->S_rowptr[0] == 0 && pr->S_rowptr[n] == pr->S_nnz, DME_ERR_INVALID,
                "CSR S: row pointers must start at 0 and end at S_nnz");
    for (int64_t i = 0; i < n; ++i)
      DME_REQUIRE(pr->S_rowptr[i + 1] >= pr->S_rowptr[i], DME_ERR_INVALID, "CSR S: decreasing row pointers");
    for (int64_t e = 0; e < pr->S_nnz; ++e) {
      DME_REQUIRE(pr->S_colind[e] >= 0 && pr->S_colind[e] < n, DME_ERR_INVALID, "CSR S: column index out of range");
      DME_REQUIRE(std::isfinite(pr->S_values[e]), DME_ERR_INVALID, "CSR S: non-finite value");
    }
  }
  if (pr->p) DME_REQUIRE(all_finite(pr->C, (size_t)pr->p * pr->n), DME_ERR_INVALID, "C non-finite");
  if (pr->r0) DME_REQUIRE(all_finite(pr->L0, (size_t)pr->n * pr->r0), DME_ERR_INVALID, "L0 non-finite");
  if (pr->m) {
    DME_REQUIRE(all_finite(pr->B, (size_t)pr->n * pr->m) && all_finite(pr->R, (size_t)pr->m * pr->m),
                DME_ERR_INVALID, "B or R non-finite");
  }
}

// Host preprocessing of the m x m input weight: R = L_R L_R^T (validates SPD), returns L_R^{-1}.
std::vector<double> chol_inverse_lower(const double* R, int m) {
  std::vector<double> L(m * m, 0.0), Li(m * m, 0.0);
  for (int i = 0; i < m; ++i)
    for (int j = 0; j < m; ++j)
      DME_REQUIRE(std::fabs(R[i * m + j] - R[j * m + i]) <= 1e-12 * (std::fabs(R[i * m + j]) + 1e-300),
                  DME_ERR_INVALID, "R is not symmetric");
  for (int j = 0; j < m; ++j) {
    double d = R[j * m + j];
    for (int k = 0; k < j; ++k) d -= L[j * m + k] * L[j * m + k];
    DME_REQUIRE(d > 0, DME_ERR_INVALID, "R is not positive definite");
    L[j * m + j] = std::sqrt(d);
    for (int i = j + 1; i < m; ++i) {
      double s = R[i * m + j];
      for (int k = 0; k < j; ++k) s -= L[i * m + k] * L[j * m + k];
      L[i * m + j] = s / L[j * m + j];
    }
  }
  for (int c = 0; c < m; ++c) {
    for (int i = 0; i < m; ++i) {
      double s = (i == c) ? 1.0 : 0.0;
      for (int k = 0; k < i; ++k) s -= L[i * m + k] * Li[k * m + c];
      Li[i * m + c] = s / L[i * m + i];
    }
  }
  return Li;
}

void check_psd_host(const double* D, int64_t r) {
  // symmetric and positive semidefinite up to round-off (LDL^T with diagonal pivoting)
  std::vector<double> a(D, D + r * r);
  double mx = 0;
  for (int64_t i = 0; i < r * r; ++i) mx = std::max(mx, std::fabs(a[i]));
  for (int64_t i = 0; i < r; ++i)
    for (int64_t j = 0; j < r; ++j)
      DME_REQUIRE(std::fabs(a[i * r + j] - a[j * r + i]) <= 1e-12 * mx, DME_ERR_INVALID,
                  "D0 is not symmetric");
  std::vector<char> used(r, 0);
  for (int64_t step = 0; step < r; ++step) {
    int64_t pv = -1;
    double best = -1e300;
    for (int64_t i = 0; i < r; ++i)
      if (!used[i] && a[i * r + i] > best) { best = a[i * r + i]; pv = i; }
    if (pv < 0 || best <= 1e-13 * mx) {
      for (int64_t i = 0; i < r; ++i)
        if (!used[i]) DME_REQUIRE(a[i * r + i] >= -1e-10 * mx, DME_ERR_INVALID, "D0 is not PSD");
      return;
    }
    used[pv] = 1;
    for (int64_t i = 0; i < r; ++i)
      for (int64_t j = 0; j < r; ++j)
        if (!used[i] && !used[j]) a[i * r + j] -= a[i * r + pv] * a[pv * r + j] / best;
  }
}

void sync(dme_ctx* c) { DME_CUDA(cudaStreamSynchronize(c->st)); }

// ------------------------------------------------------------------ profiling (CUDA events)
enum { PROF_EPASS = 0, PROF_GRAM = 1, PROF_SMALL = 2, PROF_APPLY = 3 };
cudaEvent_t take_event(dme_ctx* c) {
  if (c->pool.empty()) {
    cudaEvent_t e;
    DME_CUDA(cudaEventCreate(&e));
    return e;
  }
  cudaEvent_t e = c->pool.back();
  c->pool.pop_back();
  return e;
}
struct ProfScope {
  dme_ctx* c;
  cudaStream_t s;
  dme_ctx::Rec r{};
  ProfScope(dme_ctx* cc, int cls, double flops = 0, double bytes = 0, cudaStream_t ss = nullptr)
      : c(cc), s(ss ? ss : cc->st) {
    if (!c->profile) return;
    r.a = take_event(c);
    r.b = take_event(c);
    r.cls = cls;
    r.flops = flops;
    r.bytes = bytes;
    DME_CUDA(cudaEventRecord(r.a, s));
  }
  ~ProfScope() {
    if (!c->profile) return;
    cudaEventRecord(r.b, s);
    c->pending.push_back(r);
  }
};
void drain_profile(dme_ctx* c) {
  static const bool timeline = getenv("DME_TIMELINE") != nullptr;
  static const char* names[] = {"epass", "gram", "small", "apply", "other"};
  for (auto& r : c->pending) {
    DME_CUDA(cudaEventSynchronize(r.b));
    float ms = 0;
    DME_CUDA(cudaEventElapsedTime(&ms, r.a, r.b));
    if (timeline && c->tl_base) {
      float t0 = 0, t1 = 0;
      if (cudaEventElapsedTime(&t0, c->tl_base, r.a) == cudaSuccess &&
          cudaEventElapsedTime(&t1, c->tl_base, r.b) == cudaSuccess)
        fprintf(stderr, "[dme timeline] %-6s %10.1f %10.1f us (%.1f)\n", names[r.cls < 5 ? r.cls : 4],
                t0 * 1e3, t1 * 1e3, (t1 - t0) * 1e3);
    }
    const double s = ms * 1e-3;
    switch (r.cls) {
      case PROF_EPASS:
        c->stats.prof_passes++;
        c->stats.prof_epass_seconds += s;
        c->stats.prof_epass_flops += r.flops;
        c->stats.prof_epass_bytes += r.bytes;
        break;
      case PROF_GRAM: c->stats.prof_gram_seconds += s; break;
      case PROF_SMALL: c->stats.prof_small_seconds += s; break;
      default: c->stats.prof_apply_seconds += s; break;
    }
    c->pool.push_back(r.a);
    c->pool.push_back(r.b);
  }
  c->pending.clear();
}

// ------------------------------------------------------------------ building blocks
// out (col-major, ldo) = alpha * E * X  (E: n x n row-major, X: n x k col-major), sharded over ranks
// rows [row0, row0 + rows) of shard s (s-th block of nloc rows)
void shard_range(const dme_ctx* c, int s, int64_t* r0, int64_t* rows) {
  *r0 = std::min<int64_t>(c->n, (int64_t)s * c->nloc);
  *rows = std::min<int64_t>(c->nloc, c->n - *r0);
}

// digit slices of the columns of X (one per pass; shared by the shards of this process)
void oz_slice_operand(dme_ctx* c, const double* X, int64_t k, cudaStream_t st, bool second) {
  oz_slice_rows(X, c->ldn, k, c->n, second ? c->ozY2 : c->ozY, c->ozld, (int64_t)OZ_NMAX * c->ozld,
                second ? c->exY2 : c->exY, second ? c->ozpm2 : c->ozpm, st);
}

// out (rows_s x k) = alpha * E[rows of shard s] * X on the int8 tensor cores; E = E_{h/2} or E_h
// (each shard's rows sliced once at init into their own tiled image); X already sliced
void oz_pass(dme_ctx* c, const double* E, int s, int64_t k, double* out, int64_t out_cs, double alpha,
             cudaStream_t st, bool second) {
  int64_t r0, rows;
  shard_range(c, s, &r0, &rows);
  if (rows <= 0) return;
  const int sl = s - c->sh0;  // local image index
  OzGemmArgs g;
  g.A = (E == c->E_full ? c->ozEf : c->ozEh) + (size_t)sl * c->img;
  g.eA = (E == c->E_full ? c->exEf : c->exEh) + (size_t)sl * c->nloc;
  g.lda = c->ozld; g.a_slice_stride = rows * c->ozld;
  g.B = second ? c->ozY2 : c->ozY; g.eB = second ? c->exY2 : c->exY;
  g.ldb = c->ozld; g.b_slice_stride = (int64_t)OZ_NMAX * c->ozld;
  g.M = rows; g.N = k; g.K = c->n; g.alpha = alpha;
  g.out = out; g.out_rs = 1; g.out_cs = out_cs;
  g.A_tiled = g.A;  // E digits in the tiled image (oz_slice_rows_tiled at the end of init)
  {
    // profiled as the E-pass kernel: the int8 product alone (the digit slicing of X, ~n k bytes,
    // is its own pair of small kernels before it)
    ProfScope ps(c, PROF_EPASS, 2.0 * g.M * c->n * k, 1.0 * OZ_S * g.M * c->n, st);
    oz_gemm(g, second ? c->ozs2 : c->ozs, st);
  }
  c->stats.ozaki_passes++;
}

// tiled digit images of the shards this process computes, from E (its rows start at E's row erow0)
void slice_shards(dme_ctx* c, const double* E, int8_t* img, int* ex, cudaStream_t st) {
  for (int sl = 0; sl < c->nsh; ++sl) {
    int64_t r0, rows;
    shard_range(c, c->sh0 + sl, &r0, &rows);
    if (rows > 0)
      oz_slice_rows_tiled(E + (r0 - c->erow0) * c->ldn, c->ldn, rows, c->n, img + (size_t)sl * c->img,
                          ex + (size_t)sl * c->nloc, c->ozpm, st);
  }
}

// out (col-major, ldo) = alpha * E * X  (E: row-major, X: n x k col-major). E is E_{h/2} / E_h (the
// rows this process holds) or a full n x n init buffer. Row-sharded (world > 1, real ranks or
// virtual shards): every shard of this process computes its rows into its staging block
// (nloc x k, col-major), one ncclAllGather replicates the blocks, a copy kernel unpacks them.
void epass_on(dme_ctx* c, const double* E, const double* X, int64_t k, double* out, int64_t ldo,
              double alpha, cudaStream_t st, GemmScratch& gs) {
  if (k <= 0) return;
  c->stats.e_passes++;
  const bool second = &gs == &c->gs2;
  const bool held = E == c->E_half || E == c->E_full;  // rows [erow0, erow0 + erows) only
  const bool use_oz = c->oz && c->oz_ready && k <= OZ_NMAX && held;
  if (use_oz) oz_slice_operand(c, X, k, st, second);
  if (c->world == 1) {
    if (use_oz) {
      oz_pass(c, E, 0, k, out, ldo, alpha, st, second);
      return;
    }
    GemmNTArgs g;
    g.A = E; g.lda = c->ldn; g.B = X; g.ldb = c->ldn;
    g.M = c->n; g.N = k; g.K = c->n; g.alpha = alpha;
    g.out = out; g.out_rs = 1; g.out_cs = ldo;
    ProfScope ps(c, PROF_EPASS, 2.0 * c->n * c->n * k, 8.0 * c->n * c->n, st);
    gemm_nt(g, gs, st);
    return;
  }
  for (int sl = 0; sl < c->nsh; ++sl) {
    const int s = c->sh0 + sl;
    double* blk = c->stage + (size_t)s * c->nloc * k;
    int64_t r0, rows;
    shard_range(c, s, &r0, &rows);
    if (rows <= 0) continue;
    if (use_oz) {
      oz_pass(c, E, s, k, blk, c->nloc, alpha, st, second);
    } else {
      ProfScope ps(c, PROF_EPASS, 2.0 * rows * c->n * k, 8.0 * rows * c->n, st);
      GemmNTArgs g;
      g.A = E + (held ? r0 - c->erow0 : r0) * c->ldn; g.lda = c->ldn; g.B = X; g.ldb = c->ldn;
      g.M = rows; g.N = k; g.K = c->n; g.alpha = alpha;
      g.out = blk; g.out_rs = 1; g.out_cs = c->nloc;
      gemm_nt(g, gs, st);
    }
  }
  if (c->virt)  // one-rank communicator: all G blocks are "this rank's" contribution
    DME_NCCL(ncclAllGather(c->stage, c->stage, (size_t)c->world * c->nloc * k, ncclDouble, c->comm, st));
  else
    DME_NCCL(ncclAllGather(c->stage + (size_t)c->rank * c->nloc * k, c->stage, (size_t)c->nloc * k,
                           ncclDouble, c->comm, st));
  for (int gr = 0; gr < c->world; ++gr) {
    int64_t r0, rows;
    shard_range(c, gr, &r0, &rows);
    if (rows > 0)
      copy_cols(out + r0, ldo, c->stage + (size_t)gr * c->nloc * k, c->nloc, rows, k, 1.0, st);
  }
}

void epass(dme_ctx* c, const double* E, const double* X, int64_t k, double* out, int64_t ldo,
           double alpha) {
  epass_on(c, E, X, k, out, ldo, alpha, c->st, c->gs);
}

// out = exp(tau A^T) X for a sparse A: Chebyshev action (cheb.h), on chip in one cluster per
// column group. Profiled as the E pass; algorithmic work per degree and column: 2 nnz + 6 n flops.
void sparse_pass(dme_ctx* c, double tau, const double* X, int64_t k, double* out, int64_t ldo,
                 cudaStream_t st) {
  if (k <= 0) return;
  c->stats.e_passes++;
  const double bytes = 16.0 * c->n * k + 12.0 * c->cop.w * CHEB_CLUSTER * c->cop.R;
  ProfScope ps(c, PROF_EPASS, 0.0, bytes, st);
  const int deg = cheb_action(c->cop, tau, X, c->ldn, k, out, ldo, 1.0, st);
  ps.r.flops = (double)deg * k * (2.0 * c->chost.nnz + 6.0 * c->n);
  if (tau == c->h) c->stats.cheb_degree = deg;
}

// out = E_tau X, tau = h (full) or h/2: the dense E pass or the sparse Chebyshev action
void eact_on(dme_ctx* c, bool full, const double* X, int64_t k, double* out, int64_t ldo,
             cudaStream_t st, GemmScratch& gs) {
  if (c->sparse) {
    sparse_pass(c, full ? c->h : c->h / 2, X, k, out, ldo, st);
    return;
  }
  epass_on(c, full ? c->E_full : c->E_half, X, k, out, ldo, 1.0, st, gs);
}
void eact(dme_ctx* c, bool full, const double* X, int64_t k, double* out, int64_t ldo) {
  eact_on(c, full, X, k, out, ldo, c->st, c->gs);
}

// Column compression of Zc (n x k) with the Riccati flow T3(tau3) optionally fused (t3).
// Single pass (options.compression = GRAM, or trunc_tol >= SPLIT_TOL): G = Zc^T Zc = W Theta W^T,
// Tm = W_kept (theta > tol theta_max), T3 fused in the eigen kernel.
// Refined (default): the FP64 Gram resolves eigenvalues only down to ~k eps theta_max, so
//   pass 1  keeps theta > SPLIT_TOL theta_max of G (accurate): W_b (k x kb);
//   pass 2  Zs = Zc (I - W_b W_b^T) explicitly (n-row product), G_s = Zs^T Zs: its eigenvalues are
//           the rest of P's spectrum resolved to ~eps^2 theta_max (the explicit columns carry an
//           absolute error ~eps sqrt(theta_max), not eps theta_max); keep mu > tol theta_max, at
//           most cap - kb: V_s;
//   Tm = [W_b | V_s] (P = Zc W_b W_b^T Zc^T + Zs Zs^T exactly, the two projectors being
//   complementary), then T3 on Tm.
// This is the paper's truncation (reduced SVD + diagonalisation, tol 1e-16 P:L331):
// every kept and dropped eigenvalue is resolved at the tolerance.
struct Compression {
  SmallArgs a;
  bool fast = false, do_compress = true, t3 = false, refine = false;
  bool fin_in_cb = false;  // refined, split first pass: FIN's work done by the queued complement
  double tau3 = 0.0;
  double* Zc = nullptr;
  int64_t k = 0;
};

void launch_eig(dme_ctx* c, SmallArgs& a, bool& fast) {
  fast = a.compress && a.k <= FAST_K_MAX && !c->force_jacobi;
  ProfScope ps(c, PROF_SMALL);
  if (fast && a.k >= EIG_SPLIT_MIN) eig_split(a, c->st);
  else if (fast) eig_fast(a, c->st);
  else compress_t3(a, c->st);
}

// Launch the Gram matrix (extended by B when T3 is fused: the B columns are copied next to the
// factor, so G_ext = [Zc, B]^T [Zc, B] yields G and H = Zc^T B in one pass) and the first eigen
// pass. Zc must have KMAX columns of capacity.
void compress_launch(dme_ctx* c, double* Zc, int64_t k, bool t3, double tau3, bool do_compress,
                     Compression& cp, cudaEvent_t after_gram = nullptr,
                     double* Tm_out = nullptr, bool gram_ready = false) {
  DME_REQUIRE(k <= KMAX && (!t3 || k + c->m <= KMAX), DME_ERR_DIM,
              "factor width exceeds the small-system limit (224)");
  c->stats.compressions += do_compress ? 1 : 0;
  cp = Compression();
  cp.Zc = Zc; cp.k = k; cp.t3 = t3; cp.tau3 = tau3; cp.do_compress = do_compress;
  const double tol = c->opt.trunc_tol * c->tol_scale;
  // (the tail pass needs the complement basis in one CTA's shared memory: k <= FAST_K_MAX; wider
  // concatenations -- T4 at rank > 53, ladder rungs at q > 80 -- use the single Gram pass)
  cp.refine = do_compress && c->refine && tol < SPLIT_TOL && k <= FAST_K_MAX;
  SmallArgs& a = cp.a;
  if (gram_ready) {  // G (and H = G + k KMAX) assembled by the caller (gram_congruence)
    DME_REQUIRE(do_compress && t3, DME_ERR_CONFIG, "assembled Gram path needs compress + T3");
    a.H = c->G + k * KMAX;
  } else if (do_compress) {
    const int64_t kk = t3 ? k + c->m : k;
    if (t3) {
      ProfScope pc(c, 4);
      copy_cols(Zc + k * c->ldn, c->ldn, c->Bcol, c->ldn, c->n, c->m, 1.0, c->st);
    }
    ProfScope ps(c, PROF_GRAM);
    GemmNTArgs g;
    g.A = Zc; g.lda = c->ldn; g.B = Zc; g.ldb = c->ldn;
    g.M = kk; g.N = kk; g.K = c->n;
    g.out = c->G; g.out_rs = 1; g.out_cs = KMAX;
    gemm_nt(g, c->gs, c->st);
    a.H = c->G + k * KMAX;
  } else if (t3) {
    ProfScope ps(c, PROF_GRAM);
    GemmNTArgs g;
    g.A = Zc; g.lda = c->ldn; g.B = c->Bcol; g.ldb = c->ldn;
    g.M = k; g.N = c->m; g.K = c->n;
    g.out = c->H; g.out_rs = 1; g.out_cs = KMAX;
    gemm_nt(g, c->gs, c->st);
    a.H = c->H;
  }
  if (after_gram) DME_CUDA(cudaEventRecord(after_gram, c->st));
  a.k = (int)k;
  a.compress = do_compress ? 1 : 0;
  a.G = c->G; a.ldg = KMAX;
  a.tol = cp.refine ? SPLIT_TOL : (c->refine ? tol : std::max(tol, GRAM_FLOOR));
  a.cap = c->rank_cap;
  a.t3 = (t3 && !cp.refine) ? 1 : 0;
  a.m = (int)c->m;
  a.ldh = KMAX;
  a.LRinv = c->LRinv;
  a.tau = tau3;
  a.Tm = Tm_out ? Tm_out : c->Tm; a.ldt = KMAX;
  a.V = c->Vg; a.ldv = KMAX;
  a.Es = c->Es;
  static const int msec_p = [] {
    const char* e = std::getenv("DME_MSEC_P");
    const int v = e ? std::atoi(e) : 128;
    return v < 1 ? 1 : (v > 512 ? 512 : v);
  }();
  a.msec_p = msec_p;
  a.r_out = c->r_dev;
  a.stats = c->sstats;
  if (c->hmap_dev) {
    a.map = c->hmap_dev;
    a.map_seq = ++c->map_seq;
  }
  // refined + split first pass (t3 = 0): no FIN kernel, the complement basis queued right behind
  // the pass checks, publishes kb and builds U in one launch (compress_finish)
  cp.fin_in_cb = cp.refine && !c->no_fused_fin && k >= EIG_SPLIT_MIN && k <= FAST_K_MAX &&
                 !c->force_jacobi && complement_dev_available((int)k);
  a.skip_fin = cp.fin_in_cb ? 1 : 0;
  launch_eig(c, a, cp.fast);
}

// Wait until the small kernel launched with sequence number `seq` has published its rank in the
// host-mapped record (spinning on pinned memory: no D2H copy, no stream synchronisation on the
// step's critical path); the stream is polled now and then so a failed launch surfaces as an error.
void wait_published(dme_ctx* c, int seq) {
  volatile HostMap* m = c->hmap;
  for (int64_t spins = 1; m->seq != seq; ++spins) {
    if ((spins & 1023) == 0) {
      const cudaError_t q = cudaStreamQuery(c->st);
      if (q == cudaSuccess) {
        if (m->seq == seq) break;
        throw DmeError(DME_ERR_CUDA, "small kernel finished without publishing its rank");
      }
      if (q != cudaErrorNotReady) DME_CUDA(q);
    }
  }
  std::atomic_thread_fence(std::memory_order_acquire);
}

// Wait for an eigen pass (main stream), fall back to Jacobi if the fast path refused; the pass's
// stats land in c->last_st.
int64_t eig_finish(dme_ctx* c, const SmallArgs& a, bool fast) {
  int r_host = 0;
  double* st_host = c->last_st;
  auto fetch = [&](const SmallArgs& x) {
    if (x.map) {
      wait_published(c, x.map_seq);
      r_host = c->hmap->r;
      for (int i = 0; i < 5; ++i) st_host[i] = c->hmap->stats[i];
    } else {
      DME_CUDA(cudaMemcpyAsync(&r_host, c->r_dev, sizeof(int), cudaMemcpyDeviceToHost, c->st));
      DME_CUDA(cudaMemcpyAsync(st_host, c->sstats, 5 * sizeof(double), cudaMemcpyDeviceToHost, c->st));
      sync(c);
    }
  };
  fetch(a);
  if (fast && r_host < 0) {  // near-degenerate cluster: orthogonality check failed -> Jacobi
    c->stats.eig_fallbacks++;
    SmallArgs b = a;
    if (b.map) b.map_seq = ++c->map_seq;
    {
      ProfScope ps(c, PROF_SMALL);
      compress_t3(b, c->st);
    }
    fetch(b);
  }
  return r_host;
}

// Finish a compression: first pass, then (refined) the tail pass and T3. zc_ready: an event after
// which Zc is complete (the pipeline writes part of it on the second stream), or null.
int64_t compress_finish(dme_ctx* c, Compression& cp, cudaEvent_t zc_ready = nullptr) {
  // refined: the complement basis of the first pass's kept vectors is queued before the host has
  // seen kb (the kernel reads the published rank on the device; a Jacobi fallback publishes -1,
  // turning it into a no-op, and it is queued again below with the host's kb)
  bool cb_queued = false;
  if (cp.refine && cp.fast) {
    ProfScope ps(c, PROF_SMALL);
    cb_queued = complement_basis_dev(cp.a.Tm, KMAX, (int)cp.k, c->r_dev, c->Us, KMAX, c->st,
                                     cp.fin_in_cb ? &cp.a : nullptr);
    DME_REQUIRE(cb_queued || !cp.fin_in_cb, DME_ERR_CUDA, "first pass without FIN needs the complement");
  }
  const int64_t fb0 = c->stats.eig_fallbacks;
  const int64_t kb = eig_finish(c, cp.a, cp.fast);
  if (c->stats.eig_fallbacks != fb0) cb_queued = false;
  if (!cp.refine) {
    if (cp.do_compress) c->stats.last_drop = c->last_st[2];
    return kb;
  }
  const double tmax = c->last_st[1];
  int64_t r = kb;
  double drop = (kb < cp.k) ? SPLIT_TOL : 0.0;
  const int64_t k = cp.k;
  const int cap = cp.a.cap;
  int64_t ks = 0, s = 0;
  bool tail_done = false;
  if (kb < k && tmax > 0.0 && kb < cap) {
    // U (k x s): orthonormal basis of the complement of span(W_b); Zs = Zc U (n x s), Gs = Zs^T Zs
    s = k - kb;
    if (!cb_queued) {
      ProfScope ps(c, PROF_SMALL);
      complement_basis(cp.a.Tm, KMAX, (int)k, (int)kb, c->Us, KMAX, c->st);
    }
    if (zc_ready) DME_CUDA(cudaStreamWaitEvent(c->st, zc_ready, 0));
    // fused: Zs rows are formed chunk by chunk in shared memory, never stored
    bool fused;
    {
      ProfScope ps(c, PROF_GRAM);
      fused = !c->no_proj_gram &&
              proj_gram(cp.Zc, c->ldn, c->n, (int)k, c->Us, KMAX, (int)s, c->Gs, KMAX, c->gs.partial,
                        GemmScratch::partial_doubles(c->gs.max_grid), c->st);
    }
    if (!fused) {
      {
        ProfScope ps(c, PROF_APPLY);
        tall_small(cp.Zc, c->ldn, c->Us, KMAX, c->Zs, c->ldn, c->n, s, k, c->st);
      }
      ProfScope ps(c, PROF_GRAM);
      GemmNTArgs g;
      g.A = c->Zs; g.lda = c->ldn; g.B = c->Zs; g.ldb = c->ldn;
      g.M = s; g.N = s; g.K = c->n;
      g.out = c->Gs; g.out_rs = 1; g.out_cs = KMAX;
      gemm_nt(g, c->gs, c->st);
    }
    SmallArgs b = cp.a;
    b.k = (int)s;
    b.G = c->Gs;
    b.t3 = 0;
    b.tol = c->opt.trunc_tol * c->tol_scale;
    b.ref_max = tmax;
    b.cap = cap - (int)kb;
    b.Tm = c->Ts;
    if (b.map) b.map_seq = ++c->map_seq;
    bool fast2 = false;
    // split tail pass: no FIN kernel; the tail assembly checks, publishes and assembles in one launch
    const int ks_bound0 = std::min<int>(b.cap, (int)s);
    const bool fin_fused = !c->no_fused_fin && s >= EIG_SPLIT_MIN && s <= FAST_K_MAX && !c->force_jacobi &&
                           tail_assemble_smem((int)k, (int)c->m, (int)s, (int)kb, ks_bound0) <=
                               (size_t)SMALL_SMEM_MAX;
    b.skip_fin = fin_fused ? 1 : 0;
    launch_eig(c, b, fast2);
    // the tail assembly (+ T3) is queued right behind the eigen pass and reads ks on the device,
    // so the critical stream does not idle through this host round trip; a Jacobi fallback of the
    // pass (ks < 0 published) turns it into a no-op and it is queued again below
    const int ks_bound = std::min<int>(b.cap, (int)s);
    const bool dev_ks = fast2 && tail_assemble_smem((int)k, (int)c->m, (int)s, (int)kb, ks_bound) <=
                                     (size_t)SMALL_SMEM_MAX;
    if (dev_ks) {
      SmallArgs t = cp.a;
      t.k = (int)k;
      t.t3 = cp.t3 ? 1 : 0;
      ProfScope ps(c, PROF_SMALL);
      tail_assemble_t3(t, c->Us, KMAX, (int)s, c->Ts, KMAX, (int)kb, ks_bound, c->st, c->r_dev,
                       fin_fused ? &b : nullptr);
    }
    const int64_t pubs = c->stats.eig_fallbacks;
    ks = eig_finish(c, b, fast2);
    r = kb + ks;
    drop = c->last_st[2];
    tail_done = dev_ks && c->stats.eig_fallbacks == pubs;
    if (std::getenv("DME_DEBUG_REFINE"))
      std::fprintf(stderr, "refine: k %lld kb %lld s %lld ks %lld\n", (long long)k, (long long)kb,
                   (long long)s, (long long)ks);
  }
  if (!tail_done && (ks > 0 || (cp.t3 && r > 0))) {  // Tm[:, kb:r] = U V_s, then T3 on Tm
    SmallArgs t = cp.a;
    t.k = (int)k;
    t.t3 = cp.t3 ? 1 : 0;
    ProfScope ps(c, PROF_SMALL);
    tail_assemble_t3(t, c->Us, KMAX, (int)s, c->Ts, KMAX, (int)kb, (int)ks, c->st);
  }
  c->stats.last_drop = drop;
  return r;
}

// Compress the factor Zc (n x k, col-major ldn) into out (n x r); optionally fuse T3(tau3).
int64_t compress(dme_ctx* c, double* Zc, int64_t k, double* out, bool t3, double tau3,
                 bool do_compress = true) {
  NvtxRange nvtx_("dme::compress");
  if (k <= 0) return 0;
  Compression cp;
  compress_launch(c, Zc, k, t3, tau3, do_compress, cp);
  const int64_t r_host = compress_finish(c, cp);
  if (r_host > 0) {
    ProfScope ps(c, PROF_APPLY);
    tall_small(Zc, c->ldn, cp.a.Tm, KMAX, out, c->ldn, c->n, r_host, k, c->st);
  }
  if (c->profile) drain_profile(c);
  return r_host;
}

// ------------------------------------------------------------------ flows on the state Z
void swapZ(dme_ctx* c) { std::swap(c->Z, c->Ztmp); }

void flow_T1(dme_ctx* c, double tau) {
  NvtxRange nvtx_("dme::T1");
  eact(c, tau == c->h, c->Z, c->r, c->Ztmp, c->ldn);
  swapZ(c);
}

void finish_compress(dme_ctx* c, double* Zc, int64_t k, bool t3, double tau3) {
  c->r = compress(c, Zc, k, c->Ztmp, t3, tau3);
  swapZ(c);
  c->stats.max_rank = std::max<int64_t>(c->stats.max_rank, c->r);
}

void flow_T2(dme_ctx* c, double tau, bool t3, double tau3) {
  NvtxRange nvtx_("dme::T2");
  copy_cols(c->Zc2, c->ldn, c->Z, c->ldn, c->n, c->r, 1.0, c->st);
  copy_cols(c->Zc2 + c->r * c->ldn, c->ldn, c->LQ, c->ldn, c->n, c->p, std::sqrt(tau), c->st);
  finish_compress(c, c->Zc2, c->r + c->p, t3, tau3);
}

void flow_T12(dme_ctx* c, double tau, bool t3, double tau3) {
  NvtxRange nvtx_("dme::T12");
  const bool full = (tau == c->h);
  double* Zc = full ? c->Zc12f : c->Zc12h;
  const int64_t q = full ? c->qf : c->qh;
  eact(c, full, c->Z, c->r, Zc + q * c->ldn, c->ldn);
  finish_compress(c, Zc, q + c->r, t3, tau3);
}

void flow_T3(dme_ctx* c, double tau) {
  NvtxRange nvtx_("dme::T3");
  if (c->r == 0) return;
  const int64_t r = compress(c, c->Z, c->r, c->Ztmp, true, tau, /*do_compress=*/false);
  (void)r;
  swapZ(c);
}

// out = alpha S X for the bilinear flow: the dense S through the E-pass GEMM (row-sharded like E),
// or the CSR S by a sparse x skinny product (every rank all rows: n nnz-sized work, no collective)
void s_pass(dme_ctx* c, const double* X, int64_t k, double* out, int64_t ldo, double alpha) {
  if (k <= 0) return;
  if (!c->sparse_S) {
    epass(c, c->S, X, k, out, ldo, alpha);
    return;
  }
  ProfScope ps(c, PROF_EPASS, 2.0 * c->S_nnz * k, 12.0 * c->S_nnz + 16.0 * c->n * k, c->st);
  spmm_csr(c->S_rp, c->S_ci, c->S_v, c->n, X, c->ldn, k, out, ldo, alpha, c->st);
}

void flow_T4(dme_ctx* c, double tau, int order, bool t3, double tau3) {
  NvtxRange nvtx_("dme::T4");
  if (c->r == 0) return;
  const int64_t r = c->r, ld = c->ldn;
  copy_cols(c->Zc2, ld, c->Z, ld, c->n, r, 1.0, c->st);
  s_pass(c, c->Z, r, c->Zc2 + r * ld, ld, std::sqrt(tau));                         // sqrt(tau) S L
  int64_t k = 2 * r;
  if (order == 2) {                                                                 // tau/sqrt2 S^2 L
    s_pass(c, c->Zc2 + r * ld, r, c->Zc2 + 2 * r * ld, ld, std::sqrt(tau) / std::sqrt(2.0));
    k = 3 * r;
  }
  finish_compress(c, c->Zc2, k, t3, tau3);
}

struct Op {
  int flow;
  double tau;
};

std::vector<Op> step_sequence(dme_scheme scheme, dme_composition comp, double h) {
  std::vector<int> fl;
  switch (comp) {
    case DME_F1F2: fl = {0, 1}; break;
    case DME_F12: fl = {5}; break;
    case DME_F12F3: fl = {5, 2}; break;
    case DME_F1F2F3: fl = {0, 1, 2}; break;
    case DME_F1F3F2: fl = {0, 2, 1}; break;
    case DME_F12F4: fl = {5, 3}; break;
    case DME_F1F2F4: fl = {0, 1, 3}; break;
    case DME_F1F4F2: fl = {0, 3, 1}; break;
    case DME_F12F3F4: fl = {5, 2, 3}; break;
    case DME_F1F2F3F4: fl = {0, 1, 2, 3}; break;
    default: throw DmeError(DME_ERR_CONFIG, "unknown composition");
  }
  std::vector<Op> seq;
  if (scheme == DME_LIE) {
    for (int f : fl) seq.push_back({f == 3 ? 4 : f, h});  // T4 by explicit Euler under Lie
  } else if (scheme == DME_STRANG) {
    if (fl.size() == 1) {
      seq.push_back({fl[0], h});
    } else {
      for (size_t i = 0; i + 1 < fl.size(); ++i) seq.push_back({fl[i], h / 2});
      seq.push_back({fl.back(), h});
      for (size_t i = fl.size() - 1; i-- > 0;) seq.push_back({fl[i], h / 2});
    }
  } else {
    throw DmeError(DME_ERR_CONFIG, "unknown scheme");
  }
  return seq;
}

void check_capable(dme_ctx* c, const std::vector<Op>& seq) {
  for (const Op& o : seq) {
    if (o.flow == DME_FLOW_T3) DME_REQUIRE(c->dre, DME_ERR_CONFIG, "composition uses F3 but the problem has no B");
    if (o.flow == DME_FLOW_T4_MIDPOINT || o.flow == DME_FLOW_T4_EULER)
      DME_REQUIRE(c->has_S, DME_ERR_CONFIG, "composition uses F4 but the problem has no S");
    if (o.flow == DME_FLOW_T2) DME_REQUIRE(c->p >= 0, DME_ERR_CONFIG, "bad p");
  }
}

// Execute a sequence; a compressing flow immediately followed by T3 runs T3 fused.
void run_sequence(dme_ctx* c, const std::vector<Op>& seq) {
  for (size_t i = 0; i < seq.size(); ++i) {
    const Op& o = seq[i];
    const bool next_t3 = i + 1 < seq.size() && seq[i + 1].flow == DME_FLOW_T3;
    const double tau3 = next_t3 ? seq[i + 1].tau : 0.0;
    switch (o.flow) {
      case DME_FLOW_T1: flow_T1(c, o.tau); break;
      case DME_FLOW_T2: flow_T2(c, o.tau, next_t3, tau3); if (next_t3) ++i; break;
      case DME_FLOW_T3: flow_T3(c, o.tau); break;
      case DME_FLOW_T4_MIDPOINT: flow_T4(c, o.tau, 2, next_t3, tau3); if (next_t3) ++i; break;
      case DME_FLOW_T4_EULER: flow_T4(c, o.tau, 1, next_t3, tau3); if (next_t3) ++i; break;
      case DME_FLOW_T12: flow_T12(c, o.tau, next_t3, tau3); if (next_t3) ++i; break;
      default: throw DmeError(DME_ERR_CONFIG, "unknown flow");
    }
  }
}

// Pipelined body of the merged Strang F12F3 steps: nb x [T12(h) T3(h)] (compression + fused T3).
// Step t: Zc_t = [L_I(h) | Y_t], G_t = Zc_t^T Zc_t, eigen-compression -> Tm_t (k_t x r_t),
// Z_t = Zc_t Tm_t, Y_{t+1} = E_h Z_t = [E_h L_I(h) | E_h Y_t] Tm_t = LA_t Tm_t.
// The Gram of the next step is a congruence of a Gram that does not depend on Tm_t:
//   GB_t = [L_I(h) | B | LA_t],  Ghat_t = GB_t^T GB_t,
//   G_{t+1} = [[Ghat_II, Ghat_I,LA Tm_t], [Tm_t^T Ghat_LA,I, Tm_t^T Ghat_LA,LA Tm_t]], H likewise,
// so the critical path is eigen-compression_t -> congruence (one small kernel) ->
// eigen-compression_{t+1}, while the second stream runs Y_{t+1} = LA_t Tm_t (tall-small), the E pass
// E_h Y_{t+1} and Ghat_{t+1} (n-row work) underneath. Exact reassociation of the same products
// (rounding differs only); only the last step materialises the state Z.
void run_f12f3_body(dme_ctx* c, int64_t nb, double h) {
  NvtxRange nvtx_("dme::F12F3.pipelined");
  if (nb <= 0) return;
  const int64_t ld = c->ldn, q = c->qf, n = c->n, m = c->m;
  double* Zc = c->Zc12f;
  double* Tmb[2] = {c->Tm, c->Tm2};
  eact(c, true, c->Z, c->r, Zc + q * ld, ld);  // Y_0 = E_h Z
  const int rc = (int)std::min<int64_t>(c->rank_cap, n);  // bound on every rank of the body
  const bool pipe = c->lookahead && nb > 1 && 2 * q + m + rc <= KMAX &&
                    gram_congruence_smem((int)q, (int)m, (int)(q + rc), rc) <= 220 * 1024;
  int64_t r_prev = c->r;  // columns of Y_t
  Compression cp;
  // step 0: direct Gram of Zc_0 (main stream), eigen-compression 0
  compress_launch(c, Zc, q + r_prev, true, h, true, cp, c->ev_gram, Tmb[0]);
  if (pipe) {  // second stream: E_h Y_0 into GB, Ghat_0
    DME_CUDA(cudaStreamWaitEvent(c->st2, c->ev_gram, 0));
    eact_on(c, true, Zc + q * ld, r_prev, c->GB + (2 * q + m) * ld, ld, c->st2, c->gs2);
    GemmNTArgs g;
    g.A = c->GB; g.lda = ld; g.B = c->GB; g.ldb = ld;
    g.M = g.N = 2 * q + m + r_prev; g.K = n;
    g.out = c->Ghat; g.out_rs = 1; g.out_cs = KMAX;
    gemm_nt(g, c->gs2, c->st2);
    DME_CUDA(cudaEventRecord(c->ev_ghat, c->st2));
  }
  int64_t rn = compress_finish(c, cp);
  DME_CUDA(cudaEventRecord(c->ev_tm, c->st));  // Tm_0 final (after the tail pass and T3)
  for (int64_t it = 0; it < nb; ++it) {
    NvtxRange nvtx_step("dme::step");
    double* Tm_cur = Tmb[it & 1];
    const int64_t kp = q + r_prev;  // columns of Zc_t = columns of LA_t
    const bool last = it + 1 == nb;
    if (!last && pipe) {
      // critical path: congruence -> eigen-compression t+1 (first pass)
      DME_CUDA(cudaStreamWaitEvent(c->st, c->ev_ghat, 0));
      {
        ProfScope ps(c, PROF_GRAM);
        gram_congruence(c->Ghat, KMAX, (int)q, (int)m, (int)kp, Tm_cur, KMAX, (int)rn, c->G, KMAX,
                        c->st);
      }
      DME_CUDA(cudaEventRecord(c->ev_cong, c->st));
      Compression cn;
      compress_launch(c, Zc, q + rn, true, h, true, cn, nullptr, Tmb[(it + 1) & 1], true);
      // underneath: Y_{t+1} = LA_t Tm_t, E_h Y_{t+1}, Ghat_{t+1}
      DME_CUDA(cudaStreamWaitEvent(c->st2, c->ev_tm, 0));
      if (rn > 0) {
        ProfScope ps(c, PROF_APPLY, 0, 0, c->st2);
        tall_small(c->GB + (q + m) * ld, ld, Tm_cur, KMAX, Zc + q * ld, ld, n, rn, kp, c->st2);
      }
      DME_CUDA(cudaEventRecord(c->ev_zc, c->st2));  // Zc_{t+1} = [L_I | Y_{t+1}] complete
      if (it + 2 < nb) {  // Ghat_{t+1} is needed only if step t+2 exists
        eact_on(c, true, Zc + q * ld, rn, c->GB + (2 * q + m) * ld, ld, c->st2, c->gs2);
        DME_CUDA(cudaStreamWaitEvent(c->st2, c->ev_cong, 0));
        GemmNTArgs g;
        g.A = c->GB; g.lda = ld; g.B = c->GB; g.ldb = ld;
        g.M = g.N = 2 * q + m + rn; g.K = n;
        g.out = c->Ghat; g.out_rs = 1; g.out_cs = KMAX;
        gemm_nt(g, c->gs2, c->st2);
        DME_CUDA(cudaEventRecord(c->ev_ghat, c->st2));
      }
      r_prev = rn;
      rn = compress_finish(c, cn, c->ev_zc);
      DME_CUDA(cudaEventRecord(c->ev_tm, c->st));
    } else if (!last) {  // no pipeline: Y_{t+1} = E_h (Zc_t Tm_t), direct Gram
      if (rn > 0) {
        ProfScope ps(c, PROF_APPLY);
        tall_small(Zc, ld, Tm_cur, KMAX, c->Ztmp, ld, n, rn, kp, c->st);
      }
      eact(c, true, c->Ztmp, rn, Zc + q * ld, ld);
      r_prev = rn;
      Compression cn;
      compress_launch(c, Zc, q + rn, true, h, true, cn, nullptr, Tmb[(it + 1) & 1]);
      rn = compress_finish(c, cn);
    } else {  // last step: materialise Z = Zc_t Tm_t (Y_t was written on the second stream)
      if (pipe) {
        DME_CUDA(cudaEventRecord(c->ev_y, c->st2));
        DME_CUDA(cudaStreamWaitEvent(c->st, c->ev_y, 0));
      }
      if (rn > 0) {
        ProfScope ps(c, PROF_APPLY);
        tall_small(Zc, ld, Tm_cur, KMAX, c->Ztmp, ld, n, rn, kp, c->st);
      }
      swapZ(c);
    }
    c->r = rn;
    c->stats.max_rank = std::max<int64_t>(c->stats.max_rank, c->r);
    c->stats.steps++;
    if (c->profile) drain_profile(c);
  }
}

void matmul_sq(dme_ctx* c, const double* X, const double* Y, double* out) {
  // out = X * Y  (n x n row-major): B operand rows = columns of Y = rows of Y^T.
  // Symmetric A: every factor here is a polynomial in the symmetric X0 (or E = r(X0)), so Y^T = Y
  // and X Y is symmetric: only the upper tile triangle is computed, then mirrored.
  const bool sym = c->symA;
  if (!sym) transpose_rect(Y, c->n, c->n, c->ldn, c->BT, c->ldn, c->st);
  if (c->oz_init) {
    // int8 digit slicing of both operands (ozaki.h): rows of X, rows of Y^T; the E-digit buffers
    // serve as scratch (E is sliced after the last product)
    const int64_t n = c->n, ldk = c->ozld;
    oz_slice_rows(X, c->ldn, n, n, c->ozEh, ldk, n * ldk, c->exEh, c->ozpm, c->st);
    oz_slice_rows(sym ? Y : c->BT, c->ldn, n, n, c->ozEf, ldk, n * ldk, c->exEf, c->ozpm, c->st);
    OzGemmArgs g;
    g.A = c->ozEh; g.eA = c->exEh; g.lda = ldk; g.a_slice_stride = n * ldk;
    g.B = c->ozEf; g.eB = c->exEf; g.ldb = ldk; g.b_slice_stride = n * ldk;
    g.M = n; g.N = n; g.K = n; g.alpha = 1.0;
    g.out = out; g.out_rs = c->ldn; g.out_cs = 1;
    g.tiles = sym ? c->oz_tiles_up : c->oz_tiles_all;
    g.ntiles = sym ? c->ntiles_up : c->ntiles_all;
    g.round_robin = true;
    oz_gemm(g, c->ozs, c->st);
  } else {
    GemmNTArgs g;
    g.A = X; g.lda = c->ldn; g.B = sym ? Y : c->BT; g.ldb = c->ldn;
    g.M = c->n; g.N = c->n; g.K = c->n;
    g.out = out; g.out_rs = c->ldn; g.out_cs = 1;
    g.sym_upper = sym;
    gemm_nt(g, c->gs, c->st);
  }
  if (sym) mirror_lower(out, c->n, c->ldn, false, c->st);
}

// L_I(2w) = compress([L_I(w), E_w L_I(w)])  (exact doubling of the composite rule, reading G6);
// E_w is the dense Ew, or (sparse A) the Chebyshev action with tau = w
void ladder_double(dme_ctx* c, double* LI, int64_t& q, const double* Ew, double w) {
  NvtxRange nvtx_("dme::init.quadrature_rung");
  if (q == 0) return;
  DME_REQUIRE(2 * q <= KMAX, DME_ERR_DIM, "quadrature factor rank exceeds 112");
  if (c->sparse || c->cheb_e) sparse_pass(c, w, LI, q, LI + q * c->ldn, c->ldn, c->st);
  else epass(c, Ew, LI, q, LI + q * c->ldn, c->ldn, 1.0);
  const int64_t qn = compress(c, LI, 2 * q, c->Ztmp, false, 0.0);
  copy_cols(LI, c->ldn, c->Ztmp, c->ldn, c->n, qn, 1.0, c->st);
  q = qn;
}

void init_all(dme_ctx* c, const dme_problem* pr) {
  NvtxRange nvtx_("dme::init");
  const int64_t n = c->n, ld = c->ldn;
  cudaStream_t st = c->st;
  DME_CUDA(cudaMemsetAsync(c->gs.counters, 0, sizeof(int) * c->gs.max_tiles, st));
  DME_CUDA(cudaMemsetAsync(c->gs2.counters, 0, sizeof(int) * c->gs2.max_tiles, st));
  // the Stream-K fixup counters of the int8 E pass (the workspace is uninitialised caller memory)
  if (c->oz)
    for (OzScratch* o : {&c->ozs, &c->ozs2})
      DME_CUDA(cudaMemsetAsync(o->counters, 0, sizeof(int) * o->max_tiles, st));
  if (c->oz_init) {
    DME_CUDA(cudaMemcpyAsync(c->oz_tiles_up, c->h_tiles_up.data(), c->h_tiles_up.size() * sizeof(int2),
                             cudaMemcpyHostToDevice, st));
    DME_CUDA(cudaMemcpyAsync(c->oz_tiles_all, c->h_tiles_all.data(),
                             c->h_tiles_all.size() * sizeof(int2), cudaMemcpyHostToDevice, st));
  }
  // ---------------------------------------------------------------- upload (H2D boundary)
  // A and S: host memory (pageable or pinned) or, with options.big_inputs_on_device, device memory
  const cudaMemcpyKind kbig = c->opt.big_inputs_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
  if (c->sparse) {  // partitioned ELL of A^T (built on the host from the CSR by cheb_prepare)
    DME_CUDA(cudaMemcpyAsync(c->cop.val, c->chost.val.data(), c->chost.val.size() * 8,
                             cudaMemcpyHostToDevice, st));
    DME_CUDA(cudaMemcpyAsync(c->cop.idx, c->chost.idx.data(), c->chost.idx.size() * 4,
                             cudaMemcpyHostToDevice, st));
    DME_CUDA(cudaMemcpyAsync(c->cop.rptr, c->chost.rptr.data(), c->chost.rptr.size() * 4,
                             cudaMemcpyHostToDevice, st));
    DME_CUDA(cudaMemcpyAsync(c->cop.rent, c->chost.rent.data(), c->chost.rent.size() * 4,
                             cudaMemcpyHostToDevice, st));
    if (!c->chost.push.empty())
      DME_CUDA(cudaMemcpyAsync(c->cop.push, c->chost.push.data(), c->chost.push.size() * 4,
                               cudaMemcpyHostToDevice, st));
  } else {
    DME_CUDA(cudaMemcpy2DAsync(c->Aup, ld * 8, pr->A, n * 8, n * 8, n, kbig, st));
  }
  if (c->has_S && !c->sparse_S)
    DME_CUDA(cudaMemcpy2DAsync(c->S, ld * 8, pr->S, n * 8, n * 8, n, kbig, st));
  if (c->sparse_S) {  // (validated on the host: indices in range, finite values)
    std::vector<int> rp32(n + 1), ci32(std::max<int64_t>(c->S_nnz, 1));
    for (int64_t i = 0; i <= n; ++i) rp32[i] = (int)pr->S_rowptr[i];
    for (int64_t e = 0; e < c->S_nnz; ++e) ci32[e] = pr->S_colind[e];
    DME_CUDA(cudaMemcpyAsync(c->S_rp, rp32.data(), (n + 1) * sizeof(int), cudaMemcpyHostToDevice, st));
    if (c->S_nnz > 0) {
      DME_CUDA(cudaMemcpyAsync(c->S_ci, ci32.data(), c->S_nnz * sizeof(int), cudaMemcpyHostToDevice, st));
      DME_CUDA(cudaMemcpyAsync(c->S_v, pr->S_values, c->S_nnz * 8, cudaMemcpyHostToDevice, st));
    }
    sync(c);  // (the pageable staging vectors die here)
  }
  // mass matrix (Example 4): A <- A M^-1, C <- C M^-1 by a dense LU of M
  const bool mass = pr->M != nullptr;
  if (mass) {
    int mflags[2] = {0, 0};
    DME_CUDA(cudaMemcpy2DAsync(c->X4, ld * 8, pr->M, n * 8, n * 8, n, kbig, st));
    DME_CUDA(cudaMemsetAsync(c->r_dev, 0, 2 * sizeof(int), st));
    check_square(c->X4, n, ld, c->r_dev, st);
    DME_CUDA(cudaMemcpyAsync(mflags, c->r_dev, 2 * sizeof(int), cudaMemcpyDeviceToHost, st));
    sync(c);
    DME_REQUIRE(mflags[0] == 0, DME_ERR_INVALID, "M has non-finite entries");
    lu_solve_right(c->X4, c->Aup, n, ld, c->BT, c->lu_scr, c->gs, st, c->norm_dev + 2);
    double mp = 0;
    DME_CUDA(cudaMemcpyAsync(&mp, c->norm_dev + 2, 8, cudaMemcpyDeviceToHost, st));
    sync(c);
    DME_REQUIRE(std::isfinite(mp) && mp > 0.0, DME_ERR_NUMERIC, "LU of M hit a zero pivot");
    if (c->p > 0) {  // rows of [C; 0] (n x n) times M^-1
      DME_CUDA(cudaMemcpy2DAsync(c->X4, ld * 8, pr->M, n * 8, n * 8, n, kbig, st));
      DME_CUDA(cudaMemsetAsync(c->X6, 0, (size_t)n * ld * 8, st));
      DME_CUDA(cudaMemcpy2DAsync(c->X6, ld * 8, pr->C, n * 8, n * 8, c->p, cudaMemcpyHostToDevice, st));
      lu_solve_right(c->X4, c->X6, n, ld, c->BT, c->lu_scr, c->gs, st, c->norm_dev + 2);
    }
  }
  // device-side validation of the big inputs: finiteness, and the exact symmetry of A that
  // enables the symmetric Padé products
  {
    int flags_host[4] = {0, 0, 0, 0};
    DME_CUDA(cudaMemsetAsync(c->r_dev, 0, 4 * sizeof(int), st));
    if (!c->sparse)  // (a sparse A was validated on the host by cheb_prepare)
      check_square(c->Aup, n, ld, c->r_dev, st);         // r_dev[0]: non-finite, r_dev[1]: asymmetric
    if (c->has_S && !c->sparse_S) check_square(c->S, n, ld, c->r_dev + 2, st);
    DME_CUDA(cudaMemcpyAsync(flags_host, c->r_dev, 4 * sizeof(int), cudaMemcpyDeviceToHost, st));
    sync(c);
    DME_REQUIRE(flags_host[0] == 0, DME_ERR_INVALID, "A has non-finite entries");
    DME_REQUIRE(flags_host[2] == 0, DME_ERR_INVALID, "S has non-finite entries");
    c->symA = flags_host[1] == 0;
  }
  if (c->p > 0) {  // C (p x n row-major): row i of C = column i of L_Q = C^T
    if (mass)
      DME_CUDA(cudaMemcpy2DAsync(c->LQ, ld * 8, c->X6, ld * 8, n * 8, c->p, cudaMemcpyDeviceToDevice, st));
    else
      DME_CUDA(cudaMemcpy2DAsync(c->LQ, ld * 8, pr->C, n * 8, n * 8, c->p, cudaMemcpyHostToDevice, st));
  }
  if (c->m > 0) {
    DME_CUDA(cudaMemcpyAsync(c->Wa, pr->B, n * c->m * 8, cudaMemcpyHostToDevice, st));
    rowmajor_to_colmajor(c->Bcol, ld, c->Wa, c->m, n, c->m, st);
    DME_CUDA(cudaMemcpyAsync(c->LRinv, c->lrinv_host.data(), c->m * c->m * 8, cudaMemcpyHostToDevice, st));
  }
  if (c->r0 > 0) {
    DME_CUDA(cudaMemcpyAsync(c->Yn, pr->L0, n * c->r0 * 8, cudaMemcpyHostToDevice, st));
    rowmajor_to_colmajor(c->L0d, ld, c->Yn, c->r0, n, c->r0, st);
    std::vector<double> D0(c->r0 * c->r0, 0.0);
    for (int64_t i = 0; i < c->r0; ++i)
      for (int64_t j = 0; j < c->r0; ++j)
        D0[i * c->r0 + j] = pr->D0 ? pr->D0[i * c->r0 + j] : (i == j ? 1.0 : 0.0);
    DME_CUDA(cudaMemcpyAsync(c->D0d, D0.data(), D0.size() * 8, cudaMemcpyHostToDevice, st));
    sync(c);
  }
  // ---------------------------------------------------------------- scaling: s from ||(h/2) A^T||_1
  double nrm = 0;
  if (c->sparse) {
    nrm = c->chost.norm1;
  } else {
    rowabs_max(c->Aup, n, ld, c->red_scratch, c->norm_dev, st);
    DME_CUDA(cudaMemcpyAsync(&nrm, c->norm_dev, 8, cudaMemcpyDeviceToHost, st));
    sync(c);
  }
  DME_REQUIRE(std::isfinite(nrm), DME_ERR_NUMERIC, "non-finite norm of A");
  const double tau0 = c->h / 2;
  const double tn = tau0 * nrm;
  int s = 0;
  if (tn > THETA13) s = std::max(0, (int)std::ceil(std::log2(tn / THETA13)));
  int sp_log = 0;
  while ((1 << sp_log) < c->subpanels) ++sp_log;
  const int s_total = s + sp_log;
  const double delta = tau0 / std::ldexp(1.0, s_total);
  c->stats.squarings = s;
  c->stats.quad_panels = 1 << s_total;
  c->stats.panel_width = delta;
  // X0 = delta * A^T
  if (!c->sparse) transpose_scale(c->Aup, n, ld, delta, c->X0, ld, st);

  // dense A that is exactly symmetric and sparse: Chebyshev actions (cheb.h) build E_{h/2} and the
  // quadrature factors; the partitioned ELL goes into the init-only Padé buffers (unused here)
  c->cheb_e = false;
  // (the CSR scratch lives in X2: (n + 1) rows offsets and up to 16 n entries must fit)
  // (replicated on every rank like the Padé init: identical inputs, deterministic kernels)
  if (!c->sparse && c->symA && c->opt.expm != DME_EXPM_PADE &&
      (size_t)(n + 1) * 8 + (size_t)16 * n * 12 + 16 <= (size_t)n * ld * 8) {
    std::vector<int64_t> rp;
    std::vector<int32_t> ci;
    std::vector<double> vv;
    if (cheb_csr_from_dense(c->Aup, n, ld, 16 * n, c->X2, st, rp, ci, vv)) {
      ChebHost ch;
      std::string err;
      double lm_est = 0;
      // (accuracy gate: ADVICE r1; cost model: the Chebyshev-built E costs ~K ceil(n/60) cluster
      // waves of ~2.1 us per degree (measured, §9c), Padé-13 with int8 products ~0.33 s (n/1e4)^3)
      const bool ok_prep = cheb_prepare(n, (int64_t)vv.size(), rp.data(), ci.data(), vv.data(), ch, &err) == 0;
      bool take = ok_prep && !ch.global &&
                  cheb_accurate(c->h, ch.b, n, rp.data(), ci.data(), vv.data(), &lm_est);
      if (take) {
        std::vector<double> chat;
        const double gamma = 0.5 * tau0 * (ch.b - ch.a);
        const int K = cheb_coeffs(gamma, std::ldexp(1.0, -56), chat);
        const double t_cheb = K * std::ceil(n / 60.0) * 2.1e-6;
        const double t_pade = 0.33 * std::pow(n / 1e4, 3.0) + 2e-3;
        take = t_cheb <= t_pade;
      }
      if (take &&
          (size_t)ch.w * CHEB_CLUSTER * ch.R <= (size_t)n * ld && ch.push.size() <= (size_t)n * ld &&
          ch.rptr.size() <= (size_t)n * ld && ch.rent.size() <= (size_t)n * ld) {
        c->chost = std::move(ch);
        ChebOp& op = c->cop;
        op.n = c->chost.n; op.R = c->chost.R; op.w = c->chost.w; op.C = c->chost.C;
        op.H = c->chost.H; op.P = c->chost.P;
        op.a = c->chost.a; op.b = c->chost.b; op.norm1 = c->chost.norm1;
        op.sym = c->chost.sym; op.mu = c->chost.mu; op.tnorm = c->chost.tnorm;
        op.val = c->X4;
        op.idx = reinterpret_cast<uint32_t*>(c->X6);
        op.push = reinterpret_cast<uint32_t*>(c->U);
        op.rptr = reinterpret_cast<uint32_t*>(c->V);
        op.rent = reinterpret_cast<uint32_t*>(c->BT);
        DME_CUDA(cudaMemcpyAsync(op.val, c->chost.val.data(), c->chost.val.size() * 8, cudaMemcpyHostToDevice, st));
        DME_CUDA(cudaMemcpyAsync(op.idx, c->chost.idx.data(), c->chost.idx.size() * 4, cudaMemcpyHostToDevice, st));
        if (!c->chost.push.empty())
          DME_CUDA(cudaMemcpyAsync(op.push, c->chost.push.data(), c->chost.push.size() * 4, cudaMemcpyHostToDevice, st));
        DME_CUDA(cudaMemcpyAsync(op.rptr, c->chost.rptr.data(), c->chost.rptr.size() * 4, cudaMemcpyHostToDevice, st));
        DME_CUDA(cudaMemcpyAsync(op.rent, c->chost.rent.data(), c->chost.rent.size() * 4, cudaMemcpyHostToDevice, st));
        c->cheb_e = true;
      }
    }
  }
  c->stats.expm_chebyshev = c->cheb_e ? 1 : 0;

  // ---------------------------------------------------------------- first-panel node actions
  // Y_i = exp(c_i delta A^T) L_Q = sum_j c_i^j W_j,  W_j = (delta A^T) W_{j-1} / j   (Taylor)
  const int q = c->qn;
  std::vector<double> cn, wn;
  gauss_legendre01(q, cn, wn);
  int64_t qI = 0;
  if (c->p > 0 && (c->sparse || c->cheb_e)) {  // Y_i = exp(c_i delta A^T) L_Q by the Chebyshev action
    for (int i = 0; i < q; ++i)
      sparse_pass(c, cn[i] * delta, c->LQ, c->p, c->Yn + (size_t)i * c->p * ld, ld, st);
  } else if (c->p > 0) {
    const double nx0 = delta * nrm;  // ||delta A^T||_1 bound for the truncation
    int J = 1;
    double term = 1.0;
    while (J < 200) {
      term *= nx0 / J;
      if (term < 1e-18 && J > nx0) break;
      ++J;
    }
    for (int i = 0; i < q; ++i)
      copy_cols(c->Yn + (size_t)i * c->p * ld, ld, c->LQ, ld, n, c->p, 1.0, st);
    copy_cols(c->Wa, ld, c->LQ, ld, n, c->p, 1.0, st);
    double* Wcur = c->Wa;
    double* Wnext = c->Wb;
    std::vector<double> cpow(q, 1.0);
    for (int j = 1; j <= J; ++j) {
      GemmNTArgs g;
      g.A = c->X0; g.lda = ld; g.B = Wcur; g.ldb = ld;
      g.M = n; g.N = c->p; g.K = n; g.alpha = 1.0 / j;
      g.out = Wnext; g.out_rs = 1; g.out_cs = ld;
      gemm_nt(g, c->gs, st);
      std::swap(Wcur, Wnext);
      for (int i = 0; i < q; ++i) {
        cpow[i] *= cn[i];
        double* Yi = c->Yn + (size_t)i * c->p * ld;
        axpy_cols(Yi, ld, Wcur, ld, n, c->p, cpow[i], st);  // Y_i += c_i^j W_j
      }
    }
  }
  if (c->p > 0) {
    // L_I(delta) = [sqrt(w_i delta) Y_i]  (D_I = blkdiag(w_i D_Q), D_Q = I; square-root form)
    for (int i = 0; i < q; ++i)
      copy_cols(c->Zc12h + (size_t)i * c->p * ld, ld, c->Yn + (size_t)i * c->p * ld, ld, n, c->p,
                std::sqrt(wn[i] * delta), st);
    c->tol_scale = LADDER_TOL;
    qI = compress(c, c->Zc12h, (int64_t)q * c->p, c->Ztmp, false, 0.0);
    copy_cols(c->Zc12h, ld, c->Ztmp, ld, n, qI, 1.0, st);
  }
  // final factors of the ladder: L_I(h) from the fine L_I(h/2), then L_I(h/2) itself at trunc_tol
  auto finish_ladder = [&](int64_t q_half, const double* Eh) {
    copy_cols(c->Zc12f, ld, c->Zc12h, ld, n, q_half, 1.0, st);
    int64_t qf = q_half;
    c->tol_scale = 1.0;
    ladder_double(c, c->Zc12f, qf, Eh, Eh ? 0.0 : tau0);
    c->qf = qf;
    int64_t qh = q_half;
    if (qh > 0) {
      qh = compress(c, c->Zc12h, q_half, c->Ztmp, false, 0.0);
      copy_cols(c->Zc12h, ld, c->Ztmp, ld, n, qh, 1.0, st);
    }
    c->qh = qh;
  };

  if (c->sparse || c->cheb_e) {
    // ---------------------------------------------------------------- ladder by sparse actions
    int64_t q_cur = qI;
    for (int j = 0; j < s_total; ++j) ladder_double(c, c->Zc12h, q_cur, nullptr, std::ldexp(delta, j));
    finish_ladder(q_cur, nullptr);
    if (c->cheb_e) {
      const double bound = std::sqrt((double)n) * std::exp(tau0 * std::max(c->chost.b, 0.0)) * (1 + 1e-12);
      auto check_norm = [&](const double* E, int64_t rows) {
        // sanity of the Chebyshev-built E before it is sliced for every later step:
        // finite, and ||E||_inf <= sqrt(n) ||E||_2 = sqrt(n) e^{tau lambda_max} <= sqrt(n) e^{tau b}
        double en = 0;
        rowabs_max(E, rows, ld, c->red_scratch, c->norm_dev, st);
        DME_CUDA(cudaMemcpyAsync(&en, c->norm_dev, 8, cudaMemcpyDeviceToHost, st));
        sync(c);
        DME_REQUIRE(std::isfinite(en) && en <= bound, DME_ERR_NUMERIC,
                    "Chebyshev-built E_{h/2} failed its norm check (non-finite or too large)");
      };
      lincomb(c->T1, n, ld, {}, {}, {}, {}, 1.0, st);  // identity (its columns e_j)
      if (c->world == 1) {
        // E_{h/2} = exp((h/2) A^T) I (columns = rows: A symmetric), exactly symmetrised; E_h = E_{h/2}^2
        c->stats.cheb_degree = cheb_action(c->cop, tau0, c->T1, ld, n, c->E_half, ld, 1.0, st);
        mirror_lower(c->E_half, n, ld, true, st);
        check_norm(c->E_half, n);
        matmul_sq(c, c->E_half, c->E_half, c->E_full);
      } else {
        // row-sharded: only the held rows, as columns of the symmetric E (E[rows, :] = (E I[:, rows])^T:
        // a column-major n x rows block with leading dimension ldn IS the row-major rows x n block),
        // E_h the same way with tau = h: no n x n matrix, no product, no collective
        c->stats.cheb_degree = cheb_action(c->cop, tau0, c->T1 + c->erow0 * ld, ld, c->erows, c->E_half, ld, 1.0, st);
        check_norm(c->E_half, c->erows);
        cheb_action(c->cop, c->h, c->T1 + c->erow0 * ld, ld, c->erows, c->E_full, ld, 1.0, st);
      }
      if (c->oz) {
        slice_shards(c, c->E_half, c->ozEh, c->exEh, st);
        slice_shards(c, c->E_full, c->ozEf, c->exEf, st);
        c->oz_ready = true;
      }
      c->cheb_e = false;  // the passes of the run use the dense E
    }
  } else {
  // ---------------------------------------------------------------- Padé-13 on X0 (Higham 2005)
  const double* b = PADE_B;
  matmul_sq(c, c->X0, c->X0, c->X2);
  matmul_sq(c, c->X2, c->X2, c->X4);
  matmul_sq(c, c->X4, c->X2, c->X6);
  lincomb(c->T1, n, ld, {b[13], c->X6}, {b[11], c->X4}, {b[9], c->X2}, {}, 0.0, st);
  matmul_sq(c, c->X6, c->T1, c->U);  // Y1 = X6 W1
  lincomb(c->T1, n, ld, {1.0, c->U}, {b[7], c->X6}, {b[5], c->X4}, {b[3], c->X2}, b[1], st);
  matmul_sq(c, c->X0, c->T1, c->U);  // U = X0 W2
  lincomb(c->T1, n, ld, {b[12], c->X6}, {b[10], c->X4}, {b[8], c->X2}, {}, 0.0, st);
  matmul_sq(c, c->X6, c->T1, c->V);  // Y2 = X6 Z1
  lincomb(c->V, n, ld, {1.0, c->V}, {b[6], c->X6}, {b[4], c->X4}, {b[2], c->X2}, b[0], st);
  lincomb(c->X4, n, ld, {1.0, c->V}, {-1.0, c->U}, {}, {}, 0.0, st);  // Q = V - U
  lincomb(c->X6, n, ld, {1.0, c->V}, {1.0, c->U}, {}, {}, 0.0, st);   // P = V + U
  lu_solve_right(c->X4, c->X6, n, ld, c->BT, c->lu_scr, c->gs, st, c->norm_dev + 1);
  if (c->symA) mirror_lower(c->X6, n, ld, true, st);  // exact symmetry of E_delta
  double minpiv = 0;
  DME_CUDA(cudaMemcpyAsync(&minpiv, c->norm_dev + 1, 8, cudaMemcpyDeviceToHost, st));
  sync(c);
  c->stats.pade_min_pivot = minpiv;
  // partial pivoting: a pivot 13 orders below the scale b_0 of q13(X) would mean kappa(q13) >~ 1e13,
  // which Higham's bound on ||X||_1 <= theta_13 excludes; only a corrupted input gets here
  DME_REQUIRE(std::isfinite(minpiv) && minpiv > 1e-13 * b[0], DME_ERR_NUMERIC,
              "Padé denominator is numerically singular");

  // ---------------------------------------------------------------- squaring ladder + quadrature
  double* Ecur = c->X6;
  double* spare[2] = {c->X2, c->U};
  int si = 0;
  int64_t q_cur = qI;
  for (int j = 0; j < s_total; ++j) {
    ladder_double(c, c->Zc12h, q_cur, Ecur, 0.0);  // L_I(2w) from E_w, w = delta 2^j
    double* En = spare[si];
    matmul_sq(c, Ecur, Ecur, En);
    spare[si] = (Ecur == c->X6) ? c->V : Ecur;
    si ^= 1;
    Ecur = En;
  }
  // L_I(h) = compress([L_I(h/2), E_{h/2} L_I(h/2)]),  E_h = E_{h/2}^2 (full n x n in init buffers);
  // this process keeps the rows [erow0, erow0 + erows) of both (a real rank: its own rows)
  finish_ladder(q_cur, Ecur);
  double* Eh_full = spare[si];
  matmul_sq(c, Ecur, Ecur, Eh_full);
  DME_CUDA(cudaMemcpy2DAsync(c->E_half, ld * 8, Ecur + c->erow0 * ld, ld * 8, n * 8, c->erows,
                             cudaMemcpyDeviceToDevice, st));
  DME_CUDA(cudaMemcpy2DAsync(c->E_full, ld * 8, Eh_full + c->erow0 * ld, ld * 8, n * 8, c->erows,
                             cudaMemcpyDeviceToDevice, st));
  if (c->oz) {  // digit slices of the held rows of E_{h/2} and E_h (after the last product)
    slice_shards(c, c->E_half, c->ozEh, c->exEh, st);
    slice_shards(c, c->E_full, c->ozEf, c->exEf, st);
    c->oz_ready = true;
  }
  }  // dense E
  // look-ahead operand: E_h L_I(h) stays in the leading columns of LA
  eact(c, true, c->Zc12f, c->qf, c->LA, ld);
  // fixed columns of the congruence pipeline's GB = [L_I(h) | B | E_h L_I(h) | (E_h Y)]
  if (c->m > 0 && 2 * c->qf + c->m <= KMAX) {
    copy_cols(c->GB, ld, c->Zc12f, ld, n, c->qf, 1.0, st);
    copy_cols(c->GB + c->qf * ld, ld, c->Bcol, ld, n, c->m, 1.0, st);
    copy_cols(c->GB + (c->qf + c->m) * ld, ld, c->LA, ld, n, c->qf, 1.0, st);
  }
  c->stats.q_half = c->qh;
  c->stats.q_full = c->qf;

  // ---------------------------------------------------------------- P0: Z0 = L0 D0^{1/2}, compressed
  c->r = 0;
  if (c->r0 > 0) {
    // square-root factor of D0 through the same kernel: D0 = W Theta W^T, Tm = W Theta^{1/2}
    DME_CUDA(cudaMemcpy2DAsync(c->G, KMAX * 8, c->D0d, c->r0 * 8, c->r0 * 8, c->r0,
                               cudaMemcpyDeviceToDevice, st));
    SmallArgs a;
    a.k = (int)c->r0; a.compress = 1; a.G = c->G; a.ldg = KMAX; a.tol = 1e-15; a.cap = (int)c->r0;
    a.Tm = c->Tm; a.ldt = KMAX; a.r_out = c->r_dev; a.stats = c->sstats;
    a.V = c->Vg; a.ldv = KMAX; a.sqrt_scale = 1;
    compress_t3(a, st);
    int rd = 0;
    DME_CUDA(cudaMemcpyAsync(&rd, c->r_dev, 4, cudaMemcpyDeviceToHost, st));
    sync(c);
    if (rd > 0) {
      tall_small(c->L0d, ld, c->Tm, KMAX, c->Zc2, ld, n, rd, c->r0, st);
      c->r = compress(c, c->Zc2, rd, c->Z, false, 0.0);
    }
  }
  c->stats.rank = c->r;
  c->stats.max_rank = c->r;
  sync(c);
}

dme_status fail(const std::exception& e, dme_status code, dme_ctx* c = nullptr) {
  g_last_error = e.what();
  if (c && (code == DME_ERR_CUDA || code == DME_ERR_NCCL)) c->poisoned = true;
  return code;
}

template <class F>
dme_status guarded(dme_ctx* c, F&& f) {
  if (c && c->poisoned) {
    g_last_error = "context poisoned by an earlier CUDA/NCCL failure";
    return DME_ERR_POISONED;
  }
  try {
    f();
    return DME_OK;
  } catch (const DmeError& e) {
    return fail(e, e.code, c);
  } catch (const CudaError& e) {
    return fail(e, DME_ERR_CUDA, c);
  } catch (const std::bad_alloc& e) {
    return fail(e, DME_ERR_NOMEM, c);
  } catch (const std::exception& e) {
    return fail(e, DME_ERR_CUDA, c);
  }
}

dme_status init_common(const dme_problem* pr, const dme_options* o, dme_ctx** out, bool dre) {
  if (!out) {
    g_last_error = "NULL ctx out-pointer";
    return DME_ERR_INVALID;
  }
  *out = nullptr;
  dme_ctx* c = nullptr;
  dme_status s = guarded(nullptr, [&] {
    validate(pr, o, dre);
    auto t0 = std::chrono::steady_clock::now();
    std::unique_ptr<dme_ctx> cp(new dme_ctx());
    c = cp.get();
    fill_dims(c, pr, o);
    c->dre = dre;

    if (dre) c->lrinv_host = chol_inverse_lower(pr->R, (int)pr->m);
    if (pr->r0 > 0 && pr->D0) check_psd_host(pr->D0, pr->r0);
    DME_CUDA(cudaSetDevice(o->device));
    c->st = reinterpret_cast<cudaStream_t>(o->stream);
    int lo_pri = 0, hi_pri = 0;
    DME_CUDA(cudaDeviceGetStreamPriorityRange(&lo_pri, &hi_pri));
    DME_CUDA(cudaStreamCreateWithPriority(&c->st2, cudaStreamNonBlocking, lo_pri));
    // (pinned host memory for the rank record: the library's only host allocation besides the
    // ctx; device memory stays the caller's workspace)
    DME_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&c->hmap), sizeof(HostMap), cudaHostAllocMapped));
    std::memset(c->hmap, 0, sizeof(HostMap));
    DME_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&c->hmap_dev), c->hmap, 0));
    DME_CUDA(cudaEventCreateWithFlags(&c->ev_gram, cudaEventDisableTiming));
    DME_CUDA(cudaEventCreateWithFlags(&c->ev_ahead, cudaEventDisableTiming));
    for (cudaEvent_t* e : {&c->ev_ghat, &c->ev_cong, &c->ev_y, &c->ev_zc, &c->ev_tm})
      DME_CUDA(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
    Planner sizing;
    plan_buffers(c, sizing);
    DME_REQUIRE(o->workspace && o->workspace_bytes >= sizing.off + 256, DME_ERR_CAPACITY,
                "workspace too small: need " + std::to_string(sizing.off + 256) + " bytes");
    Planner P;
    P.base = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(o->workspace) + 255) & ~uintptr_t(255));
    plan_buffers(c, P);
    // the look-ahead stream (E pass, Gram) leaves SMs to the critical path: the eigen kernels and the
    // n-row kernels of the refined compression (DME_LOOKAHEAD_SMS overrides, for measurements)
    int la = num_sms() - LOOKAHEAD_RESERVE;
    if (const char* e = std::getenv("DME_LOOKAHEAD_SMS")) la = std::atoi(e);
    la = std::max(1, std::min(la, num_sms()));
    c->gs2.max_grid = la;
    c->ozs.max_grid = std::min(256, num_sms());
    c->ozs2.max_grid = la;
    if (c->virt) {  // one-rank communicator: the allgather of the virtual shards is a real NCCL call
      ncclUniqueId uid;
      DME_NCCL(ncclGetUniqueId(&uid));
      DME_NCCL(ncclCommInitRank(&c->comm, 1, uid, 0));
    } else if (c->world > 1) {
      ncclUniqueId uid;
      std::memcpy(&uid, o->nccl_uid, sizeof(uid));
      DME_NCCL(ncclCommInitRank(&c->comm, c->world, uid, c->rank));
    }
    init_all(c, pr);
    c->stats.init_seconds =
        std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    *out = cp.release();
  });
  if (s != DME_OK && c && *out == nullptr) {
    // the unique_ptr already freed it
  }
  return s;
}

}  // namespace

// axpy on a column block: Y[:, j] += alpha X[:, j]
namespace {
__global__ void axpy_cols_kernel(double* Y, int64_t ldy, const double* X, int64_t ldx, int64_t rows,
                                 int64_t cols, double alpha) {
  const int64_t total = rows * cols;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e % rows, j = e / rows;
    Y[i + j * ldy] += alpha * X[i + j * ldx];
  }
}
}  // namespace
void axpy_cols(double* Y, int64_t ldy, const double* X, int64_t ldx, int64_t rows, int64_t cols,
               double alpha, cudaStream_t st) {
  const int64_t total = rows * cols;
  int blocks = (int)std::min<int64_t>((total + 255) / 256, 148 * 8);
  axpy_cols_kernel<<<blocks > 0 ? blocks : 1, 256, 0, st>>>(Y, ldy, X, ldx, rows, cols, alpha);
  DME_KCHECK();
}

// ====================================================================== C ABI
extern "C" {

void dme_default_options(dme_options* o) {
  if (!o) return;
  std::memset(o, 0, sizeof(*o));
  o->h = 0.005;
  o->trunc_tol = 1e-16;
  o->rank_cap = 0;
  o->quad_nodes = 14;
  o->quad_subpanels = 1;
  o->world_size = 1;
}

const char* dme_status_string(dme_status s) {
  switch (s) {
    case DME_OK: return "ok";
    case DME_ERR_INVALID: return "invalid argument";
    case DME_ERR_DIM: return "dimension error";
    case DME_ERR_CONFIG: return "configuration error";
    case DME_ERR_SINGULAR: return "singular system";
    case DME_ERR_NUMERIC: return "numerical failure";
    case DME_ERR_CAPACITY: return "capacity exceeded";
    case DME_ERR_CUDA: return "CUDA error";
    case DME_ERR_NCCL: return "NCCL error";
    case DME_ERR_NOMEM: return "out of memory";
    case DME_ERR_POISONED: return "context poisoned";
  }
  return "unknown status";
}

const char* dme_last_error(void) { return g_last_error.c_str(); }

dme_status dme_workspace_size(const dme_problem* pr, const dme_options* o, size_t* bytes) {
  return guarded(nullptr, [&] {
    DME_REQUIRE(pr && o && bytes, DME_ERR_INVALID, "NULL argument");
    DME_REQUIRE(pr->n > 0, DME_ERR_INVALID, "n must be positive");
    dme_ctx c;
    fill_dims(&c, pr, o);
    Planner P;
    plan_buffers(&c, P);
    *bytes = P.off + 512;
  });
}

dme_status dme_shard_rows(int64_t n, int32_t world, int32_t rank, int64_t* row0, int64_t* rows,
                          int64_t* nloc) {
  return guarded(nullptr, [&] {
    DME_REQUIRE(n > 0 && world >= 1 && rank >= 0 && rank < world && row0 && rows && nloc,
                DME_ERR_INVALID, "bad shard arguments");
    shard_rows(n, world, rank, row0, rows, nloc);
  });
}

dme_status dme_get_unique_id(void* uid128) {
  return guarded(nullptr, [&] {
    DME_REQUIRE(uid128, DME_ERR_INVALID, "NULL uid");
    ncclUniqueId id;
    DME_NCCL(ncclGetUniqueId(&id));
    std::memcpy(uid128, &id, sizeof(id));
  });
}

dme_status dme_dle_init(const dme_problem* pr, const dme_options* o, dme_ctx** ctx) {
  return init_common(pr, o, ctx, false);
}
dme_status dme_dre_init(const dme_problem* pr, const dme_options* o, dme_ctx** ctx) {
  return init_common(pr, o, ctx, true);
}

dme_status dme_split_step(dme_ctx* c, dme_scheme scheme, dme_composition comp, int64_t nsteps) {
  if (!c) { g_last_error = "NULL ctx"; return DME_ERR_INVALID; }
  return guarded(c, [&] {
    DME_REQUIRE(nsteps >= 0, DME_ERR_INVALID, "nsteps must be >= 0");
    auto seq = step_sequence(scheme, comp, c->h);
    check_capable(c, seq);
    if (c->profile && getenv("DME_TIMELINE")) {
      if (!c->tl_base) DME_CUDA(cudaEventCreate(&c->tl_base));
      DME_CUDA(cudaEventRecord(c->tl_base, c->st));
      fprintf(stderr, "[dme timeline] split_step start\n");
    }
    // FSAL: under Strang, the trailing A(h/2) of a step and the leading A(h/2) of the next are one
    // A(h) when A is a semigroup flow computed exactly (T1: E_{h/2}^2 = E_h; T12: the ladder rule
    // gives I(h) = I(h/2) + E_{h/2} I(h/2) E_{h/2}^T exactly), so nsteps steps run as
    //   A(h/2) X [A(h) X]^{nsteps-1} A(h/2)   (X = the middle flows) — half the E passes.
    const bool merge = c->fsal && scheme == DME_STRANG && seq.size() > 1 && nsteps > 1 &&
                       seq.front().flow == seq.back().flow &&
                       (seq.front().flow == DME_FLOW_T1 || seq.front().flow == DME_FLOW_T12);
    if (merge) {
      std::vector<Op> first(seq.begin(), seq.end() - 1), mid(seq.begin() + 1, seq.end() - 1);
      std::vector<Op> body{{seq.front().flow, c->h}};
      body.insert(body.end(), mid.begin(), mid.end());
      run_sequence(c, first);
      c->stats.steps++;
      if (comp == DME_F12F3 && c->dre) {
        run_f12f3_body(c, nsteps - 1, c->h);  // pipelined (look-ahead E pass)
      } else {
        for (int64_t s = 1; s < nsteps; ++s) {
          run_sequence(c, body);
          c->stats.steps++;
        }
      }
      run_sequence(c, {seq.back()});
    } else {
      for (int64_t s = 0; s < nsteps; ++s) {
        run_sequence(c, seq);
        c->stats.steps++;
      }
    }
    c->stats.t = c->stats.steps * c->h;
    c->stats.rank = c->r;
    DME_CUDA(cudaGetLastError());
  });
}

dme_status dme_get_factor(dme_ctx* c, int64_t* r, double* L, double* D, int64_t cap) {
  if (!c) { g_last_error = "NULL ctx"; return DME_ERR_INVALID; }
  return guarded(c, [&] {
    DME_REQUIRE(r, DME_ERR_INVALID, "NULL r");
    *r = c->r;
    if (!L && !D) return;
    DME_REQUIRE(c->r <= cap, DME_ERR_CAPACITY, "factor has more columns than capacity_cols");
    if (L && c->r > 0) {
      std::vector<double> tmp((size_t)c->n * c->r);
      DME_CUDA(cudaMemcpy2DAsync(tmp.data(), c->n * 8, c->Z, c->ldn * 8, c->n * 8, c->r,
                                 cudaMemcpyDeviceToHost, c->st));
      sync(c);
      for (int64_t j = 0; j < c->r; ++j)
        for (int64_t i = 0; i < c->n; ++i) L[i * c->r + j] = tmp[(size_t)j * c->n + i];
    }
    if (D)  // square-root form: P = Z Z^T, i.e. D = I
      for (int64_t i = 0; i < c->r; ++i)
        for (int64_t j = 0; j < c->r; ++j) D[i * c->r + j] = i == j ? 1.0 : 0.0;
  });
}

dme_status dme_extrapolate(dme_ctx* fine, dme_ctx* coarse, int64_t* r, double* L, double* D,
                           int64_t cap) {
  if (!fine || !coarse) { g_last_error = "NULL ctx"; return DME_ERR_INVALID; }
  return guarded(fine, [&] {
    dme_ctx* c = fine;
    dme_ctx* d = coarse;
    DME_REQUIRE(r, DME_ERR_INVALID, "NULL r");
    DME_REQUIRE(c != d && c->n == d->n && c->ldn == d->ldn && c->opt.device == d->opt.device,
                DME_ERR_CONFIG, "fine and coarse must be two contexts of one problem on one device");
    DME_REQUIRE(std::fabs(2.0 * c->h - d->h) <= 1e-12 * d->h, DME_ERR_CONFIG,
                "the fine step must be half the coarse step");
    DME_REQUIRE(c->stats.steps == 2 * d->stats.steps && d->stats.steps > 0, DME_ERR_CONFIG,
                "the fine run must have taken twice the coarse run's steps (same time t > 0)");
    const int64_t n = c->n, ld = c->ldn, kf = c->r, kc = d->r, k = kf + kc;
    DME_REQUIRE(k <= KMAX, DME_ERR_DIM, "combined rank exceeds the factor capacity");
    cudaStream_t st = c->st;
    // both states ready, on the fine context's stream
    DME_CUDA(cudaStreamSynchronize(d->st));
    *r = 0;
    if (k > 0) {
      // Zc = [Z_fine | Z_coarse],  P = Zc S Zc^T,  S = diag(4/3 I, -1/3 I). A Gram-based basis
      // loses ~eps kappa(Zc)^2 here (the two factors span nearly the same space: measured 5e-9
      // in P), so the basis is built by classical Gram-Schmidt with reorthogonalisation (CGS2,
      // backward stable like Householder for kappa < 1/eps): Q (n x r1) orthonormal, then
      // R^T = Zc^T Q, the signed core M = R S R^T = U Lambda U^T, L = Q U_kept, D = Lambda_kept.
      double* Zc = c->Zc2;
      double* Q = c->Ztmp;
      double* v = c->X2;          // init-only n x n scratch, free after init
      double* w = c->X2 + ld;     // second column
      double* hcol = c->Vg;       // Q^T v (KMAX)
      double* nrm = c->norm_dev + 8;
      copy_cols(Zc, ld, c->Z, ld, n, kf, 1.0, st);
      copy_cols(Zc + kf * ld, ld, d->Z, ld, n, kc, 1.0, st);
      int64_t r1 = 0;
      for (int64_t j = 0; j < k; ++j) {
        copy_cols(v, ld, Zc + j * ld, ld, n, 1, 1.0, st);
        double z2 = 0.0;
        {
          GemmNTArgs g;
          g.A = v; g.lda = ld; g.B = v; g.ldb = ld; g.M = 1; g.N = 1; g.K = n;
          g.out = nrm; g.out_rs = 1; g.out_cs = 1;
          gemm_nt(g, c->gs, st);
          DME_CUDA(cudaMemcpyAsync(&z2, nrm, 8, cudaMemcpyDeviceToHost, st));
        }
        for (int pass = 0; pass < 2 && r1 > 0; ++pass) {  // v -= Q (Q^T v), twice
          GemmNTArgs g;
          g.A = Q; g.lda = ld; g.B = v; g.ldb = ld; g.M = r1; g.N = 1; g.K = n;
          g.out = hcol; g.out_rs = 1; g.out_cs = KMAX;
          gemm_nt(g, c->gs, st);
          tall_small(Q, ld, hcol, KMAX, w, ld, n, 1, r1, st);
          axpy_cols(v, ld, w, ld, n, 1, -1.0, st);
        }
        double v2 = 0.0;
        {
          GemmNTArgs g;
          g.A = v; g.lda = ld; g.B = v; g.ldb = ld; g.M = 1; g.N = 1; g.K = n;
          g.out = nrm; g.out_rs = 1; g.out_cs = 1;
          gemm_nt(g, c->gs, st);
          DME_CUDA(cudaMemcpyAsync(&v2, nrm, 8, cudaMemcpyDeviceToHost, st));
          sync(c);
        }
        // a column inside span(Q) to working precision adds nothing (rank deficiency)
        if (!(v2 > 1e-28 * z2) || !(v2 > 0.0)) continue;
        copy_cols(Q + r1 * ld, ld, v, ld, n, 1, 1.0 / std::sqrt(v2), st);
        ++r1;
      }
      DME_REQUIRE(r1 <= 112, DME_ERR_DIM, "combined rank exceeds 112");
      // R^T = Zc^T Q (k x r1), as "Tm" of the signed core: M = Tm^T S Tm = R S R^T
      {
        GemmNTArgs g;
        g.A = Zc; g.lda = ld; g.B = Q; g.ldb = ld; g.M = k; g.N = r1; g.K = n;
        g.out = c->Tm; g.out_rs = 1; g.out_cs = KMAX;
        gemm_nt(g, c->gs, st);
      }
      signed_core(c->Tm, KMAX, (int)k, (int)r1, (int)kf, 4.0 / 3.0, -1.0 / 3.0, c->opt.trunc_tol,
                  c->Tm2, KMAX, c->H, c->r_dev + 1, st, true);
      int r2 = 0;
      DME_CUDA(cudaMemcpyAsync(&r2, c->r_dev + 1, sizeof(int), cudaMemcpyDeviceToHost, st));
      sync(c);
      *r = r2;
      if (r2 > 0 && (L || D)) {
        DME_REQUIRE(r2 <= cap, DME_ERR_CAPACITY, "factor has more columns than capacity_cols");
        double* Lout = c->X4;  // init-only scratch
        tall_small(Q, ld, c->Tm2, KMAX, Lout, ld, n, r2, r1, st);  // L = Q U_kept
        std::vector<double> tmp((size_t)n * r2), lam(r2);
        DME_CUDA(cudaMemcpy2DAsync(tmp.data(), n * 8, Lout, ld * 8, n * 8, r2,
                                   cudaMemcpyDeviceToHost, st));
        DME_CUDA(cudaMemcpyAsync(lam.data(), c->H, r2 * 8, cudaMemcpyDeviceToHost, st));
        sync(c);
        if (L)
          for (int64_t j = 0; j < r2; ++j)
            for (int64_t i = 0; i < n; ++i) L[i * r2 + j] = tmp[(size_t)j * n + i];
        if (D)
          for (int64_t i = 0; i < r2; ++i)
            for (int64_t j = 0; j < r2; ++j) D[i * r2 + j] = i == j ? lam[i] : 0.0;
      }
    }
  });
}

dme_status dme_get_stats(dme_ctx* c, dme_stats* st) {
  if (!c || !st) { g_last_error = "NULL argument"; return DME_ERR_INVALID; }
  return guarded(c, [&] {
    drain_profile(c);
    c->stats.rank = c->r;
    c->stats.kernel_launches = launch_count();
    *st = c->stats;
  });
}

dme_status dme_set_profiling(dme_ctx* c, int32_t on) {
  if (!c) { g_last_error = "NULL ctx"; return DME_ERR_INVALID; }
  return guarded(c, [&] {
    drain_profile(c);
    c->profile = on != 0;
    c->stats.prof_passes = 0;
    c->stats.prof_epass_seconds = c->stats.prof_epass_flops = c->stats.prof_epass_bytes = 0;
    c->stats.prof_gram_seconds = c->stats.prof_small_seconds = c->stats.prof_apply_seconds = 0;
  });
}

dme_status dme_cheb_coeffs(double gamma, double tol, double* out, int64_t cap, int32_t* K) {
  return guarded(nullptr, [&] {
    DME_REQUIRE(out && K && std::isfinite(gamma) && gamma >= 0 && tol > 0, DME_ERR_INVALID,
                "bad Chebyshev coefficient arguments");
    std::vector<double> chat;
    const int k = cheb_coeffs(gamma, tol, chat);
    DME_REQUIRE(k + 1 <= cap, DME_ERR_CAPACITY, "coefficient buffer too small");
    std::memcpy(out, chat.data(), chat.size() * 8);
    *K = k;
  });
}

dme_status dme_destroy(dme_ctx* c) {
  delete c;  // ~dme_ctx releases streams, events and the NCCL communicator
  return DME_OK;
}

dme_status dme_debug_apply(dme_ctx* c, int32_t flow, double tau) {
  if (!c) { g_last_error = "NULL ctx"; return DME_ERR_INVALID; }
  return guarded(c, [&] {
    if (flow == DME_FLOW_T1 || flow == DME_FLOW_T12)
      DME_REQUIRE(tau == c->h || tau == c->h / 2, DME_ERR_CONFIG, "tau must be h or h/2");
    switch (flow) {
      case DME_FLOW_T1: flow_T1(c, tau); break;
      case DME_FLOW_T2: flow_T2(c, tau, false, 0); break;
      case DME_FLOW_T3: DME_REQUIRE(c->dre, DME_ERR_CONFIG, "no B"); flow_T3(c, tau); break;
      case DME_FLOW_T4_MIDPOINT: DME_REQUIRE(c->has_S, DME_ERR_CONFIG, "no S"); flow_T4(c, tau, 2, false, 0); break;
      case DME_FLOW_T4_EULER: DME_REQUIRE(c->has_S, DME_ERR_CONFIG, "no S"); flow_T4(c, tau, 1, false, 0); break;
      case DME_FLOW_T12: flow_T12(c, tau, false, 0); break;
      case DME_FLOW_COMPRESS:
        if (c->r > 0) {
          copy_cols(c->Zc2, c->ldn, c->Z, c->ldn, c->n, c->r, 1.0, c->st);
          finish_compress(c, c->Zc2, c->r, false, 0);
        }
        break;
      default: throw DmeError(DME_ERR_CONFIG, "unknown flow");
    }
    sync(c);
  });
}

dme_status dme_debug_set_factor(dme_ctx* c, int64_t r, const double* L) {
  if (!c) { g_last_error = "NULL ctx"; return DME_ERR_INVALID; }
  return guarded(c, [&] {
    DME_REQUIRE(r >= 0 && r <= KMAX && (r == 0 || L), DME_ERR_INVALID, "bad factor");
    if (r > 0) {
      DME_CUDA(cudaMemcpyAsync(c->Ztmp, L, c->n * r * 8, cudaMemcpyHostToDevice, c->st));
      rowmajor_to_colmajor(c->Z, c->ldn, c->Ztmp, r, c->n, r, c->st);
    }
    c->r = r;
    sync(c);
  });
}

dme_status dme_debug_set_exp(dme_ctx* c, int32_t which, const double* E) {
  if (!c || !E) { g_last_error = "NULL argument"; return DME_ERR_INVALID; }
  return guarded(c, [&] {
    DME_REQUIRE(!c->sparse, DME_ERR_CONFIG, "no dense E with a sparse A");
    DME_REQUIRE(which == 0 || which == 1, DME_ERR_INVALID, "which must be 0 (E_{h/2}) or 1 (E_h)");
    DME_REQUIRE(c->erows == c->n, DME_ERR_CONFIG, "this rank holds only its rows of E");
    double* dst = which ? c->E_full : c->E_half;
    DME_CUDA(cudaMemcpy2DAsync(dst, c->ldn * 8, E, c->n * 8, c->n * 8, c->n,
                               cudaMemcpyHostToDevice, c->st));
    if (c->oz && c->oz_ready)  // the int8 E pass reads the digit images: re-slice them
      slice_shards(c, dst, which ? c->ozEf : c->ozEh, which ? c->exEf : c->exEh, c->st);
    if (which == 1 && c->qf > 0)  // the look-ahead operand E_h L_I(h) of the pipelined body
      eact(c, true, c->Zc12f, c->qf, c->LA, c->ldn);
    if (which == 1 && c->m > 0 && 2 * c->qf + c->m <= KMAX)
      copy_cols(c->GB + (c->qf + c->m) * c->ldn, c->ldn, c->LA, c->ldn, c->n, c->qf, 1.0, c->st);
    sync(c);
  });
}

dme_status dme_debug_get_exp(dme_ctx* c, int32_t which, double* E) {
  if (!c || !E) { g_last_error = "NULL argument"; return DME_ERR_INVALID; }
  return guarded(c, [&] {
    DME_REQUIRE(!c->sparse, DME_ERR_CONFIG, "no dense E with a sparse A");
    DME_REQUIRE(c->erows == c->n, DME_ERR_CONFIG, "this rank holds only its rows of E");
    const double* src = which ? c->E_full : c->E_half;
    DME_CUDA(cudaMemcpy2DAsync(E, c->n * 8, src, c->ldn * 8, c->n * 8, c->n,
                               cudaMemcpyDeviceToHost, c->st));
    sync(c);
  });
}

dme_status dme_debug_get_integral(dme_ctx* c, int32_t which, int64_t* q, double* L, int64_t cap) {
  if (!c || !q) { g_last_error = "NULL argument"; return DME_ERR_INVALID; }
  return guarded(c, [&] {
    const int64_t qq = which ? c->qf : c->qh;
    *q = qq;
    if (!L) return;
    DME_REQUIRE(qq <= cap, DME_ERR_CAPACITY, "capacity too small");
    std::vector<double> tmp((size_t)c->n * std::max<int64_t>(qq, 1));
    if (qq > 0)
      DME_CUDA(cudaMemcpy2DAsync(tmp.data(), c->n * 8, which ? c->Zc12f : c->Zc12h, c->ldn * 8,
                                 c->n * 8, qq, cudaMemcpyDeviceToHost, c->st));
    sync(c);
    for (int64_t j = 0; j < qq; ++j)
      for (int64_t i = 0; i < c->n; ++i) L[i * qq + j] = tmp[(size_t)j * c->n + i];
  });
}

dme_status dme_debug_small_stats(dme_ctx* c, double* out16) {
  if (!c || !out16) { g_last_error = "NULL argument"; return DME_ERR_INVALID; }
  return guarded(c, [&] {
    DME_CUDA(cudaMemcpyAsync(out16, c->sstats, 16 * sizeof(double), cudaMemcpyDeviceToHost, c->st));
    sync(c);
  });
}

dme_status dme_debug_complement(int64_t k, int64_t kb, const double* W, double* U) {
  return guarded(nullptr, [&] {
    DME_REQUIRE(W && U && kb >= 0 && kb < k && k <= FAST_K_MAX, DME_ERR_INVALID, "bad complement args");
    const int64_t s = k - kb;
    std::vector<double> wc((size_t)k * (kb > 0 ? kb : 1)), uc((size_t)k * s);
    for (int64_t i = 0; i < k; ++i)
      for (int64_t j = 0; j < kb; ++j) wc[j * k + i] = W[i * kb + j];  // column-major, ld k
    double *dW, *dU;
    DME_CUDA(cudaMalloc(&dW, wc.size() * 8));
    DME_CUDA(cudaMalloc(&dU, uc.size() * 8));
    DME_CUDA(cudaMemcpy(dW, wc.data(), wc.size() * 8, cudaMemcpyHostToDevice));
    complement_basis(dW, k, (int)k, (int)kb, dU, k, nullptr);
    DME_CUDA(cudaDeviceSynchronize());
    DME_CUDA(cudaMemcpy(uc.data(), dU, uc.size() * 8, cudaMemcpyDeviceToHost));
    cudaFree(dW);
    cudaFree(dU);
    for (int64_t i = 0; i < k; ++i)
      for (int64_t j = 0; j < s; ++j) U[i * s + j] = uc[j * k + i];
  });
}

dme_status dme_debug_matmul(int64_t M, int64_t N, int64_t K, const double* A, const double* B,
                            double* C) {
  return guarded(nullptr, [&] {
    DME_REQUIRE(M > 0 && N > 0 && K > 0 && A && B && C, DME_ERR_INVALID, "bad matmul args");
    const int64_t ldk = (K + 15) / 16 * 16;
    double *dA, *dBT, *dC, *part;
    int* cnt;
    GemmScratch gs;
    gs.max_grid = 256;
    gs.max_tiles = 1 << 16;
    DME_CUDA(cudaMalloc(&dA, M * ldk * 8));
    DME_CUDA(cudaMalloc(&dBT, N * ldk * 8));
    DME_CUDA(cudaMalloc(&dC, M * N * 8));
    DME_CUDA(cudaMalloc(&part, GemmScratch::partial_doubles(gs.max_grid) * 8));
    DME_CUDA(cudaMalloc(&cnt, gs.max_tiles * sizeof(int)));
    DME_CUDA(cudaMemset(cnt, 0, gs.max_tiles * sizeof(int)));
    gs.partial = part;
    gs.counters = cnt;
    DME_CUDA(cudaMemcpy2D(dA, ldk * 8, A, K * 8, K * 8, M, cudaMemcpyHostToDevice));
    std::vector<double> bt((size_t)N * K);
    for (int64_t i = 0; i < K; ++i)
      for (int64_t j = 0; j < N; ++j) bt[j * K + i] = B[i * N + j];
    DME_CUDA(cudaMemcpy2D(dBT, ldk * 8, bt.data(), K * 8, K * 8, N, cudaMemcpyHostToDevice));
    GemmNTArgs g;
    g.A = dA; g.lda = ldk; g.B = dBT; g.ldb = ldk;
    g.M = M; g.N = N; g.K = K;
    g.out = dC; g.out_rs = N; g.out_cs = 1;
    gemm_nt(g, gs, 0);
    DME_CUDA(cudaDeviceSynchronize());
    DME_CUDA(cudaMemcpy(C, dC, M * N * 8, cudaMemcpyDeviceToHost));
    cudaFree(dA); cudaFree(dBT); cudaFree(dC); cudaFree(part); cudaFree(cnt);
  });
}

dme_status dme_debug_matmul_ozaki(int64_t M, int64_t N, int64_t K, const double* A, const double* B,
                                  double* C) {
  return guarded(nullptr, [&] {
    DME_REQUIRE(M > 0 && N > 0 && K > 0 && A && B && C, DME_ERR_INVALID, "bad matmul args");
    DME_REQUIRE(N <= OZ_NMAX && K <= OZ_KMAX, DME_ERR_DIM, "ozaki matmul: N <= 64, K <= 32768");
    const int64_t ldd = (K + 15) / 16 * 16, ldq = oz_ldk(K);
    double *dA, *dBT, *dC, *part;
    int8_t *qa, *qb;
    int *ea, *eb, *cnt;
    double* pm;
    OzScratch ws;
    ws.max_tiles = ceil_div(M, 128);
    ws.max_grid = std::min(256, num_sms());
    DME_CUDA(cudaMalloc(&dA, M * ldd * 8));
    DME_CUDA(cudaMalloc(&dBT, OZ_NMAX * ldd * 8));
    DME_CUDA(cudaMalloc(&dC, M * N * 8));
    DME_CUDA(cudaMalloc(&qa, std::max<size_t>((size_t)OZ_S * M * ldq, (size_t)oz_tiled_bytes(M, K))));
    DME_CUDA(cudaMalloc(&qb, (size_t)OZ_S * OZ_NMAX * ldq));
    DME_CUDA(cudaMalloc(&ea, M * sizeof(int)));
    DME_CUDA(cudaMalloc(&eb, OZ_NMAX * sizeof(int)));
    DME_CUDA(cudaMalloc(&part, OzScratch::partial_doubles(ws.max_tiles, ws.max_grid) * 8));
    DME_CUDA(cudaMalloc(&cnt, ws.max_tiles * sizeof(int)));
    DME_CUDA(cudaMalloc(&pm, oz_slice_scratch_doubles(std::max<int64_t>(M, N), K) * 8));
    DME_CUDA(cudaMemset(cnt, 0, ws.max_tiles * sizeof(int)));
    DME_CUDA(cudaMemset(qb, 0, (size_t)OZ_S * OZ_NMAX * ldq));
    ws.partial = part;
    ws.counters = cnt;
    DME_CUDA(cudaMemcpy2D(dA, ldd * 8, A, K * 8, K * 8, M, cudaMemcpyHostToDevice));
    std::vector<double> bt((size_t)N * K);
    for (int64_t i = 0; i < K; ++i)
      for (int64_t j = 0; j < N; ++j) bt[j * K + i] = B[i * N + j];
    DME_CUDA(cudaMemcpy2D(dBT, ldd * 8, bt.data(), K * 8, K * 8, N, cudaMemcpyHostToDevice));
    // A in the tiled image, as the E pass reads E
    oz_slice_rows_tiled(dA, ldd, M, K, qa, ea, pm, 0);
    oz_slice_rows(dBT, ldd, N, K, qb, ldq, OZ_NMAX * ldq, eb, pm, 0);
    OzGemmArgs g;
    g.A = qa; g.A_tiled = qa; g.eA = ea; g.lda = ldq; g.a_slice_stride = M * ldq;
    g.B = qb; g.eB = eb; g.ldb = ldq; g.b_slice_stride = OZ_NMAX * ldq;
    g.M = M; g.N = N; g.K = K;
    g.out = dC; g.out_rs = N; g.out_cs = 1;
    oz_gemm(g, ws, 0);
    DME_CUDA(cudaDeviceSynchronize());
    DME_CUDA(cudaMemcpy(C, dC, M * N * 8, cudaMemcpyDeviceToHost));
    cudaFree(dA); cudaFree(dBT); cudaFree(dC); cudaFree(part); cudaFree(cnt);
    cudaFree(qa); cudaFree(qb); cudaFree(ea); cudaFree(eb); cudaFree(pm);
  });
}

}  // extern "C"
