// nfft45.cu — C ABI (include/nfft45.h): node sets, forward NFFTs, Lagrange
// quantities, inverse plans and the type-4/5 solves with refinement.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <thread>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <tuple>
#include <numeric>
#include <set>
#include <string>
#include <vector>

#include "fft.cuh"
#include "ops.cuh"

namespace nfft45 {

std::atomic<int64_t> g_launches{0};
const bool g_debug_sync = getenv("NFFT45_DEBUG_SYNC") != nullptr;
const bool g_pdl = getenv("NFFT45_NO_PDL") == nullptr;
std::atomic<int> g_profiling{0};
static thread_local std::string tl_err;

// ------------------------------------------------- per-launch profiling
struct ProfRec {
  cudaEvent_t e0, e1;
  std::string name;
  bool used;
};
static std::mutex g_prof_mu;
static std::vector<ProfRec> g_prof;

int prof_begin(cudaStream_t st) {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  ProfRec r;
  if (cudaEventCreate(&r.e0) != cudaSuccess || cudaEventCreate(&r.e1) != cudaSuccess) return -1;
  r.used = false;
  cudaEventRecord(r.e0, st);
  g_prof.push_back(r);
  return (int)g_prof.size() - 1;
}

void prof_end(int slot, const char* name, cudaStream_t st) {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  if (slot < 0 || slot >= (int)g_prof.size()) return;
  g_prof[slot].name = name;
  g_prof[slot].used = true;
  cudaEventRecord(g_prof[slot].e1, st);
}

void set_error(int code, const std::string& msg) {
  (void)code;
  tl_err = msg;
}

int cuda_fail(cudaError_t e, const char* what) {
  tl_err = std::string("CUDA error in ") + what + ": " + cudaGetErrorString(e);
  return NFFT45_ERR_CUDA;
}

static int fail(int code, const std::string& msg) {
  tl_err = msg;
  return code;
}

// Restores the caller's current device on scope exit.
struct DeviceGuard {
  int prev = -1;
  int status = NFFT45_OK;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    cudaError_t e = cudaSetDevice(dev);
    if (e != cudaSuccess) status = cuda_fail(e, "cudaSetDevice");
    static std::once_flag once[64];
    if (status == NFFT45_OK && dev < 64) {
      std::call_once(once[dev], [dev]() {
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
          uint64_t thr = UINT64_MAX;
          cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
        }
      });
    }
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

// Stream-ordered scratch buffer.
struct Scratch {
  void* p = nullptr;
  cudaStream_t st;
  explicit Scratch(cudaStream_t s) : st(s) {}
  int alloc(size_t bytes) {
    if (bytes == 0) bytes = 16;
    cudaError_t e = cudaMallocAsync(&p, bytes, st);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMallocAsync");
    return NFFT45_OK;
  }
  double2* c() { return reinterpret_cast<double2*>(p); }
  double* d() { return reinterpret_cast<double*>(p); }
  ~Scratch() {
    if (p) cudaFreeAsync(p, st);
  }
};

// Lagrange guards (lagrange.py:25-29).
static const double kReVLimit = std::log(1.79769313486231570815e308) - 16.0;
static const double kDerivativeFloor = 1e-300;

}  // namespace nfft45

using namespace nfft45;

struct nfft45_grid {
  GridDev d;
};

// CUDA-graph cache for launch-bound solves (small P x batch): the second call
// with the same (kind, batch, passes, pointers) captures the launch sequence
// on a library-owned stream; later calls replay it with one graph launch.
struct GraphKey {
  int kind, passes;
  int64_t batch;
  const void* in;
  void* out;
  bool operator<(const GraphKey& o) const {
    return std::tie(kind, passes, batch, in, out) < std::tie(o.kind, o.passes, o.batch, o.in, o.out);
  }
};
struct GraphCache {
  std::mutex mu;
  std::map<GraphKey, cudaGraphExec_t> execs;
  std::map<GraphKey, int64_t> kernels;  // kernel nodes per graph (for nfft45_launch_count)
  std::map<GraphKey, int> seen;
};

struct nfft45_plan {
  GraphCache* gc = nullptr;
  const nfft45_grid* g;
  int64_t P;
  double a;
  int eta;
  int m;
  double2* tables;  // one allocation holding everything below
  double2 *v, *ks, *L, *dL, *nw, *decay, *coef;
  double2 *c5, *c4;  // ascending-node fused factors nw * cis(-/+ K t)
  double* rtab;      // real copies: decay, coef_scale, deconvolution (length P each)
  double *rdecay, *rcoef, *rdeconv;
  double *rdd, *rcd;  // deconv*decay, coef*deconv
  // tile-major copies for the batch-minor hybrid chain kernels (null when P has none)
  double *tdd = nullptr, *tcd = nullptr, *tdeconv = nullptr, *tdecay = nullptr, *tcoef = nullptr;
  double2* tks = nullptr;
};

// ------------------------------------------------------------- kernels

namespace nfft45 {

__global__ void k_log_series(double2* lam, int64_t R, double a) {
  int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (p >= R) return;
  // lagrange.py:52  lam[1:] = -exp(-2 pi p a) / p
  double v = p == 0 ? 0.0 : -exp(-2.0 * 3.141592653589793 * (double)p * a) / (double)p;
  lam[p] = make_double2(v, 0.0);
}

// ks = exp(i pi P + 2 pi i sum t + v) (lagrange.py:92-97).  The constant
// phase arrives in turns (from a double-double instant sum) and Im v is
// split into whole turns plus an exactly computed remainder, so the
// argument handed to sincospi is O(1) however large |Im v| grows.
__global__ void k_kernel_samples(const double2* __restrict__ v, double2* __restrict__ ks, int64_t P,
                                 double c_turns, double* __restrict__ max_re) {
  __shared__ double red[256];
  const double kTwoPiHi = 6.283185307179586232, kTwoPiLo = 2.4492935982947064e-16;
  const double kInvTwoPi = 0.15915494309189533577;
  double mx = 0.0;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < P; q += (int64_t)gridDim.x * blockDim.x) {
    double2 x = v[q];
    mx = fmax(mx, fabs(x.x));
    double tv = x.y * kInvTwoPi;
    double resid = fma(-tv, kTwoPiHi, x.y) - tv * kTwoPiLo;  // Im v - 2 pi tv
    double f = (tv - rint(tv)) + c_turns;
    f -= rint(f);
    double s, c;
    sincospi(2.0 * f + resid * 0.31830988618379067154, &s, &c);
    double mag = exp(x.x);
    ks[q] = make_double2(mag * c, mag * s);
  }
  red[threadIdx.x] = mx;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (threadIdx.x < w) red[threadIdx.x] = fmax(red[threadIdx.x], red[threadIdx.x + w]);
    __syncthreads();
  }
  if (threadIdx.x == 0) max_re[blockIdx.x] = red[0];
}

// Eq. 43: L = (FFT(ks) - P e^{-2 pi P a} delta_0) * e^{2 pi p a} / P, in place.
__global__ void k_coeff_fix(double2* L, int64_t P, double a) {
  int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (p >= P) return;
  double2 x = L[p];
  if (p == 0) x.x -= (double)P * exp(-2.0 * 3.141592653589793 * (double)P * a);
  double boost = exp(2.0 * 3.141592653589793 * (double)p * a);
  double s = boost / (double)P;
  L[p] = make_double2(x.x * s, x.y * s);
}

// dcoef_k = (k+1) L_{k+1} (k < P-1), dcoef_{P-1} = P (lagrange.py:150-152)
__global__ void k_dcoef(const double2* __restrict__ L, double2* __restrict__ d, int64_t P) {
  int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= P) return;
  if (k < P - 1) {
    double2 x = L[k + 1];
    double f = (double)(k + 1);
    d[k] = make_double2(f * x.x, f * x.y);
  } else {
    d[k] = make_double2((double)P, 0.0);
  }
}

__global__ void k_min_abs(const double2* __restrict__ x, int64_t n, double* __restrict__ out) {
  __shared__ double red[256];
  double mn = INFINITY;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    mn = fmin(mn, hypot(x[i].x, x[i].y));
  red[threadIdx.x] = mn;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (threadIdx.x < w) red[threadIdx.x] = fmin(red[threadIdx.x], red[threadIdx.x + w]);
    __syncthreads();
  }
  if (threadIdx.x == 0) out[blockIdx.x] = red[0];
}

// Plan scalars per node (inverse.py:70-78) and the fused solve factors.
__global__ void k_plan_tables(const double* __restrict__ t, const double* __restrict__ ts,
                              const int* __restrict__ perm, const double2* __restrict__ dL, int64_t P, double a,
                              double2* __restrict__ nw, double2* __restrict__ decay, double2* __restrict__ coef) {
  int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (q >= P) return;
  const double twopi = 2.0 * 3.141592653589793;
  // decay = e^{-2 pi p a}; coef_scale = (1/decay)/P
  double dec = exp(-twopi * (double)q * a);
  decay[q] = make_double2(dec, 0.0);
  coef[q] = make_double2((1.0 / dec) / (double)P, 0.0);
  // h = 1 / (cis(-P t) e^{-2 pi P a} - 1);  nw = h / (L' cis(t))
  double tq = t[q];
  double2 cpt = cis_turns(-turns_of_product((double)P, tq));
  double damp = exp(-twopi * (double)P * a);
  double2 den = make_double2(cpt.x * damp - 1.0, cpt.y * damp);
  double2 h = cdiv(make_double2(1.0, 0.0), den);
  double2 ct = cis_turns(tq >= 0.5 ? tq - 1.0 : tq);
  double2 w = cdiv(h, cmul(dL[q], ct));
  nw[q] = w;
}

// tile-major copies of the per-index solve tables for the P = R x C layout
// p = k + R m (chain_bm.cu): a chain tile then stages its slice as one
// contiguous run (the stride-R gather cost 16x the shared-memory wavefronts)
__global__ void k_tile_major_tables(int64_t P, int R, int C, const double* __restrict__ rdd,
                                    const double* __restrict__ rcd, const double* __restrict__ rdeconv,
                                    const double* __restrict__ rdecay, const double* __restrict__ rcoef,
                                    const double2* __restrict__ ks, double* __restrict__ tdd, double* __restrict__ tcd,
                                    double* __restrict__ tdeconv, double* __restrict__ tdecay,
                                    double* __restrict__ tcoef, double2* __restrict__ tks) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= P) return;
  {
    const int64_t k = i / C, m = i % C, p = k + (int64_t)R * m;
    tdd[i] = rdd[p];
    tcd[i] = rcd[p];
    tdeconv[i] = rdeconv[p];
    tdecay[i] = rdecay[p];
    tcoef[i] = rcoef[p];
  }
  {
    const int64_t r = i / R, k = i % R;
    tks[i] = ks[r + (int64_t)C * k];
  }
}

// real solve tables for the fused chains
__global__ void k_real_tables(const double2* __restrict__ decay, const double2* __restrict__ coef, int64_t P,
                              double b, double* __restrict__ rdecay, double* __restrict__ rcoef,
                              double* __restrict__ rdeconv, double* __restrict__ rdd, double* __restrict__ rcd) {
  int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (p >= P) return;
  const double dec = decay[p].x, cf = coef[p].x, dc = deconv_weight(p, P / 2, 2 * P, b);
  rdecay[p] = dec;
  rcoef[p] = cf;
  rdeconv[p] = dc;
  rdd[p] = dc * dec;
  rcd[p] = cf * dc;
}

__global__ void k_fused_factors(const double* __restrict__ ts, const int* __restrict__ perm,
                                const double2* __restrict__ nw, int64_t P, double K, double2* __restrict__ c5,
                                double2* __restrict__ c4) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= P) return;
  double x = turns_of_product(K, ts[i]);
  double2 w = nw[perm[i]];
  c5[i] = cmul(w, cis_turns(-x));
  c4[i] = cmul(w, cis_turns(x));
}

// max (or min) of the per-CTA partials: one CTA of 256 threads (max / min are exact and
// order-independent, so the tree gives the value of the serial loop it replaces, which took
// 40 us for 1024 partials: dependent L2 loads from one thread)
__global__ void k_max_reduce(const double* in, int n, double* out, int is_min) {
  __shared__ double red[256];
  double r = is_min ? INFINITY : 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) r = is_min ? fmin(r, in[i]) : fmax(r, in[i]);
  red[threadIdx.x] = r;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w)
      red[threadIdx.x] = is_min ? fmin(red[threadIdx.x], red[threadIdx.x + w]) : fmax(red[threadIdx.x], red[threadIdx.x + w]);
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = red[0];
}

}  // namespace nfft45

// ------------------------------------------------------- internal steps

namespace nfft45 {

static cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// A = type1(grid, a, R) (forward.py:26-64) with optional fold onto P,
// optional spectral table and optional subtraction: the shared backbone of
// nfft_type1, nonuniform_conv, compute_v_samples and the type-4 refinement.
static int type1_core(const GridDev& g, const double2* a, int64_t batch, int64_t R, int m, int64_t P,
                      const double2* tab, const double2* sub, double2* out, cudaStream_t st) {
  if (a && !tab && R == P && forward_bm_usable(g.Q, R, m, batch))  // batched: batch-minor passes
    return forward_run_bm(g, 1, a, batch, sub, out, st);
  const int64_t n = 2 * R;
  const int64_t K = R / 2;
  Window win = Window::make(m);
  Scratch H(st);
  NFFT_CHECK(H.alloc(sizeof(double2) * batch * n));
  NodeFactor f{nullptr, (double)K, -1};
  NFFT_CHECK(spread(g, n, win, a, batch, f, H.c(), st));
  NFFT_CHECK(fft_run(H.c(), H.c(), batch, n, -1, nullptr, nullptr, st));
  NFFT_CHECK(band_fold(H.c(), n, R, K, P, win, true, tab, sub, out, batch, st));
  return NFFT45_OK;
}

// s = type2(S, grid) (forward.py:67-102), optional subtraction.
static int type2_core(const GridDev& g, const double2* Sc, int64_t batch, int64_t P, int m, const double2* sub,
                      double2* out, cudaStream_t st) {
  if (forward_bm_usable(g.Q, P, m, batch)) return forward_run_bm(g, 2, Sc, batch, sub, out, st);  // batched
  const int64_t n = 2 * P;
  const int64_t K = P / 2;
  Window win = Window::make(m);
  Scratch F(st);
  NFFT_CHECK(F.alloc(sizeof(double2) * batch * n));
  NFFT_CHECK(band_pad(Sc, P, n, K, win, true, nullptr, F.c(), batch, st));
  NFFT_CHECK(fft_run(F.c(), F.c(), batch, n, +1, nullptr, nullptr, st));
  NodeFactor f{nullptr, (double)K, +1};
  NFFT_CHECK(gather(g, n, win, F.c(), batch, f, sub, out, st));
  return NFFT45_OK;
}

// R = number of log-series terms (eta P in the reference; any R >= 2 for the
// fractional-oversampling extension: the fold then sums a partial last slice).
static int v_core(const GridDev& g, double a, int64_t R, int m, double2* v, cudaStream_t st) {
  const int64_t P = g.Q;
  Scratch lam(st), V(st);
  NFFT_CHECK(lam.alloc(sizeof(double2) * R));
  NFFT_CHECK(V.alloc(sizeof(double2) * P));
  LAUNCH(k_log_series, (unsigned)ceil_div(R, 256), 256, 0, st, lam.c(), R, a);
  NFFT_CHECK(type1_core(g, nullptr, 1, R, m, P, lam.c(), nullptr, V.c(), st));
  NFFT_CHECK(fft_run(V.c(), v, 1, P, +1, nullptr, nullptr, st));
  return NFFT45_OK;
}

static double const_turns(const GridDev& g) {
  // i pi P + 2 pi i sum(t)  ->  turns P/2 + sum t  (mod 1)
  double half = (g.Q % 2) ? 0.5 : 0.0;
  double hi = g.sum_hi - std::rint(g.sum_hi);
  double c = (hi + half) + g.sum_lo;
  return c - std::rint(c);
}

static int ks_core(const GridDev& g, const double2* v, double2* ks, double* d_maxre, cudaStream_t st) {
  const int64_t P = g.Q;
  int blocks = (int)std::min<int64_t>(ceil_div(P, 256), 1024);
  Scratch part(st);
  NFFT_CHECK(part.alloc(sizeof(double) * blocks));
  LAUNCH(k_kernel_samples, blocks, 256, 0, st, v, ks, P, const_turns(g), part.d());
  LAUNCH(k_max_reduce, 1, 256, 0, st, part.d(), blocks, d_maxre, 0);
  return NFFT45_OK;
}

static int coeff_core(const double2* ks, int64_t P, double a, double2* L, cudaStream_t st) {
  NFFT_CHECK(fft_run(ks, L, 1, P, -1, nullptr, nullptr, st));
  LAUNCH(k_coeff_fix, (unsigned)ceil_div(P, 256), 256, 0, st, L, P, a);
  return NFFT45_OK;
}

static int deriv_core(const GridDev& g, const double2* L, int m, double2* dL, double* d_minabs, cudaStream_t st) {
  const int64_t P = g.Q;
  Scratch d(st), part(st);
  NFFT_CHECK(d.alloc(sizeof(double2) * P));
  LAUNCH(k_dcoef, (unsigned)ceil_div(P, 256), 256, 0, st, L, d.c(), P);
  NFFT_CHECK(type2_core(g, d.c(), 1, P, m, nullptr, dL, st));
  int blocks = (int)std::min<int64_t>(ceil_div(P, 256), 1024);
  NFFT_CHECK(part.alloc(sizeof(double) * blocks));
  LAUNCH(k_min_abs, blocks, 256, 0, st, dL, P, part.d());
  LAUNCH(k_max_reduce, 1, 256, 0, st, part.d(), blocks, d_minabs, 1);
  return NFFT45_OK;
}

static int check_guards(const double* d_guard, int have_re, int have_dl, cudaStream_t st) {
  double h[2] = {0.0, INFINITY};
  NFFT_CUDA(cudaMemcpyAsync(h, d_guard, sizeof(h), cudaMemcpyDeviceToHost, st));
  NFFT_CUDA(cudaStreamSynchronize(st));
  char buf[256];
  if (have_re && !(h[0] <= kReVLimit)) {
    snprintf(buf, sizeof buf,
             "|Re v| reaches %.1f, beyond the exp() overflow margin (%.1f); the grid is too strongly clustered "
             "for this damping",
             h[0], kReVLimit);
    return fail(NFFT45_ERR_KERNEL_OVERFLOW, buf);
  }
  if (have_dl && !(h[1] >= kDerivativeFloor)) {
    snprintf(buf, sizeof buf, "derivative sample magnitude %.3e below 1e-300; interpolation weights would overflow",
             h[1]);
    return fail(NFFT45_ERR_SINGULAR_DERIVATIVE, buf);
  }
  return NFFT45_OK;
}

// ------------------------------------------------------------- solves

static ChainPlanView chain_view(const nfft45_plan* p) {
  ChainPlanView v;
  v.g = &p->g->d;
  v.P = p->P;
  v.ks = p->ks;
  v.c5 = p->c5;
  v.c4 = p->c4;
  v.decay = p->rdecay;
  v.coef = p->rcoef;
  v.deconv = p->rdeconv;
  v.dd = p->rdd;
  v.cd = p->rcd;
  v.tdd = p->tdd;
  v.tcd = p->tcd;
  v.tdeconv = p->tdeconv;
  v.tdecay = p->tdecay;
  v.tcoef = p->tcoef;
  v.tks = p->tks;
  return v;
}

static bool use_chain(const nfft45_plan* p, int64_t batch) {
  static const bool off = getenv("NFFT45_NO_CHAIN") != nullptr;  // A/B switch for tests
  return !off && chain_usable(p->P, p->m, batch);
}

static int type5_core(const nfft45_plan* p, const double2* s, int64_t batch, double2* out, cudaStream_t st) {
  if (use_chain(p, batch)) return chain_run(chain_view(p), 5, s, batch, 0, out, nullptr, st);
  const GridDev& g = p->g->d;
  const int64_t P = p->P, n = 2 * P, K = P / 2;
  Window win = Window::make(p->m);
  Scratch H(st), V(st);
  NFFT_CHECK(H.alloc(sizeof(double2) * batch * n));
  NFFT_CHECK(V.alloc(sizeof(double2) * batch * P));
  NodeFactor f{p->c5, 0.0, 0};
  NFFT_CHECK(spread(g, n, win, s, batch, f, H.c(), st));                                  // forward.py:47-54
  NFFT_CHECK(fft_run(H.c(), H.c(), batch, n, -1, nullptr, nullptr, st));                  // forward.py:55
  NFFT_CHECK(band_fold(H.c(), n, P, K, P, win, true, p->decay, nullptr, V.c(), batch, st));  // :64, :153
  NFFT_CHECK(fft_run(V.c(), V.c(), batch, P, +1, nullptr, p->ks, st));                    // :162, inverse.py:114
  NFFT_CHECK(fft_run(V.c(), out, batch, P, -1, nullptr, p->coef, st));                    // inverse.py:115
  return NFFT45_OK;
}

static int type4_core(const nfft45_plan* p, const double2* A, int64_t batch, double2* out, cudaStream_t st) {
  if (use_chain(p, batch)) return chain_run(chain_view(p), 4, A, batch, 0, out, nullptr, st);
  const GridDev& g = p->g->d;
  const int64_t P = p->P, n = 2 * P, K = P / 2;
  Window win = Window::make(p->m);
  Scratch V(st), F(st);
  NFFT_CHECK(V.alloc(sizeof(double2) * batch * P));
  NFFT_CHECK(F.alloc(sizeof(double2) * batch * n));
  NFFT_CHECK(fft_run(A, V.c(), batch, P, +1, p->decay, p->ks, st));       // inverse.py:132-133
  NFFT_CHECK(fft_run(V.c(), V.c(), batch, P, -1, nullptr, p->coef, st));   // inverse.py:134
  NFFT_CHECK(band_pad(V.c(), P, n, K, win, true, nullptr, F.c(), batch, st));  // forward.py:88-89
  NFFT_CHECK(fft_run(F.c(), F.c(), batch, n, +1, nullptr, nullptr, st));  // forward.py:90
  NodeFactor f{p->c4, 0.0, 0};
  NFFT_CHECK(gather(g, n, win, F.c(), batch, f, nullptr, out, st));        // forward.py:91-102, inverse.py:143
  return NFFT45_OK;
}

typedef int (*SolveFn)(const nfft45_plan*, const double2*, int64_t, double2*, cudaStream_t);

// Section V refinement (inverse.py:146-162).  fwd5: residual via type-2
// (sample domain) else via type-1 of length P (spectrum domain).
static int check_norms(const double* d_norms, int64_t batch, int passes, cudaStream_t st) {
  std::vector<double> h((size_t)batch * passes);
  NFFT_CUDA(cudaMemcpyAsync(h.data(), d_norms, sizeof(double) * h.size(), cudaMemcpyDeviceToHost, st));
  NFFT_CUDA(cudaStreamSynchronize(st));
  for (int pass = 1; pass < passes; pass++)
    for (int64_t b = 0; b < batch; b++) {
      double prev = h[(size_t)(pass - 1) * batch + b], cur = h[(size_t)pass * batch + b];
      if (cur > prev) {
        char buf[200];
        snprintf(buf, sizeof buf,
                 "residual norm grew between passes (%.3e -> %.3e); method error >= 1 at these parameters", prev,
                 cur);
        return fail(NFFT45_ERR_NON_CONVERGENCE, buf);
      }
    }
  return NFFT45_OK;
}

static int refine_core(const nfft45_plan* p, const double2* data, int64_t batch, int passes, double2* out,
                       bool type5, cudaStream_t st) {
  if (use_chain(p, batch)) {
    Scratch norms(st);
    if (passes >= 2) NFFT_CHECK(norms.alloc(sizeof(double) * batch * passes));
    NFFT_CHECK(chain_run(chain_view(p), type5 ? 5 : 4, data, batch, passes, out, passes >= 2 ? norms.d() : nullptr,
                         st));
    if (passes >= 2) return check_norms(norms.d(), batch, passes, st);
    return NFFT45_OK;
  }
  SolveFn solve = type5 ? type5_core : type4_core;
  NFFT_CHECK(solve(p, data, batch, out, st));
  if (passes <= 0) return NFFT45_OK;
  const GridDev& g = p->g->d;
  const int64_t P = p->P;
  Scratch r(st), y(st), norms(st);
  NFFT_CHECK(r.alloc(sizeof(double2) * batch * P));
  NFFT_CHECK(y.alloc(sizeof(double2) * batch * P));
  NFFT_CHECK(norms.alloc(sizeof(double) * batch * passes));
  for (int pass = 0; pass < passes; pass++) {
    if (type5) NFFT_CHECK(type2_core(g, out, batch, P, p->m, data, r.c(), st));
    else NFFT_CHECK(type1_core(g, out, batch, P, p->m, P, nullptr, data, r.c(), st));
    if (passes >= 2) NFFT_CHECK(row_norms(r.c(), P, batch, norms.d() + (int64_t)pass * batch, st));
    NFFT_CHECK(solve(p, r.c(), batch, y.c(), st));
    NFFT_CHECK(csub_batch(out, y.c(), out, batch * P, st));
  }
  if (passes >= 2) {
    std::vector<double> h((size_t)batch * passes);
    NFFT_CUDA(cudaMemcpyAsync(h.data(), norms.d(), sizeof(double) * h.size(), cudaMemcpyDeviceToHost, st));
    NFFT_CUDA(cudaStreamSynchronize(st));
    for (int pass = 1; pass < passes; pass++)
      for (int64_t b = 0; b < batch; b++) {
        double prev = h[(size_t)(pass - 1) * batch + b], cur = h[(size_t)pass * batch + b];
        if (cur > prev) {
          char buf[200];
          snprintf(buf, sizeof buf,
                   "residual norm grew between passes (%.3e -> %.3e); method error >= 1 at these parameters", prev,
                   cur);
          return fail(NFFT45_ERR_NON_CONVERGENCE, buf);
        }
      }
  }
  return NFFT45_OK;
}

}  // namespace nfft45

namespace nfft45 {

// per-thread library stream used for capture / replay (forked from and joined
// back to the caller's stream with events)
static cudaStream_t lib_stream() {
  static thread_local cudaStream_t s[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) return nullptr;
  if (!s[dev]) cudaStreamCreateWithFlags(&s[dev], cudaStreamNonBlocking);
  return s[dev];
}

// set by the host pipeline around its solves (see nfft45_solve_host)
static thread_local bool tl_host_pipe_no_graph = false;

static bool graph_eligible(const nfft45_plan* p, int64_t batch, int passes) {
  static const bool off = getenv("NFFT45_NO_GRAPH") != nullptr;
  // per-kernel profiling needs the individual launches (graph replays bypass LAUNCH)
  return !off && !tl_host_pipe_no_graph && !g_profiling.load(std::memory_order_relaxed) && passes <= 1 && p->P * batch <= (int64_t(1) << 22);
}

// run `fn(stream)` directly, or capture/replay it as a CUDA graph
template <class Fn>
static int run_graphed(const nfft45_plan* p, int kind, int64_t batch, int passes, const void* in, void* out,
                       cudaStream_t user, const Fn& fn) {
  if (!graph_eligible(p, batch, passes)) return fn(user);
  nfft45_plan* mp = const_cast<nfft45_plan*>(p);
  GraphKey key{kind, passes, batch, in, out};
  cudaGraphExec_t exec = nullptr;
  bool capture = false;
  int64_t nkern = 0;
  {
    std::lock_guard<std::mutex> lk(mp->gc->mu);
    auto it = mp->gc->execs.find(key);
    if (it != mp->gc->execs.end()) {
      exec = it->second;
      nkern = mp->gc->kernels[key];
    }
    else if (mp->gc->execs.size() < 64) {
      // `seen` only counts keys while the cache can still take a graph, and is
      // trimmed so a long-lived plan fed fresh output pointers stays bounded
      if (mp->gc->seen.size() >= 512) mp->gc->seen.clear();
      if (++mp->gc->seen[key] >= 2) {
        capture = true;
        mp->gc->seen.erase(key);
      }
    }
  }
  if (!exec && !capture) return fn(user);
  if (exec) {  // replay straight into the caller's stream (independent solves on different streams overlap)
    NFFT_CUDA(cudaGraphLaunch(exec, user));
    g_launches.fetch_add(nkern, std::memory_order_relaxed);
    return NFFT45_OK;
  }
  cudaStream_t ls = lib_stream();
  if (!ls) return fn(user);
  cudaEvent_t e0, e1;
  NFFT_CUDA(cudaEventCreateWithFlags(&e0, cudaEventDisableTiming));
  NFFT_CUDA(cudaEventCreateWithFlags(&e1, cudaEventDisableTiming));
  int status = NFFT45_OK;
  NFFT_CUDA(cudaEventRecord(e0, user));
  NFFT_CUDA(cudaStreamWaitEvent(ls, e0, 0));
  if (!exec) {
    cudaGraph_t graph = nullptr;
    NFFT_CUDA(cudaStreamBeginCapture(ls, cudaStreamCaptureModeThreadLocal));
    status = fn(ls);
    cudaError_t ce = cudaStreamEndCapture(ls, &graph);
    if (status == NFFT45_OK && ce == cudaSuccess) {
      size_t nn = 0;
      cudaGraphGetNodes(graph, nullptr, &nn);
      std::vector<cudaGraphNode_t> nodes(nn);
      if (nn) cudaGraphGetNodes(graph, nodes.data(), &nn);
      for (auto nd : nodes) {
        cudaGraphNodeType ty;
        if (cudaGraphNodeGetType(nd, &ty) == cudaSuccess && ty == cudaGraphNodeTypeKernel) nkern++;
      }
      // the captured launches were counted by LAUNCH already; replays add nkern each
      ce = cudaGraphInstantiate(&exec, graph, 0);
      if (ce != cudaSuccess) {
        // could not instantiate: drop the capture and run directly on the caller's stream
        exec = nullptr;
        cudaGraphDestroy(graph);
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        cudaGetLastError();
        return fn(user);
      }
      {
        std::lock_guard<std::mutex> lk(mp->gc->mu);
        auto it = mp->gc->execs.find(key);
        if (it == mp->gc->execs.end()) {
          mp->gc->execs[key] = exec;
          mp->gc->kernels[key] = nkern;
        } else {
          cudaGraphExecDestroy(exec);
          exec = it->second;
        }
      }
      NFFT_CUDA(cudaGraphLaunch(exec, ls));
      NFFT_CUDA(cudaEventRecord(e1, ls));
      NFFT_CUDA(cudaStreamWaitEvent(user, e1, 0));
      cudaEventDestroy(e0);
      cudaEventDestroy(e1);
      if (graph) cudaGraphDestroy(graph);
      return status;
    }
    if (graph) cudaGraphDestroy(graph);
    if (status != NFFT45_OK || ce != cudaSuccess || !exec) {
      cudaGetLastError();
      // fall back to a direct run on the caller's stream
      cudaEventDestroy(e0);
      cudaEventDestroy(e1);
      return status != NFFT45_OK ? status : fn(user);
    }
  }
  NFFT_CUDA(cudaGraphLaunch(exec, ls));
  g_launches.fetch_add(nkern, std::memory_order_relaxed);
  NFFT_CUDA(cudaEventRecord(e1, ls));
  NFFT_CUDA(cudaStreamWaitEvent(user, e1, 0));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  return status;
}

}  // namespace nfft45

namespace nfft45 {
void host_pipes_forget(const nfft45_plan* p);
}

// ================================================================== C ABI

namespace nfft45 {
// Rows per kernel launch: several launch paths put the row count in
// gridDim.y (capped at 65535), so every batched C entry point walks its rows
// in slices of at most kMaxRows (rows are independent solves / transforms).
constexpr int64_t kMaxRows = 65535;
template <class F>
static int by_rows(int64_t batch, const F& f) {
  if (batch <= kMaxRows) return f((int64_t)0, batch);
  for (int64_t b0 = 0; b0 < batch; b0 += kMaxRows) NFFT_CHECK(f(b0, std::min(kMaxRows, batch - b0)));
  return NFFT45_OK;
}
}  // namespace nfft45

extern "C" {

const char* nfft45_last_error(void) { return tl_err.c_str(); }
int nfft45_version(void) { return 100; }
int64_t nfft45_launch_count(void) { return g_launches.load(); }

int nfft45_profile_enable(int on) {
  g_profiling.store(on ? 1 : 0);
  return NFFT45_OK;
}

int nfft45_profile_read(char* buf, int64_t cap) {
  // synchronizes on every recorded event; emits "name count total_ms\n" lines
  std::lock_guard<std::mutex> lk(g_prof_mu);
  std::vector<std::pair<std::string, std::pair<int64_t, double>>> agg;
  for (auto& r : g_prof) {
    float ms = 0.f;
    if (r.used && cudaEventSynchronize(r.e1) == cudaSuccess && cudaEventElapsedTime(&ms, r.e0, r.e1) == cudaSuccess) {
      bool found = false;
      for (auto& a : agg)
        if (a.first == r.name) { a.second.first++; a.second.second += ms; found = true; break; }
      if (!found) agg.push_back({r.name, {1, (double)ms}});
    }
    cudaEventDestroy(r.e0);
    cudaEventDestroy(r.e1);
  }
  g_prof.clear();
  std::string out;
  for (auto& a : agg) {
    char line[512];
    snprintf(line, sizeof line, "%s %lld %.6f\n", a.first.c_str(), (long long)a.second.first, a.second.second);
    out += line;
  }
  if (buf && cap > 0) {
    size_t n = std::min<size_t>(out.size(), (size_t)cap - 1);
    memcpy(buf, out.data(), n);
    buf[n] = 0;
  }
  return (int)out.size();
}

int nfft45_validate_grid(const double* t, int64_t Q, double min_gap, int64_t* order) {
  char buf[256];
  if (Q < 1 || !t) return fail(NFFT45_ERR_OUT_OF_RANGE, "grid must be a nonempty 1-D sequence of instants");
  for (int64_t i = 0; i < Q; i++)
    if (!std::isfinite(t[i])) return fail(NFFT45_ERR_OUT_OF_RANGE, "grid contains non-finite instants");
  for (int64_t i = 0; i < Q; i++)
    if (t[i] < 0.0 || t[i] >= 1.0) {
      snprintf(buf, sizeof buf, "instant %.17g outside the fundamental period [0, 1)", t[i]);
      return fail(NFFT45_ERR_OUT_OF_RANGE, buf);
    }
  std::vector<int64_t> ord((size_t)Q);
  std::iota(ord.begin(), ord.end(), 0);
  std::stable_sort(ord.begin(), ord.end(), [&](int64_t a, int64_t b) { return t[a] < t[b]; });
  if (Q > 1) {
    double gmin = INFINITY;
    int64_t at = 0;
    for (int64_t i = 0; i < Q; i++) {
      double gap = i + 1 < Q ? t[ord[i + 1]] - t[ord[i]] : 1.0 - t[ord[Q - 1]] + t[ord[0]];
      if (gap < gmin) { gmin = gap; at = i; }
    }
    if (gmin < min_gap) {
      snprintf(buf, sizeof buf, "circular gap %.3e below floor %.3e near t=%.17g", gmin, min_gap, t[ord[at]]);
      return fail(NFFT45_ERR_DUPLICATE_NODE, buf);
    }
  }
  if (order) std::copy(ord.begin(), ord.end(), order);
  return NFFT45_OK;
}

int nfft45_grid_create(const double* t, const int64_t* order, int64_t Q, int device, nfft45_grid** out) {
  if (!out || !t || !order || Q < 1) return fail(NFFT45_ERR_INVALID_ARGUMENT, "invalid grid arguments");
  if (Q > (int64_t)1 << 30) return fail(NFFT45_ERR_INVALID_ARGUMENT, "grid too large (max 2^30 nodes)");
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    return fail(NFFT45_ERR_NO_DEVICE, "no CUDA device available (the product path has no CPU fallback)");
  DeviceGuard dg(device);
  if (dg.status) return dg.status;
  std::vector<double> ts((size_t)Q);
  std::vector<int> perm((size_t)Q);
  for (int64_t i = 0; i < Q; i++) {
    perm[i] = (int)order[i];
    ts[i] = t[order[i]];
  }
  // double-double running sum of the instants (caller order; lagrange.py:92)
  double hi = 0.0, lo = 0.0;
  for (int64_t i = 0; i < Q; i++) {
    double s = hi + t[i];
    double bb = s - hi;
    double err = (hi - (s - bb)) + (t[i] - bb);
    hi = s;
    lo += err;
  }
  nfft45_grid* g = new nfft45_grid();
  g->d.device = device;
  g->d.Q = Q;
  g->d.sum_hi = hi;
  g->d.sum_lo = lo;
  g->d.rc = range_cache_new();
  size_t bytes = sizeof(double) * 2 * Q + sizeof(int) * Q;
  char* base = nullptr;
  cudaError_t e = cudaMalloc(&base, bytes);
  if (e != cudaSuccess) {
    tile_ranges_free(g->d);
    delete g;
    return cuda_fail(e, "cudaMalloc(grid)");
  }
  g->d.t = reinterpret_cast<double*>(base);
  g->d.ts = g->d.t + Q;
  g->d.perm = reinterpret_cast<int*>(g->d.ts + Q);
  e = cudaMemcpy(g->d.t, t, sizeof(double) * Q, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(g->d.ts, ts.data(), sizeof(double) * Q, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(g->d.perm, perm.data(), sizeof(int) * Q, cudaMemcpyHostToDevice);
  if (e != cudaSuccess) {
    cudaFree(base);
    tile_ranges_free(g->d);
    delete g;
    return cuda_fail(e, "cudaMemcpy(grid)");
  }
  *out = g;
  return NFFT45_OK;
}

void nfft45_grid_destroy(nfft45_grid* g) {
  if (!g) return;
  DeviceGuard dg(g->d.device);
  tile_ranges_free(g->d);
  cudaFree(g->d.t);
  delete g;
}

int64_t nfft45_grid_size(const nfft45_grid* g) { return g ? g->d.Q : 0; }

#define C2(p) reinterpret_cast<const double2*>(p)
#define D2(p) reinterpret_cast<double2*>(p)

int nfft45_type1(const nfft45_grid* g, const double* a, int64_t batch, int64_t R, int m, double* out, void* st) {
  if (!g || R < 1 || m < 1) return fail(NFFT45_ERR_INVALID_ARGUMENT, "invalid type-1 arguments");
  DeviceGuard dg(g->d.device);
  if (dg.status) return dg.status;
  const int64_t Q = g->d.Q;
  return by_rows(batch, [&](int64_t b0, int64_t nb) {
    return type1_core(g->d, C2(a) + b0 * Q, nb, R, m, R, nullptr, nullptr, D2(out) + b0 * R, S(st));
  });
}

int nfft45_type2(const nfft45_grid* g, const double* Sc, int64_t batch, int64_t P, int m, double* out, void* st) {
  if (!g || P < 1 || m < 1) return fail(NFFT45_ERR_INVALID_ARGUMENT, "invalid type-2 arguments");
  DeviceGuard dg(g->d.device);
  if (dg.status) return dg.status;
  const int64_t Q = g->d.Q;
  return by_rows(batch, [&](int64_t b0, int64_t nb) {
    return type2_core(g->d, C2(Sc) + b0 * P, nb, P, m, nullptr, D2(out) + b0 * Q, S(st));
  });
}

int nfft45_nonuniform_conv(const nfft45_grid* g, const double* a, int64_t batch, const double* lam, int64_t R,
                           int64_t P, int m, double* out, void* st) {
  if (!g || P < 1 || R < 1 || m < 1) return fail(NFFT45_ERR_INVALID_ARGUMENT, "invalid convolution arguments");
  if (R % P) {
    char buf[160];
    snprintf(buf, sizeof buf, "kernel length %lld is not a multiple of output length %lld", (long long)R,
             (long long)P);
    return fail(NFFT45_ERR_SIZE_MISMATCH, buf);
  }
  DeviceGuard dg(g->d.device);
  if (dg.status) return dg.status;
  cudaStream_t s = S(st);
  const int64_t Q = g->d.Q;
  return by_rows(batch, [&](int64_t b0, int64_t nb) {
    Scratch V(s);
    NFFT_CHECK(V.alloc(sizeof(double2) * nb * P));
    NFFT_CHECK(type1_core(g->d, C2(a) + b0 * Q, nb, R, m, P, C2(lam), nullptr, V.c(), s));
    return fft_run(V.c(), D2(out) + b0 * P, nb, P, +1, nullptr, nullptr, s);
  });
}

// cg_solve(grid, rhs, which, tol, max_iter, spread_width) — baselines.py:108-181.
namespace {
struct GridCgOps final : CgOps {
  const GridDev& g;
  int64_t P;
  int m;
  bool type4;
  GridCgOps(const GridDev& g_, int64_t P_, int m_, bool t4) : g(g_), P(P_), m(m_), type4(t4) {}
  int t1(const double2* in, double2* out, int64_t batch, cudaStream_t st) const {
    return type1_core(g, in, batch, P, m, P, nullptr, nullptr, out, st);
  }
  int t2(const double2* in, double2* out, int64_t batch, cudaStream_t st) const {
    return type2_core(g, in, batch, P, m, nullptr, out, st);
  }
  int A(const double2* in, double2* out, int64_t batch, cudaStream_t st) const override {
    return type4 ? t1(in, out, batch, st) : t2(in, out, batch, st);
  }
  int AH(const double2* in, double2* out, int64_t batch, cudaStream_t st) const override {
    return type4 ? t2(in, out, batch, st) : t1(in, out, batch, st);
  }
};
}  // namespace

int nfft45_cg_solve(const nfft45_grid* g, int kind, const double* rhs, int64_t batch, double tol, int64_t max_iter,
                    int m, double* x, int64_t* iterations, int* converged, double* relres, int* stalled, void* st) {
  if (!g || batch < 0 || m < 1 || max_iter < 0 || !iterations || !converged || !relres)
    return fail(NFFT45_ERR_INVALID_ARGUMENT, "invalid cg_solve arguments");
  if (!(tol > 0.0)) return fail(NFFT45_ERR_INVALID_ARGUMENT, "tolerance must be positive");
  if (kind != 4 && kind != 5) return fail(NFFT45_ERR_INVALID_ARGUMENT, "unknown system kind");
  DeviceGuard dg(g->d.device);
  if (dg.status) return dg.status;
  GridCgOps ops(g->d, g->d.Q, m, kind == 4);
  return cg_run(ops, C2(rhs), batch, g->d.Q, tol, max_iter, D2(x), iterations, converged, relres, stalled, S(st));
}

int nfft45_ge_solve(double* A, double* b, int64_t n, double* x, double pivot_floor, int64_t* bad_step,
                    double* bad_pivot, void* st) {
  if (!A || !b || !x || n < 1 || !bad_step || !bad_pivot)
    return fail(NFFT45_ERR_INVALID_ARGUMENT, "invalid ge_solve arguments");
  int dev = 0;
  cudaGetDevice(&dev);
  DeviceGuard dg(dev);
  if (dg.status) return dg.status;
  NFFT_CHECK(ge_run(D2(A), D2(b), n, D2(x), pivot_floor, bad_step, bad_pivot, S(st)));
  if (*bad_step < n) {
    char buf[96];
    if (*bad_step < n - 1)
      snprintf(buf, sizeof buf, "pivot %.3e below %.0e", *bad_pivot, pivot_floor);
    else
      snprintf(buf, sizeof buf, "matrix is numerically singular");
    return fail(NFFT45_ERR_SINGULAR_MATRIX, buf);
  }
  return NFFT45_OK;
}

int nfft45_type1_direct(const nfft45_grid* g, const double* a, int64_t batch, int64_t R, double* out, void* st) {
  if (!g || R < 1) return fail(NFFT45_ERR_INVALID_ARGUMENT, "invalid direct type-1 arguments");
  DeviceGuard dg(g->d.device);
  if (dg.status) return dg.status;
  const int64_t Q = g->d.Q;
  return by_rows(batch, [&](int64_t b0, int64_t nb) {
    return direct_type1(g->d, C2(a) + b0 * Q, nb, R, D2(out) + b0 * R, S(st));
  });
}

int nfft45_type2_direct(const nfft45_grid* g, const double* Sc, int64_t batch, int64_t P, double* out, void* st) {
  if (!g || P < 1) return fail(NFFT45_ERR_INVALID_ARGUMENT, "invalid direct type-2 arguments");
  DeviceGuard dg(g->d.device);
  if (dg.status) return dg.status;
  const int64_t Q = g->d.Q;
  return by_rows(batch, [&](int64_t b0, int64_t nb) {
    return direct_type2(g->d, C2(Sc) + b0 * P, nb, P, D2(out) + b0 * Q, S(st));
  });
}

int nfft45_dft(const double* in, double* out, int64_t batch, int64_t N, int sign, void* st) {
  if (N < 1) return fail(NFFT45_ERR_INVALID_ARGUMENT, "DFT length must be >= 1");
  // current device: the guard's first use keeps freed scratch in the stream-ordered pool (a process
  // that only calls the DFT entry points would otherwise re-map its scratch on every call)
  int dev = 0;
  NFFT_CUDA(cudaGetDevice(&dev));
  DeviceGuard dg(dev);
  if (dg.status) return dg.status;
  return by_rows(batch, [&](int64_t b0, int64_t nb) {
    return fft_run(C2(in) + b0 * N, D2(out) + b0 * N, nb, N, sign, nullptr, nullptr, S(st));
  });
}

int nfft45_v_samples(const nfft45_grid* g, double a, int eta, int m, double* v, void* st) {
  if (!g || eta < 1 || m < 1) return fail(NFFT45_ERR_INVALID_ARGUMENT, "invalid v-samples arguments");
  return nfft45_v_samples_terms(g, a, (int64_t)eta * g->d.Q, m, v, st);
}

int nfft45_v_samples_terms(const nfft45_grid* g, double a, int64_t R, int m, double* v, void* st) {
  if (!g || m < 1) return fail(NFFT45_ERR_INVALID_ARGUMENT, "invalid v-samples arguments");
  if (R < 2) return fail(NFFT45_ERR_INVALID_ARGUMENT, "need eta * P >= 2 so the truncated series has at least one term");
  DeviceGuard dg(g->d.device);
  if (dg.status) return dg.status;
  return v_core(g->d, a, R, m, D2(v), S(st));
}

int nfft45_kernel_samples(const nfft45_grid* g, const double* v, double* ks, void* st) {
  if (!g) return fail(NFFT45_ERR_INVALID_ARGUMENT, "invalid grid");
  DeviceGuard dg(g->d.device);
  if (dg.status) return dg.status;
  cudaStream_t s = S(st);
  Scratch guard(s);
  NFFT_CHECK(guard.alloc(sizeof(double) * 2));
  NFFT_CHECK(ks_core(g->d, C2(v), D2(ks), guard.d(), s));
  return check_guards(guard.d(), 1, 0, s);
}

int nfft45_kernel_coefficients(const double* ks, int64_t P, double a, double* L, void* st) {
  if (P < 1) return fail(NFFT45_ERR_INVALID_ARGUMENT, "invalid coefficient arguments");
  return coeff_core(C2(ks), P, a, D2(L), S(st));
}

int nfft45_derivative_coefficients(const double* L, int64_t P, double* d, void* st) {
  if (P < 1) return fail(NFFT45_ERR_INVALID_ARGUMENT, "invalid coefficient length");
  LAUNCH(k_dcoef, (unsigned)ceil_div(P, 256), 256, 0, S(st), C2(L), D2(d), P);
  return NFFT45_OK;
}

int nfft45_min_abs(const double* x, int64_t n, double* out, void* st) {
  if (n < 1 || !out) return fail(NFFT45_ERR_INVALID_ARGUMENT, "invalid min-abs arguments");
  cudaStream_t s = S(st);
  int blocks = (int)std::min<int64_t>(ceil_div(n, 256), 1024);
  Scratch part(s), res(s);
  NFFT_CHECK(part.alloc(sizeof(double) * blocks));
  NFFT_CHECK(res.alloc(sizeof(double)));
  LAUNCH(k_min_abs, blocks, 256, 0, s, C2(x), n, part.d());
  LAUNCH(k_max_reduce, 1, 256, 0, s, part.d(), blocks, res.d(), 1);
  NFFT_CUDA(cudaMemcpyAsync(out, res.d(), sizeof(double), cudaMemcpyDeviceToHost, s));
  NFFT_CUDA(cudaStreamSynchronize(s));
  return NFFT45_OK;
}

int nfft45_derivative_samples(const nfft45_grid* g, const double* L, int m, double* dL, void* st) {
  if (!g || m < 1) return fail(NFFT45_ERR_INVALID_ARGUMENT, "invalid derivative arguments");
  DeviceGuard dg(g->d.device);
  if (dg.status) return dg.status;
  cudaStream_t s = S(st);
  Scratch guard(s);
  NFFT_CHECK(guard.alloc(sizeof(double) * 2));
  NFFT_CHECK(deriv_core(g->d, C2(L), m, D2(dL), guard.d() + 1, s));
  return check_guards(guard.d(), 0, 1, s);
}

int nfft45_plan_create(const nfft45_grid* g, double a, int eta, int m, void* st, nfft45_plan** out) {
  if (!g || !out) return fail(NFFT45_ERR_INVALID_ARGUMENT, "invalid plan arguments");
  if (eta < 1 || m < 1) return fail(NFFT45_ERR_INVALID_ARGUMENT, "eta and m must be >= 1");
  return nfft45_plan_create_terms(g, a, (int64_t)eta * g->d.Q, m, st, out);
}

int nfft45_plan_create_terms(const nfft45_grid* g, double a, int64_t R, int m, void* st, nfft45_plan** out) {
  if (!g || !out) return fail(NFFT45_ERR_INVALID_ARGUMENT, "invalid plan arguments");
  if (!(a > 0.0)) return fail(NFFT45_ERR_NON_POSITIVE_DAMPING, "damping must be positive");
  if (m < 1) return fail(NFFT45_ERR_INVALID_ARGUMENT, "eta and m must be >= 1");
  const int64_t P = g->d.Q;
  if (R < 2)
    return fail(NFFT45_ERR_INVALID_ARGUMENT, "need eta * P >= 2 so the truncated series has at least one term");
  const int eta = (int)((R + P - 1) / P);
  DeviceGuard dg(g->d.device);
  if (dg.status) return dg.status;
  cudaStream_t s = S(st);
  static const bool timing = getenv("NFFT45_PLAN_TIMING") != nullptr;  // host-side breakdown (probe)
  auto now = [] { return std::chrono::steady_clock::now(); };
  auto ms = [](std::chrono::steady_clock::time_point a, std::chrono::steady_clock::time_point b) {
    return std::chrono::duration<double, std::milli>(b - a).count();
  };
  const auto T0 = now();
  nfft45_plan* p = new nfft45_plan();
  p->gc = new GraphCache();
  p->g = g;
  p->P = P;
  p->a = a;
  p->eta = eta;
  p->m = m;
  // stream-ordered pool allocation (release threshold infinite, DeviceGuard):
  // a rebuilt plan reuses pooled memory instead of a fresh cudaMalloc (1-20 ms
  // for the 184 MB of tables at P = 2^20); the build ends with a stream
  // synchronize (check_guards), after which every stream may use the tables
  int hR = 0, hC = 0;
  const bool tile_major = m == kFastM && chain_bm_hybrid_factors(P, &hR, &hC);
  cudaError_t e = cudaMallocAsync(&p->tables, sizeof(double2) * (9 + (tile_major ? 1 : 0)) * P +
                                                  sizeof(double) * (5 + (tile_major ? 5 : 0)) * P, s);
  if (e != cudaSuccess) {
    delete p;
    return cuda_fail(e, "cudaMalloc(plan)");
  }
  p->rtab = reinterpret_cast<double*>(p->tables + (9 + (tile_major ? 1 : 0)) * P);
  if (tile_major) {
    p->tks = p->tables + 9 * P;
    p->tdd = p->rtab + 5 * P;
    p->tcd = p->rtab + 6 * P;
    p->tdeconv = p->rtab + 7 * P;
    p->tdecay = p->rtab + 8 * P;
    p->tcoef = p->rtab + 9 * P;
  }
  p->rdecay = p->rtab;
  p->rcoef = p->rtab + P;
  p->rdeconv = p->rtab + 2 * P;
  p->rdd = p->rtab + 3 * P;
  p->rcd = p->rtab + 4 * P;
  double2* t = p->tables;
  p->v = t;
  p->ks = t + P;
  p->L = t + 2 * P;
  p->dL = t + 3 * P;
  p->nw = t + 4 * P;
  p->decay = t + 5 * P;
  p->coef = t + 6 * P;
  p->c5 = t + 7 * P;
  p->c4 = t + 8 * P;
  int status = NFFT45_OK;
  const auto T1 = now();
  {
    Scratch guard(s);
    status = guard.alloc(sizeof(double) * 2);
    if (!status) status = v_core(g->d, a, R, m, p->v, s);
    if (!status) status = ks_core(g->d, p->v, p->ks, guard.d(), s);
    if (!status) status = coeff_core(p->ks, P, a, p->L, s);
    if (!status) status = deriv_core(g->d, p->L, m, p->dL, guard.d() + 1, s);
    if (!status) {
      k_plan_tables<<<(unsigned)ceil_div(P, 256), 256, 0, s>>>(g->d.t, g->d.ts, g->d.perm, p->dL, P, a, p->nw,
                                                              p->decay, p->coef);
      g_launches++;
      k_fused_factors<<<(unsigned)ceil_div(P, 256), 256, 0, s>>>(g->d.ts, g->d.perm, p->nw, P, (double)(P / 2),
                                                                p->c5, p->c4);
      g_launches++;
      k_real_tables<<<(unsigned)ceil_div(P, 256), 256, 0, s>>>(p->decay, p->coef, P, Window::make(m).b, p->rdecay,
                                                              p->rcoef, p->rdeconv, p->rdd, p->rcd);
      g_launches++;
      if (tile_major) {
        k_tile_major_tables<<<(unsigned)ceil_div(P, 256), 256, 0, s>>>(P, hR, hC, p->rdd, p->rcd, p->rdeconv, p->rdecay,
                                                                      p->rcoef, p->ks, p->tdd, p->tcd, p->tdeconv,
                                                                      p->tdecay, p->tcoef, p->tks);
        g_launches++;
      }
      cudaError_t le = cudaGetLastError();
      if (le != cudaSuccess) status = cuda_fail(le, "plan tables");
    }
    // node-set caches of the solve grid n = 2P (per-tile node ranges of the spreading kernels,
    // overflow flags of the persistent gather): launched behind the tables so the build pays
    // one stream synchronize (check_guards), published after it
    GridCachePending* pend = nullptr;
    if (!status && m == kFastM) {
      int tcs[3] = {64, getenv("NFFT45_STILE") && atoi(getenv("NFFT45_STILE")) == 256 ? 256 : 128, 32};  // 32: warp tiles
      status = grid_caches_begin(g->d, 2 * P, m, tcs, 2 * P <= (int64_t(1) << 17) ? 3 : 2, s, &pend);
    }
    if (!status) status = check_guards(guard.d(), 1, 1, s);
    else cudaStreamSynchronize(s);
    grid_caches_end(g->d, pend, status == NFFT45_OK, s);
  }
  const auto T2 = now();
  if (timing)
    fprintf(stderr, "plan P=%lld: alloc %.3f ms, tables + caches + guards %.3f ms\n", (long long)P, ms(T0, T1),
            ms(T1, T2));
  if (status) {
    cudaStreamSynchronize(s);
    cudaFreeAsync(p->tables, s);
    cudaStreamSynchronize(s);
    delete p->gc;
    delete p;
    return status;
  }
  *out = p;
  return NFFT45_OK;
}

void nfft45_plan_destroy(nfft45_plan* p) {
  if (!p) return;
  DeviceGuard dg(p->g->d.device);
  nfft45::host_pipes_forget(p);
  // solves on any stream may still read the tables (cudaFree used to imply this
  // device-wide wait); the memory then returns to the stream-ordered pool
  cudaDeviceSynchronize();
  if (p->gc) {
    for (auto& kv : p->gc->execs) cudaGraphExecDestroy(kv.second);
    delete p->gc;
  }
  cudaFreeAsync(p->tables, 0);
  delete p;
}

int nfft45_plan_table(const nfft45_plan* p, int which, double* dst, void* st) {
  if (!p || which < 0 || which > 6) return fail(NFFT45_ERR_INVALID_ARGUMENT, "invalid plan table");
  DeviceGuard dg(p->g->d.device);
  if (dg.status) return dg.status;
  const double2* src = p->tables + (int64_t)which * p->P;
  NFFT_CUDA(cudaMemcpyAsync(dst, src, sizeof(double2) * p->P, cudaMemcpyDeviceToDevice, S(st)));
  return NFFT45_OK;
}

int nfft45_type5(const nfft45_plan* p, const double* s, int64_t batch, double* out, void* st) {
  if (!p) return fail(NFFT45_ERR_INVALID_ARGUMENT, "invalid plan");
  if (batch > kMaxRows)  // independent rows: slices keep every launch's gridDim.y in range
    return by_rows(batch, [&](int64_t b0, int64_t nb) {
      return nfft45_type5(p, s + 2 * b0 * p->P, nb, out + 2 * b0 * p->P, st);
    });
  DeviceGuard dg(p->g->d.device);
  if (dg.status) return dg.status;
  if (tiny_eligible(p->P, p->m, 0, batch))
    return tiny_solve(p->g->d, p->P, p->c5, p->c4, p->decay, p->ks, p->coef, 5, C2(s), batch, 0, D2(out), S(st));
  return run_graphed(p, 5, batch, -1, s, out, S(st),
                     [&](cudaStream_t ss) { return type5_core(p, C2(s), batch, D2(out), ss); });
}

int nfft45_type4(const nfft45_plan* p, const double* A, int64_t batch, double* out, void* st) {
  if (!p) return fail(NFFT45_ERR_INVALID_ARGUMENT, "invalid plan");
  if (batch > kMaxRows)  // independent rows: slices keep every launch's gridDim.y in range
    return by_rows(batch, [&](int64_t b0, int64_t nb) {
      return nfft45_type4(p, A + 2 * b0 * p->P, nb, out + 2 * b0 * p->P, st);
    });
  DeviceGuard dg(p->g->d.device);
  if (dg.status) return dg.status;
  if (tiny_eligible(p->P, p->m, 0, batch))
    return tiny_solve(p->g->d, p->P, p->c5, p->c4, p->decay, p->ks, p->coef, 4, C2(A), batch, 0, D2(out), S(st));
  return run_graphed(p, 4, batch, -1, A, out, S(st),
                     [&](cudaStream_t ss) { return type4_core(p, C2(A), batch, D2(out), ss); });
}

}  // extern "C"

namespace nfft45 {
// The refinement re-reads its operand after writing the first solution x into
// `out` (residual = forward(x) - data), so an operand that overlaps `out` is
// first copied to stream-ordered scratch (the one-CTA small solves consume each
// row before writing it and need no copy).  Returns the operand to use.
static int unalias(const double* in, const double* out, int64_t n_doubles, cudaStream_t st, Scratch& copy,
                   const double** use) {
  *use = in;
  const uintptr_t a0 = (uintptr_t)in, a1 = a0 + sizeof(double) * n_doubles;
  const uintptr_t b0 = (uintptr_t)out, b1 = b0 + sizeof(double) * n_doubles;
  if (n_doubles <= 0 || a1 <= b0 || b1 <= a0) return NFFT45_OK;
  NFFT_CHECK(copy.alloc(sizeof(double) * n_doubles));
  NFFT_CUDA(cudaMemcpyAsync(copy.d(), in, sizeof(double) * n_doubles, cudaMemcpyDeviceToDevice, st));
  *use = copy.d();
  return NFFT45_OK;
}
}  // namespace nfft45

extern "C" {

int nfft45_refine_type5(const nfft45_plan* p, const double* s, int64_t batch, int passes, double* out, void* st) {
  if (!p || passes < 0) return fail(NFFT45_ERR_INVALID_ARGUMENT, "invalid refine arguments");
  if (batch > kMaxRows)  // independent rows: slices keep every launch's gridDim.y in range
    return by_rows(batch, [&](int64_t b0, int64_t nb) {
      return nfft45_refine_type5(p, s + 2 * b0 * p->P, nb, passes, out + 2 * b0 * p->P, st);
    });
  DeviceGuard dg(p->g->d.device);
  if (dg.status) return dg.status;
  if (tiny_eligible(p->P, p->m, passes, batch))
    return tiny_solve(p->g->d, p->P, p->c5, p->c4, p->decay, p->ks, p->coef, 5, C2(s), batch, passes, D2(out),
                      S(st));
  if (passes > 0) {
    Scratch copy(S(st));
    const double* use = s;
    NFFT_CHECK(unalias(s, out, 2 * batch * p->P, S(st), copy, &use));
    if (use != s) return refine_core(p, C2(use), batch, passes, D2(out), true, S(st));
  }
  return run_graphed(p, 15, batch, passes, s, out, S(st),
                     [&](cudaStream_t ss) { return refine_core(p, C2(s), batch, passes, D2(out), true, ss); });
}

int nfft45_refine_type4(const nfft45_plan* p, const double* A, int64_t batch, int passes, double* out, void* st) {
  if (!p || passes < 0) return fail(NFFT45_ERR_INVALID_ARGUMENT, "invalid refine arguments");
  if (batch > kMaxRows)  // independent rows: slices keep every launch's gridDim.y in range
    return by_rows(batch, [&](int64_t b0, int64_t nb) {
      return nfft45_refine_type4(p, A + 2 * b0 * p->P, nb, passes, out + 2 * b0 * p->P, st);
    });
  DeviceGuard dg(p->g->d.device);
  if (dg.status) return dg.status;
  if (tiny_eligible(p->P, p->m, passes, batch))
    return tiny_solve(p->g->d, p->P, p->c5, p->c4, p->decay, p->ks, p->coef, 4, C2(A), batch, passes, D2(out),
                      S(st));
  if (passes > 0) {
    Scratch copy(S(st));
    const double* use = A;
    NFFT_CHECK(unalias(A, out, 2 * batch * p->P, S(st), copy, &use));
    if (use != A) return refine_core(p, C2(use), batch, passes, D2(out), false, S(st));
  }
  return run_graphed(p, 14, batch, passes, A, out, S(st),
                     [&](cudaStream_t ss) { return refine_core(p, C2(A), batch, passes, D2(out), false, ss); });
}

}  // extern "C"

// ------------------------------------------------- host-resident solves
//
// Pipelined host -> device -> host solves (the reference API on host arrays,
// inverse.py:101-202): one pipeline per (device, caller stream) with
// persistent H2D / solve / D2H streams and two staging slots, so consecutive
// calls keep both copy directions busy across call boundaries.  Ordering:
//   * downloads of a call wait for the caller's stream at entry (the
//     destination may still be in use there);
//   * the caller's stream waits for the call's last download (results are
//     valid once it is synchronized);
//   * uploads wait only for their staging slot and for this library's own
//     in-flight non-blocking destinations that overlap the input (an output
//     fed straight back as the next input);
//   * a plan's first solve in a pipeline waits for the caller's stream.
// Stable staging pointers also keep the CUDA-graph cache of small solves hot.
namespace nfft45 {
namespace {
struct HostPipe {
  int dev = 0;
  cudaStream_t h2d = nullptr, comp = nullptr, d2h = nullptr;
  cudaEvent_t loaded[2] = {}, done[2] = {}, drained[2] = {};
  double2* bin[2] = {};
  double2* bout[2] = {};
  int64_t cap = 0;  // elements per staging slot
  int64_t turn = 0;  // staging slot of the next call's first chunk
  // pageable operands (numpy arrays): pinned host staging slots filled / drained
  // by the copy pool, and a device flag for the non-finite input check
  double2* hin[2] = {};
  double2* hout[2] = {};
  int64_t hcap = 0;
  int* d_flag = nullptr;
  std::set<const nfft45_plan*> plans;
  std::mutex mu;
};
struct PendingDest {
  uintptr_t lo, hi;
  cudaEvent_t ev;
};
std::mutex g_pipes_mu;  // lock order: g_pipes_mu -> HostPipe::mu -> g_pending_mu
std::map<std::pair<int, cudaStream_t>, HostPipe*> g_pipes;
std::mutex g_pending_mu;
std::vector<PendingDest> g_pending;

int pipe_get(int dev, cudaStream_t user, HostPipe** out) {
  std::lock_guard<std::mutex> lk(g_pipes_mu);
  auto& hp = g_pipes[{dev, user}];
  if (!hp) {
    auto* p = new HostPipe();
    p->dev = dev;
    cudaError_t e = cudaSuccess;
    for (cudaStream_t* s : {&p->h2d, &p->comp, &p->d2h})
      if (e == cudaSuccess) e = cudaStreamCreateWithFlags(s, cudaStreamNonBlocking);
    for (int k = 0; k < 2 && e == cudaSuccess; k++)
      for (cudaEvent_t* ev : {&p->loaded[k], &p->done[k], &p->drained[k]})
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(ev, cudaEventDisableTiming);
    if (e != cudaSuccess) {
      delete p;
      g_pipes.erase({dev, user});
      return cuda_fail(e, "host pipeline streams");
    }
    hp = p;
  }
  *out = hp;
  return NFFT45_OK;
}

int pipe_reserve(HostPipe* hp, int64_t elems) {
  if (hp->cap >= elems) return NFFT45_OK;
  // the old slots may still be in use by queued copies / solves
  for (cudaStream_t s : {hp->h2d, hp->comp, hp->d2h}) NFFT_CUDA(cudaStreamSynchronize(s));
  for (int k = 0; k < 2; k++) {
    cudaFree(hp->bin[k]);
    cudaFree(hp->bout[k]);
    hp->bin[k] = hp->bout[k] = nullptr;
  }
  hp->cap = 0;
  for (int k = 0; k < 2; k++) {
    NFFT_CUDA(cudaMalloc(&hp->bin[k], sizeof(double2) * elems));
    NFFT_CUDA(cudaMalloc(&hp->bout[k], sizeof(double2) * elems));
  }
  hp->cap = elems;
  return NFFT45_OK;
}

int pipe_reserve_host(HostPipe* hp, int64_t elems) {
  if (!hp->d_flag) NFFT_CUDA(cudaMalloc(&hp->d_flag, sizeof(int)));
  if (hp->hcap >= elems) return NFFT45_OK;
  for (cudaStream_t s : {hp->h2d, hp->comp, hp->d2h}) NFFT_CUDA(cudaStreamSynchronize(s));
  for (int k = 0; k < 2; k++) {
    cudaFreeHost(hp->hin[k]);
    cudaFreeHost(hp->hout[k]);
    hp->hin[k] = hp->hout[k] = nullptr;
  }
  hp->hcap = 0;
  for (int k = 0; k < 2; k++) {
    NFFT_CUDA(cudaHostAlloc(&hp->hin[k], sizeof(double2) * elems, cudaHostAllocDefault));
    NFFT_CUDA(cudaHostAlloc(&hp->hout[k], sizeof(double2) * elems, cudaHostAllocDefault));
  }
  hp->hcap = elems;
  return NFFT45_OK;
}

// Host memcpy across a small pool of threads (pageable <-> pinned staging):
// one job at a time, split in >= 1 MiB parts; the caller works too.
class CopyPool {
 public:
  static CopyPool& get() {
    static CopyPool pool;
    return pool;
  }
  void copy(void* dst, const void* src, size_t bytes) {
    const size_t part = std::max<size_t>(size_t(1) << 20, (bytes + nth_) / (nth_ + 1));
    const int nparts = (int)((bytes + part - 1) / part);
    if (nparts <= 1 || th_.empty()) {
      std::memcpy(dst, src, bytes);
      return;
    }
    std::lock_guard<std::mutex> job(job_mu_);
    {
      std::lock_guard<std::mutex> lk(mu_);
      d_ = static_cast<char*>(dst);
      s_ = static_cast<const char*>(src);
      n_ = bytes;
      part_ = part;
      nparts_ = nparts;
      next_.store(0);
      finished_.store(0);
      gen_++;
    }
    cv_.notify_all();
    work();
    std::unique_lock<std::mutex> lk(mu_);
    done_cv_.wait(lk, [&] { return finished_.load() == nparts_; });
  }

 private:
  CopyPool() {
    const unsigned hw = std::max(2u, std::thread::hardware_concurrency());
    nth_ = (int)std::min(7u, hw / 2);
    if (const char* e = getenv("NFFT45_COPY_THREADS")) nth_ = std::max(0, atoi(e) - 1);
    for (int i = 0; i < nth_; i++) th_.emplace_back([this] { loop(); });
  }
  ~CopyPool() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      stop_ = true;
    }
    cv_.notify_all();
    for (auto& t : th_) t.join();
  }
  void work() {
    for (int i; (i = next_.fetch_add(1)) < nparts_;) {
      const size_t off = (size_t)i * part_;
      std::memcpy(d_ + off, s_ + off, std::min(part_, n_ - off));
      if (finished_.fetch_add(1) + 1 == nparts_) {
        std::lock_guard<std::mutex> lk(mu_);
        done_cv_.notify_all();
      }
    }
  }
  void loop() {
    uint64_t seen = 0;
    for (;;) {
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return stop_ || gen_ != seen; });
        if (stop_) return;
        seen = gen_;
      }
      work();
    }
  }
  int nth_ = 0;
  std::vector<std::thread> th_;
  std::mutex job_mu_, mu_;
  std::condition_variable cv_, done_cv_;
  char* d_ = nullptr;
  const char* s_ = nullptr;
  size_t n_ = 0, part_ = 0;
  int nparts_ = 0;
  std::atomic<int> next_{0}, finished_{0};
  uint64_t gen_ = 0;
  bool stop_ = false;
};

__global__ void k_nonfinite(const double* __restrict__ x, int64_t n, int* __restrict__ flag) {
  int bad = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    bad |= !isfinite(x[i]);
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(flag, 1);
}

bool is_pageable(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return true;
  }
  return a.type == cudaMemoryTypeUnregistered;
}
}  // namespace

void host_pipes_forget(const nfft45_plan* p) {
  std::lock_guard<std::mutex> lk(g_pipes_mu);
  for (auto& kv : g_pipes) {
    std::lock_guard<std::mutex> lk2(kv.second->mu);
    kv.second->plans.erase(p);
  }
}
}  // namespace nfft45

namespace nfft45 {
// Pageable operands: chunk i's input is copied (thread pool) into a pinned
// staging slot while the device works on chunk i-1, uploaded, solved and
// downloaded into the pinned output slot, then copied out to the caller's
// array while chunk i+1 is in flight.  Always blocking (the results are on
// the host when the call returns).
static int solve_host_pageable(const nfft45_plan* p, HostPipe* hp, int kind, int passes, const double2* src,
                               int64_t batch, double2* dst, int64_t chunk, bool check_finite) {
  const int64_t P = p->P;
  NFFT_CHECK(pipe_reserve_host(hp, chunk * P));
  if (check_finite) NFFT_CUDA(cudaMemsetAsync(hp->d_flag, 0, sizeof(int), hp->comp));
  CopyPool& pool = CopyPool::get();
  int status = NFFT45_OK;
  int64_t prev_lo = -1, prev_m = 0;
  int prev_k = 0;
  auto drain = [&]() -> int {  // copy the previous chunk's results out to the caller
    if (prev_lo < 0) return NFFT45_OK;
    NFFT_CUDA(cudaEventSynchronize(hp->drained[prev_k]));
    pool.copy(dst + prev_lo * P, hp->hout[prev_k], sizeof(double2) * prev_m * P);
    prev_lo = -1;
    return NFFT45_OK;
  };
  for (int64_t lo = 0, i = 0; lo < batch; lo += chunk, i++) {
    const int k = (int)(i & 1);
    const int64_t m = std::min(chunk, batch - lo);
    const size_t bytes = sizeof(double2) * m * P;
    NFFT_CUDA(cudaEventSynchronize(hp->loaded[k]));  // pinned slot k uploaded (chunk i-2)
    pool.copy(hp->hin[k], src + lo * P, bytes);
    NFFT_CUDA(cudaStreamWaitEvent(hp->h2d, hp->done[k], 0));  // device slot k's input consumed
    NFFT_CUDA(cudaMemcpyAsync(hp->bin[k], hp->hin[k], bytes, cudaMemcpyHostToDevice, hp->h2d));
    NFFT_CUDA(cudaEventRecord(hp->loaded[k], hp->h2d));
    NFFT_CUDA(cudaStreamWaitEvent(hp->comp, hp->loaded[k], 0));
    NFFT_CUDA(cudaStreamWaitEvent(hp->comp, hp->drained[k], 0));
    const double* bi = reinterpret_cast<const double*>(hp->bin[k]);
    double* bo = reinterpret_cast<double*>(hp->bout[k]);
    if (check_finite) {
      const int64_t nd = 2 * m * P;
      LAUNCH(k_nonfinite, (unsigned)std::min<int64_t>(ceil_div(nd, 256), 2 * 148 * 8), 256, 0, hp->comp, bi, nd,
             hp->d_flag);
    }
    if (passes < 0)
      status = kind == 5 ? nfft45_type5(p, bi, m, bo, hp->comp) : nfft45_type4(p, bi, m, bo, hp->comp);
    else
      status = kind == 5 ? nfft45_refine_type5(p, bi, m, passes, bo, hp->comp)
                         : nfft45_refine_type4(p, bi, m, passes, bo, hp->comp);
    NFFT_CUDA(cudaEventRecord(hp->done[k], hp->comp));
    if (status != NFFT45_OK) break;
    NFFT_CUDA(cudaStreamWaitEvent(hp->d2h, hp->done[k], 0));
    NFFT_CUDA(cudaMemcpyAsync(hp->hout[k], hp->bout[k], bytes, cudaMemcpyDeviceToHost, hp->d2h));
    NFFT_CUDA(cudaEventRecord(hp->drained[k], hp->d2h));
    NFFT_CHECK(drain());
    prev_lo = lo;
    prev_m = m;
    prev_k = k;
  }
  if (status != NFFT45_OK) {
    cudaStreamSynchronize(hp->comp);
    return status;
  }
  NFFT_CHECK(drain());
  if (check_finite) {
    int flag = 0;
    NFFT_CUDA(cudaMemcpyAsync(&flag, hp->d_flag, sizeof(int), cudaMemcpyDeviceToHost, hp->comp));
    NFFT_CUDA(cudaStreamSynchronize(hp->comp));
    if (flag) return fail(NFFT45_ERR_INVALID_ARGUMENT, "operand contains NaN or Inf entries");
  }
  return NFFT45_OK;
}
}  // namespace nfft45

extern "C" int nfft45_solve_host(const nfft45_plan* p, int kind, int passes, const double* in_host,
                                 int64_t batch, double* out_host, int64_t chunk, int blocking, void* stream) {
  return nfft45_solve_host_ex(p, kind, passes, in_host, batch, out_host, chunk, blocking, 0, stream);
}

extern "C" int nfft45_solve_host_ex(const nfft45_plan* p, int kind, int passes, const double* in_host,
                                    int64_t batch, double* out_host, int64_t chunk, int blocking, int flags,
                                    void* stream) {
  using namespace nfft45;
  if (!p || (kind != 4 && kind != 5) || batch < 1 || !in_host || !out_host || passes < -1)
    return fail(NFFT45_ERR_INVALID_ARGUMENT, "invalid host solve arguments");
  DeviceGuard dg(p->g->d.device);
  if (dg.status) return dg.status;
  const int64_t P = p->P;
  chunk = std::max<int64_t>(1, std::min(chunk, batch));
  cudaStream_t user = S(stream);
  HostPipe* hp = nullptr;
  NFFT_CHECK(pipe_get(p->g->d.device, user, &hp));
  std::lock_guard<std::mutex> lk(hp->mu);
  NFFT_CHECK(pipe_reserve(hp, chunk * P));
  const bool pageable = !(flags & NFFT45_HOST_NO_STAGING) && (is_pageable(in_host) || is_pageable(out_host));
  cudaEvent_t entry = nullptr, fin = nullptr;
  NFFT_CUDA(cudaEventCreateWithFlags(&entry, cudaEventDisableTiming));
  NFFT_CUDA(cudaEventRecord(entry, user));
  if (hp->plans.insert(p).second) NFFT_CUDA(cudaStreamWaitEvent(hp->comp, entry, 0));
  NFFT_CUDA(cudaStreamWaitEvent(hp->d2h, entry, 0));
  const uintptr_t in_lo = (uintptr_t)in_host, in_hi = in_lo + sizeof(double2) * batch * P;
  {
    std::lock_guard<std::mutex> lk2(g_pending_mu);
    std::vector<PendingDest> live;
    for (auto& d : g_pending) {
      if (cudaEventQuery(d.ev) == cudaSuccess) {
        cudaEventDestroy(d.ev);
        continue;
      }
      if (d.lo < in_hi && in_lo < d.hi) NFFT_CUDA(cudaStreamWaitEvent(hp->h2d, d.ev, 0));
      live.push_back(d);
    }
    g_pending.swap(live);
  }
  const double2* src = reinterpret_cast<const double2*>(in_host);
  double2* dst = reinterpret_cast<double2*>(out_host);
  int status = NFFT45_OK;
  if (pageable) {
    struct NoGraph {
      bool prev;
      explicit NoGraph(bool on) : prev(tl_host_pipe_no_graph) { tl_host_pipe_no_graph = on; }
      ~NoGraph() { tl_host_pipe_no_graph = prev; }
    } ng(chunk * P >= (int64_t(1) << 16));
    status = solve_host_pageable(p, hp, kind, passes, src, batch, dst, chunk, (flags & NFFT45_HOST_CHECK_FINITE) != 0);
    cudaEvent_t done_ev = nullptr;
    NFFT_CUDA(cudaEventCreateWithFlags(&done_ev, cudaEventDisableTiming));
    NFFT_CUDA(cudaEventRecord(done_ev, hp->d2h));
    NFFT_CUDA(cudaStreamWaitEvent(user, done_ev, 0));
    cudaEventDestroy(done_ev);
    cudaEventDestroy(entry);
    return status;
  }
  // A call's first chunk takes the slot the previous call's last solve is not
  // using, so its upload overlaps that solve.  Chunks of at least 2^16 points
  // run without the CUDA-graph cache here: next to the pipeline's copies the
  // graph replays cost more than the launches they save (C2 e2e 1.6e9 with
  // graphs vs 1.94e9 without; C3 2.36e9 vs 2.41e9), while C1-sized solves stay
  // launch-bound and keep their graphs.
  static const bool noalt = getenv("NFFT45_PIPE_NOALT") != nullptr;
  const int64_t i0 = noalt ? 0 : hp->turn;
  struct NoGraphScope {
    bool prev;
    explicit NoGraphScope(bool on) : prev(tl_host_pipe_no_graph) { tl_host_pipe_no_graph = on; }
    ~NoGraphScope() { tl_host_pipe_no_graph = prev; }
  } ngs(chunk * P >= (int64_t(1) << 16));
  for (int64_t lo = 0, i = i0; lo < batch && status == NFFT45_OK; lo += chunk, i++) {
    const int k = (int)(i & 1);
    hp->turn = i + 1;
    const int64_t m = std::min(chunk, batch - lo);
    const size_t bytes = sizeof(double2) * m * P;
    NFFT_CUDA(cudaStreamWaitEvent(hp->h2d, hp->done[k], 0));  // slot k's input consumed
    NFFT_CUDA(cudaMemcpyAsync(hp->bin[k], src + lo * P, bytes, cudaMemcpyHostToDevice, hp->h2d));
    NFFT_CUDA(cudaEventRecord(hp->loaded[k], hp->h2d));
    NFFT_CUDA(cudaStreamWaitEvent(hp->comp, hp->loaded[k], 0));
    NFFT_CUDA(cudaStreamWaitEvent(hp->comp, hp->drained[k], 0));  // slot k's output downloaded
    const double* bi = reinterpret_cast<const double*>(hp->bin[k]);
    double* bo = reinterpret_cast<double*>(hp->bout[k]);
    if (passes < 0)
      status = kind == 5 ? nfft45_type5(p, bi, m, bo, hp->comp) : nfft45_type4(p, bi, m, bo, hp->comp);
    else
      status = kind == 5 ? nfft45_refine_type5(p, bi, m, passes, bo, hp->comp)
                         : nfft45_refine_type4(p, bi, m, passes, bo, hp->comp);
    NFFT_CUDA(cudaEventRecord(hp->done[k], hp->comp));
    if (status != NFFT45_OK) break;
    NFFT_CUDA(cudaStreamWaitEvent(hp->d2h, hp->done[k], 0));
    NFFT_CUDA(cudaMemcpyAsync(dst + lo * P, hp->bout[k], bytes, cudaMemcpyDeviceToHost, hp->d2h));
    NFFT_CUDA(cudaEventRecord(hp->drained[k], hp->d2h));
  }
  NFFT_CUDA(cudaEventCreateWithFlags(&fin, cudaEventDisableTiming));
  NFFT_CUDA(cudaEventRecord(fin, hp->d2h));
  NFFT_CUDA(cudaStreamWaitEvent(user, fin, 0));
  cudaEventDestroy(entry);
  if (blocking || status != NFFT45_OK) {
    cudaError_t e = cudaEventSynchronize(fin);
    cudaEventDestroy(fin);
    if (status == NFFT45_OK && e != cudaSuccess) return cuda_fail(e, "host solve");
    return status;
  }
  std::lock_guard<std::mutex> lk2(g_pending_mu);
  g_pending.push_back({(uintptr_t)out_host, (uintptr_t)out_host + sizeof(double2) * batch * P, fin});
  return NFFT45_OK;
}
