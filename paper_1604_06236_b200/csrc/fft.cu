// fft.cu — kernels and host driver of the batched fp64 FFT engine.
#include <map>
#include <mutex>
#include <tuple>

#include "fft_fast.cuh"

namespace nfft45 {

bool fft_smooth(int64_t N) {
  if (N < 1) return false;
  for (int p : {2, 3, 5})
    while (N % p == 0) N /= p;
  return N == 1;
}

FftSeq fft_seq(int N) {
  FftSeq s;
  s.N = N;
  s.np = 0;
  int n = N;
  while (n % 8 == 0) { s.R[s.np++] = 8; n /= 8; }
  if (n % 4 == 0) { s.R[s.np++] = 4; n /= 4; }
  if (n % 2 == 0) { s.R[s.np++] = 2; n /= 2; }
  while (n % 3 == 0) { s.R[s.np++] = 3; n /= 3; }
  while (n % 5 == 0) { s.R[s.np++] = 5; n /= 5; }
  return s;
}

static bool pass_size(int64_t N);

// Runtime-radix tiles need blockDim >= Nt*C/12 with blockDim <= 256.
constexpr int kRtTileMax = 3072;

bool fft_split(int64_t N, int* N1, int* N2) {
  // Prefer a balanced split into two compile-time tile sizes; otherwise two
  // smooth runtime tiles <= kRtTileMax.
  for (int pass = 0; pass < 2; pass++) {
    int best1 = 0, best2 = 0;
    double bestScore = 1e300;
    for (int64_t a = 2; a <= kTileMax; a++) {
      if (N % a) continue;
      int64_t b = N / a;
      bool ok = pass == 0 ? (pass_size(a) && pass_size(b))
                          : (a <= kRtTileMax && b <= kRtTileMax && fft_smooth(a) && fft_smooth(b));
      if (!ok) continue;
      double score = fabs(log((double)a) - log((double)b));
      if (score < bestScore) { bestScore = score; best1 = (int)a; best2 = (int)b; }
    }
    if (best1) {
      *N1 = best1;
      *N2 = best2;
      return true;
    }
  }
  return false;
}

// -------------------------------------------------------------- twiddles

// e^{-2 pi i k / N} with the angle reduced exactly in integers first.
__global__ void k_twiddle_fill(double2* out, int64_t count, int64_t N, int64_t step) {
  int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= count) return;
  int64_t e = (k * step) % N;          // < N
  if (2 * e > N) e -= N;                // |e| <= N/2
  double s, c;
  sincospi(-2.0 * (double)e / (double)N, &s, &c);
  out[k] = make_double2(c, s);
}

static std::mutex g_tw_mu;
static std::map<std::pair<int, int64_t>, FftTables*> g_tw;

#define NFFT_CUDA_P(call)                                  \
  do {                                                     \
    cudaError_t _e = (call);                               \
    if (_e != cudaSuccess) {                               \
      *status = cuda_fail(_e, #call);                      \
      return nullptr;                                      \
    }                                                      \
  } while (0)

const FftTables* fft_tables(int64_t N, cudaStream_t st, int* status) {
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(g_tw_mu);
  auto key = std::make_pair(dev, N);
  auto it = g_tw.find(key);
  if (it != g_tw.end()) { *status = NFFT45_OK; return it->second; }
  FftTables* t = new FftTables();
  t->N = N;
  t->tw = t->lo = t->hi = nullptr;
  t->s = 0;
  auto fill = [&](double2** dst, int64_t count, int64_t step) -> int {
    NFFT_CUDA(cudaMalloc(dst, sizeof(double2) * (count > 0 ? count : 1)));
    LAUNCH(k_twiddle_fill, (unsigned)ceil_div(count, 256), 256, 0, st, *dst, count, N, step);
    return NFFT45_OK;
  };
  int s = NFFT45_OK;
  if (N <= kTileMax && is_pow2(N)) {
    // [4][N]: section q = W_N^{k 2^q} (the same sincospi values as tw[(k << q) mod N])
    NFFT_CUDA_P(cudaMalloc(&t->tw, sizeof(double2) * 4 * N));
    for (int q = 0; q < 4 && s == NFFT45_OK; q++) {
      k_twiddle_fill<<<(unsigned)ceil_div(N, 256), 256, 0, st>>>(t->tw + q * N, N, N, int64_t(1) << q);
      g_launches.fetch_add(1, std::memory_order_relaxed);
      cudaError_t le = cudaGetLastError();
      if (le != cudaSuccess) s = cuda_fail(le, "k_twiddle_fill");
    }
  } else if (N <= 65536 || !fft_smooth(N)) s = fill(&t->tw, N, 1);
  if (s == NFFT45_OK && N > 1 && fft_smooth(N)) {
    int bits = 0;
    while ((int64_t(1) << (2 * bits)) < N) bits++;
    t->s = bits;
    int64_t lo = int64_t(1) << bits;
    s = fill(&t->lo, lo, 1);
    if (s == NFFT45_OK) s = fill(&t->hi, ceil_div(N, lo), lo);
  }
  if (s == NFFT45_OK) {
    cudaError_t e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) s = cuda_fail(e, "twiddle table");
  }
  *status = s;
  if (s != NFFT45_OK) return nullptr;
  g_tw[key] = t;
  return t;
}

// ------------------------------------------------------------- kernels

// Tile load / store.  A tile is [Nt][C]; element (i, c) lives at global
// address base + c * sc + i * si.  If sc == 1 the lanes run along c
// (column-contiguous memory), otherwise along i (row-contiguous).

struct TileIO {
  int64_t si, sc;
};

__device__ __forceinline__ void tile_coords(int e, int Nt, int C, bool cfast, int& i, int& c) {
  if (cfast) { c = e % C; i = e / C; }
  else { i = e % Nt; c = e / Nt; }
}

// Single-pass: columns are signals. in/out[b][N]
template <int S>
__global__ void __launch_bounds__(256) k_fft_single(const double2* __restrict__ in, double2* __restrict__ out,
                                                     int64_t batch, FftSeq seq, int C,
                                                     const double2* __restrict__ tw,
                                                     const double2* __restrict__ pre,
                                                     const double2* __restrict__ post) {
  extern __shared__ double2 sm[];
  const int Nt = seq.N;
  const int64_t b0 = (int64_t)blockIdx.x * C;
  const int total = Nt * C;
  for (int e = threadIdx.x; e < total; e += blockDim.x) {
    int i = e % Nt, c = e / Nt;
    int64_t b = b0 + c;
    double2 v = make_double2(0.0, 0.0);
    if (b < batch) {
      v = in[b * Nt + i];
      if (pre) v = cmul(v, __ldg(&pre[i]));
    }
    sm[tpad(i * C + c)] = v;
  }
  __syncthreads();
  tile_fft<S>(sm, seq, C, tw);
  for (int e = threadIdx.x; e < total; e += blockDim.x) {
    int i = e % Nt, c = e / Nt;
    int64_t b = b0 + c;
    if (b < batch) {
      double2 v = sm[tpad(i * C + c)];
      if (post) v = cmul(v, __ldg(&post[i]));
      out[b * Nt + i] = v;
    }
  }
}

// Four-step pass A: column FFTs of length N1 over x[n1*N2 + n2], C columns
// per CTA, then the twiddle W_N^{n2 k1}; stored in place-layout [k1][n2].
template <int S>
__global__ void __launch_bounds__(256) k_fft_passA(const double2* __restrict__ in, double2* __restrict__ out,
                                                    int64_t N, int N2, FftSeq seq, int C,
                                                    const double2* __restrict__ tw,
                                                    const double2* __restrict__ lo,
                                                    const double2* __restrict__ hi, int tws,
                                                    const double2* __restrict__ pre) {
  extern __shared__ double2 sm[];
  const int N1 = seq.N;
  const int c0 = blockIdx.x * C;
  const int64_t base = (int64_t)blockIdx.y * N;
  const int total = N1 * C;
  for (int e = threadIdx.x; e < total; e += blockDim.x) {
    int c = e % C, i = e / C;
    int64_t idx = (int64_t)i * N2 + c0 + c;
    double2 v = in[base + idx];
    if (pre) v = cmul(v, __ldg(&pre[idx]));
    sm[tpad(i * C + c)] = v;
  }
  __syncthreads();
  tile_fft<S>(sm, seq, C, tw);
  const int64_t mask = (int64_t(1) << tws) - 1;
  for (int e = threadIdx.x; e < total; e += blockDim.x) {
    int c = e % C, k1 = e / C;
    int64_t n2 = c0 + c;
    int64_t ex = n2 * k1;  // < N
    double2 w = cmul(__ldg(&hi[ex >> tws]), __ldg(&lo[ex & mask]));
    double2 v = sm[tpad(k1 * C + c)];
    v = S < 0 ? cmul(v, w) : cmulc(v, w);
    out[base + (int64_t)k1 * N2 + n2] = v;
  }
}

// Four-step pass B: row FFTs of length N2 over t[k1*N2 + n2], C rows per CTA;
// X[k1 + N1 k2] stored in natural order.
template <int S>
__global__ void __launch_bounds__(256) k_fft_passB(const double2* __restrict__ in, double2* __restrict__ out,
                                                    int64_t N, int N1, FftSeq seq, int C,
                                                    const double2* __restrict__ tw,
                                                    const double2* __restrict__ post) {
  extern __shared__ double2 sm[];
  const int N2 = seq.N;
  const int r0 = blockIdx.x * C;
  const int64_t base = (int64_t)blockIdx.y * N;
  const int total = N2 * C;
  // row-contiguous load: lanes along n2
  for (int e = threadIdx.x; e < total; e += blockDim.x) {
    int i = e % N2, c = e / N2;
    sm[tpad(i * C + c)] = in[base + (int64_t)(r0 + c) * N2 + i];
  }
  __syncthreads();
  tile_fft<S>(sm, seq, C, tw);
  // column-contiguous store: lanes along k1
  for (int e = threadIdx.x; e < total; e += blockDim.x) {
    int c = e % C, k2 = e / C;
    int64_t idx = (int64_t)(r0 + c) + (int64_t)N1 * k2;
    double2 v = sm[tpad(k2 * C + c)];
    if (post) v = cmul(v, __ldg(&post[idx]));
    out[base + idx] = v;
  }
}

// Direct DFT for non-smooth N: X_k = sum_j x_j W^{jk mod N}.
template <int S>
__global__ void k_dft_direct(const double2* __restrict__ in, double2* __restrict__ out, int64_t N,
                             const double2* __restrict__ tw, const double2* __restrict__ pre,
                             const double2* __restrict__ post) {
  int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t b = blockIdx.y;
  if (k >= N) return;
  const double2* x = in + b * N;
  double2 acc = make_double2(0.0, 0.0);
  int64_t idx = 0;
  for (int64_t j = 0; j < N; j++) {
    double2 v = x[j];
    if (pre) v = cmul(v, __ldg(&pre[j]));
    double2 w = __ldg(&tw[idx]);
    double2 p = S < 0 ? cmul(v, w) : cmulc(v, w);
    acc = cadd(acc, p);
    idx += k;
    if (idx >= N) idx -= N;
  }
  if (post) acc = cmul(acc, __ldg(&post[k]));
  out[b * N + k] = acc;
}

__global__ void k_scale_copy(const double2* __restrict__ in, double2* __restrict__ out, int64_t total,
                             int64_t N, const double2* __restrict__ pre,
                             const double2* __restrict__ post) {
  int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= total) return;
  double2 v = in[e];
  int64_t i = e % N;
  if (pre) v = cmul(v, pre[i]);
  if (post) v = cmul(v, post[i]);
  out[e] = v;
}

// ---------------------------------------------------- compile-time sized kernels

template <int N, int C, int S>
__global__ void __launch_bounds__(fast_threads<N, C>()) kf_single(const double2* __restrict__ in,
                                                                 double2* __restrict__ out, int64_t batch,
                                                                 const double2* __restrict__ tw,
                                                                 const double2* __restrict__ pre,
                                                                 const double2* __restrict__ post) {
  extern __shared__ double2 sm[];
  const int64_t b0 = (int64_t)blockIdx.x * C;
  auto ld = [&](int i, int c) -> double2 {
    const int64_t b = b0 + c;
    if (b >= batch) return make_double2(0.0, 0.0);
    double2 v = in[b * N + i];
    if (pre) v = cmul(v, __ldg(&pre[i]));
    return v;
  };
  auto st = [&](int k, int c, double2 v) {
    const int64_t b = b0 + c;
    if (b < batch) {
      if (post) v = cmul(v, __ldg(&post[k]));
      out[b * N + k] = v;
    }
  };
  fast_tile_fft<N, C, S, false>(sm, ld, st, tw);
}

template <int N1, int C, int S>
__global__ void __launch_bounds__(fast_threads<N1, C>()) kf_passA(const double2* __restrict__ in,
                                                                 double2* __restrict__ out, int64_t N, int N2,
                                                                 const double2* __restrict__ tw,
                                                                 const double2* __restrict__ lo,
                                                                 const double2* __restrict__ hi, int tws,
                                                                 const double2* __restrict__ pre) {
  extern __shared__ double2 sm[];
  const int c0 = blockIdx.x * C;
  const int64_t base = (int64_t)blockIdx.y * N;
  const int64_t mask = (int64_t(1) << tws) - 1;
  auto ld = [&](int i, int c) -> double2 {
    const int64_t idx = (int64_t)i * N2 + c0 + c;
    double2 v = in[base + idx];
    if (pre) v = cmul(v, __ldg(&pre[idx]));
    return v;
  };
  auto st = [&](int k1, int c, double2 v) {
    const int64_t n2 = c0 + c;
    const int64_t ex = n2 * k1;
    const double2 w = cmul(__ldg(&hi[ex >> tws]), __ldg(&lo[ex & mask]));
    out[base + (int64_t)k1 * N2 + n2] = S < 0 ? cmul(v, w) : cmulc(v, w);
  };
  fast_tile_fft<N1, C, S, true>(sm, ld, st, tw);
}

template <int N2, int C, int S>
__global__ void __launch_bounds__(fast_threads<N2, C>()) kf_passB(const double2* __restrict__ in,
                                                                 double2* __restrict__ out, int64_t N, int N1,
                                                                 const double2* __restrict__ tw,
                                                                 const double2* __restrict__ post) {
  extern __shared__ double2 sm[];
  const int r0 = blockIdx.x * C;
  const int64_t base = (int64_t)blockIdx.y * N;
  auto ld = [&](int i, int c) -> double2 { return in[base + (int64_t)(r0 + c) * N2 + i]; };
  auto st = [&](int k2, int c, double2 v) {
    const int64_t idx = (int64_t)(r0 + c) + (int64_t)N1 * k2;
    if (post) v = cmul(v, __ldg(&post[idx]));
    out[base + idx] = v;
  };
  fast_tile_fft<N2, C, S, true>(sm, ld, st, tw);
}

template <int N>
constexpr int single_cols() { return FastTraits<N>::pow2 ? 4096 / N : 6144 / N; }
template <int N>
constexpr int pass_cols() { return single_cols<N>() < 8 ? single_cols<N>() : 8; }

template <typename K>
static int fast_attr(K kernel, size_t bytes) {
  if (bytes > 48 * 1024) NFFT_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
  return NFFT45_OK;
}

template <int N, int S>
static int launch_single(const double2* in, double2* out, int64_t batch, const double2* tw, const double2* pre,
                         const double2* post, cudaStream_t st) {
  constexpr int C = single_cols<N>();
  constexpr size_t smem = fast_smem<N, C>();
  auto fft_single = kf_single<N, C, S>;
  NFFT_CHECK(fast_attr(fft_single, smem));
  constexpr int T = fast_threads<N, C>();
  LAUNCH(fft_single, (unsigned)ceil_div(batch, C), T, smem, st, in, out, batch, tw, pre, post);
  return NFFT45_OK;
}

template <int N1, int S>
static int launch_passA(const double2* in, double2* out, int64_t batch, int64_t N, int N2, const double2* tw,
                        const FftTables* tN, const double2* pre, cudaStream_t st) {
  constexpr int C = pass_cols<N1>();
  constexpr size_t smem = fast_smem<N1, C>();
  auto fft_passA = kf_passA<N1, C, S>;
  NFFT_CHECK(fast_attr(fft_passA, smem));
  dim3 grid((unsigned)(N2 / C), (unsigned)batch);
  constexpr int T = fast_threads<N1, C>();
  LAUNCH(fft_passA, grid, T, smem, st, in, out, N, N2, tw, tN->lo, tN->hi, tN->s, pre);
  return NFFT45_OK;
}

template <int N2, int S>
static int launch_passB(const double2* in, double2* out, int64_t batch, int64_t N, int N1, const double2* tw,
                        const double2* post, cudaStream_t st) {
  constexpr int C = pass_cols<N2>();
  constexpr size_t smem = fast_smem<N2, C>();
  auto fft_passB = kf_passB<N2, C, S>;
  NFFT_CHECK(fast_attr(fft_passB, smem));
  dim3 grid((unsigned)(N1 / C), (unsigned)batch);
  constexpr int T = fast_threads<N2, C>();
  LAUNCH(fft_passB, grid, T, smem, st, in, out, N, N1, tw, post);
  return NFFT45_OK;
}

#define NFFT_FAST_SIZES(X) \
  X(2) X(4) X(8) X(16) X(32) X(64) X(128) X(256) X(512) X(1024) X(2048) X(4096) \
  X(3) X(6) X(12) X(24) X(48) X(96) X(192) X(384) X(768) X(1536) X(3072)
#define NFFT_PASS_SIZES(X) \
  X(64) X(128) X(256) X(512) X(1024) X(2048) X(4096) X(96) X(192) X(384) X(768) X(1536) X(3072)

static bool fast_size(int64_t N) {
#define X(n) if (N == n) return true;
  NFFT_FAST_SIZES(X)
#undef X
  return false;
}
static bool pass_size(int64_t N) {
#define X(n) if (N == n) return true;
  NFFT_PASS_SIZES(X)
#undef X
  return false;
}

template <int S>
static int dispatch_single(int64_t N, const double2* in, double2* out, int64_t batch, const double2* tw,
                           const double2* pre, const double2* post, cudaStream_t st) {
  switch (N) {
#define X(n) case n: return launch_single<n, S>(in, out, batch, tw, pre, post, st);
    NFFT_FAST_SIZES(X)
#undef X
  }
  return NFFT45_ERR_INVALID_ARGUMENT;
}
template <int S>
static int dispatch_passA(int N1, const double2* in, double2* out, int64_t batch, int64_t N, int N2,
                          const double2* tw, const FftTables* tN, const double2* pre, cudaStream_t st) {
  switch (N1) {
#define X(n) case n: return launch_passA<n, S>(in, out, batch, N, N2, tw, tN, pre, st);
    NFFT_PASS_SIZES(X)
#undef X
  }
  return NFFT45_ERR_INVALID_ARGUMENT;
}
template <int S>
static int dispatch_passB(int N2, const double2* in, double2* out, int64_t batch, int64_t N, int N1,
                          const double2* tw, const double2* post, cudaStream_t st) {
  switch (N2) {
#define X(n) case n: return launch_passB<n, S>(in, out, batch, N, N1, tw, post, st);
    NFFT_PASS_SIZES(X)
#undef X
  }
  return NFFT45_ERR_INVALID_ARGUMENT;
}

// ------------------------------------------------------------ host driver

template <typename K>
static int set_smem(K kernel, size_t bytes) {
  static std::mutex mu;
  if (bytes > 48 * 1024) {
    std::lock_guard<std::mutex> lk(mu);
    NFFT_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
  }
  return NFFT45_OK;
}

template <int S>
static int fft_run_s(const double2* in, double2* out, int64_t batch, int64_t N, const double2* pre,
                     const double2* post, cudaStream_t st) {
  int status = NFFT45_OK;
  if (N == 1) {
    if (in == out && !pre && !post) return NFFT45_OK;
    LAUNCH(k_scale_copy, (unsigned)ceil_div(batch, 256), 256, 0, st, in, out, batch, N, pre, post);
    return NFFT45_OK;
  }
  if (!fft_smooth(N)) {
    if (N > 65536) {
      set_error(NFFT45_ERR_INVALID_ARGUMENT, "FFT length " + std::to_string(N) +
                                                 " has a prime factor > 5 and exceeds the direct-DFT limit 65536");
      return NFFT45_ERR_INVALID_ARGUMENT;
    }
    const FftTables* t = fft_tables(N, st, &status);
    if (!t) return status;
    double2* tmp = nullptr;
    const double2* src = in;
    if (in == out) {
      NFFT_CUDA(cudaMallocAsync(&tmp, sizeof(double2) * batch * N, st));
      NFFT_CUDA(cudaMemcpyAsync(tmp, in, sizeof(double2) * batch * N, cudaMemcpyDeviceToDevice, st));
      src = tmp;
    }
    dim3 grid((unsigned)ceil_div(N, 128), (unsigned)batch);
    LAUNCH(k_dft_direct<S>, grid, 128, 0, st, src, out, N, t->tw, pre, post);
    if (tmp) NFFT_CUDA(cudaFreeAsync(tmp, st));
    return NFFT45_OK;
  }
  if (fast_size(N)) {
    const FftTables* t = fft_tables(N, st, &status);
    if (!t) return status;
    return dispatch_single<S>(N, in, out, batch, t->tw, pre, post, st);
  }
  if (N <= kRtTileMax) {
    const FftTables* t = fft_tables(N, st, &status);
    if (!t) return status;
    int C = 1;
    while (C < 512 && N * C * 2 <= kRtTileMax) C *= 2;
    if (C > batch) {
      C = 1;
      while (C < batch) C *= 2;
    }
    FftSeq seq = fft_seq((int)N);
    size_t smem = tile_smem_bytes((int)N, C);
    NFFT_CHECK(set_smem(k_fft_single<S>, smem));
    LAUNCH(k_fft_single<S>, (unsigned)ceil_div(batch, C), tile_threads((int)N, C), smem, st, in, out, batch,
           seq, C, t->tw, pre, post);
    return NFFT45_OK;
  }
  int N1, N2;
  if (!fft_split(N, &N1, &N2)) {
    set_error(NFFT45_ERR_INVALID_ARGUMENT, "FFT length " + std::to_string(N) + " is not supported");
    return NFFT45_ERR_INVALID_ARGUMENT;
  }
  const FftTables* tN = fft_tables(N, st, &status);
  if (!tN) return status;
  const FftTables* t1 = fft_tables(N1, st, &status);
  if (!t1) return status;
  const FftTables* t2 = fft_tables(N2, st, &status);
  if (!t2) return status;
  double2* tmp = nullptr;
  NFFT_CUDA(cudaMallocAsync(&tmp, sizeof(double2) * batch * N, st));
  if (pass_size(N1) && pass_size(N2)) {
    NFFT_CHECK(dispatch_passA<S>(N1, in, tmp, batch, N, N2, t1->tw, tN, pre, st));
    NFFT_CHECK(dispatch_passB<S>(N2, tmp, out, batch, N, N1, t2->tw, post, st));
    NFFT_CUDA(cudaFreeAsync(tmp, st));
    return NFFT45_OK;
  }
  {
    int C = 8;
    while (C > 1 && N1 * C > kRtTileMax) C /= 2;
    while (C > 1 && N2 % C) C /= 2;
    FftSeq seq = fft_seq(N1);
    size_t smem = tile_smem_bytes(N1, C);
    NFFT_CHECK(set_smem(k_fft_passA<S>, smem));
    dim3 grid((unsigned)(N2 / C), (unsigned)batch);
    LAUNCH(k_fft_passA<S>, grid, tile_threads(N1, C), smem, st, in, tmp, N, N2, seq, C, t1->tw, tN->lo,
           tN->hi, tN->s, pre);
  }
  {
    int C = 8;
    while (C > 1 && N2 * C > kRtTileMax) C /= 2;
    while (C > 1 && N1 % C) C /= 2;
    FftSeq seq = fft_seq(N2);
    size_t smem = tile_smem_bytes(N2, C);
    NFFT_CHECK(set_smem(k_fft_passB<S>, smem));
    dim3 grid((unsigned)(N1 / C), (unsigned)batch);
    LAUNCH(k_fft_passB<S>, grid, tile_threads(N2, C), smem, st, tmp, out, N, N1, seq, C, t2->tw, post);
  }
  NFFT_CUDA(cudaFreeAsync(tmp, st));
  return NFFT45_OK;
}

int fft_run(const double2* in, double2* out, int64_t batch, int64_t N, int sign, const double2* pre,
            const double2* post, cudaStream_t st) {
  if (batch <= 0 || N <= 0) return NFFT45_OK;
  return sign < 0 ? fft_run_s<-1>(in, out, batch, N, pre, post, st)
                  : fft_run_s<+1>(in, out, batch, N, pre, post, st);
}

}  // namespace nfft45
