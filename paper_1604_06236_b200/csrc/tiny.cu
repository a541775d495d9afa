// tiny.cu — the whole type-5 / type-4 solve (and its Section V refinement
// pass) of one small signal in ONE CTA, everything in shared memory.
//
// For P <= 256 every stage of the solve (spreading, FFT_2P, band selection,
// IFFT_P, the Lagrange kernel samples, FFT_P, zero padding, IFFT_2P,
// interpolation, residual and correction) is a few microseconds of work but a
// separate launch on the general path, so a plain solve costs ~10 launches
// and a refined one ~25 even when replayed from a CUDA graph.  Here a CTA per
// signal runs the same stage sequence with barriers in between:
//
//   type 5 (inverse.py:101-120):  a_q = s_{perm q} c5_q  -> spread onto n = 2P
//       -> FFT_n -> U_p = Ĥ[(p-K) mod n] deconv_p decay_p -> IFFT_P * ks
//       -> FFT_P * coef
//   type 4 (inverse.py:123-143):  IFFT_P(A decay) * ks -> FFT_P * coef
//       -> pad F[(p-K) mod n] = V_p deconv_p -> IFFT_n -> gather * c4 (caller order)
//   refinement (inverse.py:146-162): r = fwd(x) - data with the forward
//       NFFT of forward.py:26-102 (type 2 for type 5, type 1 of length P for
//       type 4), then x -= solve(r).
//
// Window: Gaussian, m = 14 (29 taps, the factorised weights of gridding.cu);
// every cell sums its nodes in ascending order and every FFT is a fixed
// radix-2 Stockham sequence, so results are deterministic and identical for
// batched and single calls.  Requires P a power of two, 32 <= P <= 256 (so a
// 29-tap window never wraps onto itself on the n = 2P grid).
#include "ops.cuh"

namespace nfft45 {

namespace {
constexpr int kTM = 14;
constexpr int kTTaps = 2 * kTM + 1;
constexpr int kTThreads = 256;

struct TinyArgs {
  const double* ts;     // ascending nodes
  const int* perm;      // ts[q] = t[perm[q]]
  const double2* c5;    // ascending-node factors (type 5 spread)
  const double2* c4;    // (type 4 gather)
  const double2* decay;  // P-tables
  const double2* ks;
  const double2* coef;
  int P;
  double alpha, b;
  GaussTab G;
};

// in-place (ping-pong) radix-2 Stockham FFT of length N in shared memory,
// sign S (-1 forward, +1 unnormalised inverse); returns the buffer holding the
// result (x or y)
// tw[i] = e^{-2 pi i i / n}, i < n/2 (n = 2P >= N): e^{S 2 pi i k / (2 Ns)} = tw[k n / (2 Ns)] (conjugated for S = +1)
__device__ double2* tiny_fft(double2* x, double2* y, int N, int S, const double2* tw, int n) {
  for (int Ns = 1; Ns < N; Ns <<= 1) {
    const int step = n / (2 * Ns);
    for (int j = threadIdx.x; j < N / 2; j += blockDim.x) {
      const int k = j & (Ns - 1);
      double2 w = tw[k * step];
      if (S > 0) w.y = -w.y;
      const double2 a = x[j];
      const double2 bb = cmul(x[j + N / 2], w);
      const int d = (j - k) * 2 + k;
      y[d] = cadd(a, bb);
      y[d + Ns] = csub(a, bb);
    }
    __syncthreads();
    double2* t = x;
    x = y;
    y = t;
  }
  return x;
}

struct TinySmem {
  double* W;   // [P][29] weights, ascending nodes
  int* i0;     // [P] rounded centres
  double* tq;  // [P] ascending nodes
  double2* H;  // [n] grid
  double2* T;  // [n] FFT ping-pong
  double2* X;  // [P] current solution (type 5: p order; type 4: ascending-node order)
  double2* R;  // [P] residual / solve input
  double2* Y;  // [P] scratch
  double2* tw;  // [n/2] e^{-2 pi i k / n}
};

// H[j] = sum over ascending nodes q with |j - i0_q| <= 14 (mod n) of w_q,k amp_q
// first q with i0[q] >= x (i0 ascending, values in [0, n])
__device__ __forceinline__ int tiny_lower(const int* i0, int P, int x) {
  int lo = 0, hi = P;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (i0[mid] >= x) hi = mid;
    else lo = mid + 1;
  }
  return lo;
}

// Centres ascend with q (i0 in [0, n]), so the nodes reaching cell j form one
// contiguous range per periodic image (centre i0 + n, i0, i0 - n); the images
// are visited in ascending q (img = +1 reaches j from the smallest centres),
// i.e. every cell sums its nodes in ascending order.
__device__ void tiny_spread(const TinySmem& s, const double2* amp, int P) {
  const int n = 2 * P;
  for (int j = threadIdx.x; j < n; j += blockDim.x) {
    double2 acc = make_double2(0.0, 0.0);
#pragma unroll
    for (int img = 1; img >= -1; img--) {  // centre i0 + img n reaches j <=> i0 in [j - 14 - img n, j + 14 - img n]
      const int lo = tiny_lower(s.i0, P, j - kTM - img * n);
      const int hi = tiny_lower(s.i0, P, j + kTM + 1 - img * n);
      for (int q = lo; q < hi; q++) caxpy(acc, s.W[q * kTTaps + (j - s.i0[q] - img * n) + kTM], amp[q]);
    }
    s.H[j] = acc;
  }
  __syncthreads();
}

// out_q = sum_k w_q,k G[(i0_q + k - 14) mod n], ascending k
__device__ __forceinline__ double2 tiny_gather1(const TinySmem& s, const double2* G, int q, int n) {
  double2 acc = make_double2(0.0, 0.0);
  int c = s.i0[q] - kTM;
  c %= n;
  if (c < 0) c += n;
#pragma unroll
  for (int k = 0; k < kTTaps; k++) {
    caxpy(acc, s.W[q * kTTaps + k], G[c]);
    c = c + 1 == n ? 0 : c + 1;
  }
  return acc;
}

// plain type-5 solve of in[P] (amplitudes already in ascending-node order,
// multiplied by c5) -> out[P] (p order)
__device__ void tiny_t5(const TinySmem& s, const TinyArgs& a, const double2* amp, double2* out) {
  const int P = a.P, n = 2 * P, K = P / 2;
  tiny_spread(s, amp, P);
  double2* F = tiny_fft(s.H, s.T, n, -1, s.tw, n);
  for (int p = threadIdx.x; p < P; p += blockDim.x) {
    int bin = (p - K) % n;
    if (bin < 0) bin += n;
    s.Y[p] = cmul(a.decay[p], cscale(F[bin], deconv_weight(p, K, n, a.b)));
  }
  __syncthreads();
  double2* V = tiny_fft(s.Y, s.H, P, +1, s.tw, n);  // s.H is free scratch of length >= P
  for (int p = threadIdx.x; p < P; p += blockDim.x) V[p] = cmul(V[p], a.ks[p]);
  __syncthreads();
  double2* Wv = tiny_fft(V, V == s.Y ? s.H : s.Y, P, -1, s.tw, n);
  for (int p = threadIdx.x; p < P; p += blockDim.x) out[p] = cmul(Wv[p], a.coef[p]);
  __syncthreads();
}

// plain type-4 solve of A[P] (p order) -> out[P] in ascending-node order
__device__ void tiny_t4(const TinySmem& s, const TinyArgs& a, const double2* A, double2* out) {
  const int P = a.P, n = 2 * P, K = P / 2;
  for (int p = threadIdx.x; p < P; p += blockDim.x) s.Y[p] = cmul(A[p], a.decay[p]);
  __syncthreads();
  double2* V = tiny_fft(s.Y, s.H, P, +1, s.tw, n);
  for (int p = threadIdx.x; p < P; p += blockDim.x) V[p] = cmul(V[p], a.ks[p]);
  __syncthreads();
  double2* Wv = tiny_fft(V, V == s.Y ? s.H : s.Y, P, -1, s.tw, n);
  // pad into T (n cells): F[(p - K) mod n] = Wv_p coef_p deconv_p
  for (int j = threadIdx.x; j < n; j += blockDim.x) {
    const int p = (j + K) % n;
    s.T[j] = p < P ? cscale(cmul(Wv[p], a.coef[p]), deconv_weight(p, K, n, a.b)) : make_double2(0.0, 0.0);
  }
  __syncthreads();
  double2* G = tiny_fft(s.T, s.H, n, +1, s.tw, n);
  for (int q = threadIdx.x; q < P; q += blockDim.x) out[q] = cmul(tiny_gather1(s, G, q, n), a.c4[q]);
  __syncthreads();
}

// kind 5 / 4; passes 0 or 1.  in/out: [batch][P] (type 5: samples in caller
// order -> coefficients in p order; type 4: spectrum in p order -> amplitudes
// in caller order).
__global__ void __launch_bounds__(kTThreads) k_tiny_solve(TinyArgs a, int kind, int passes,
                                                          const double2* __restrict__ in, double2* __restrict__ out) {
  extern __shared__ __align__(16) unsigned char smraw[];
  const int P = a.P, n = 2 * P, K = P / 2;
  TinySmem s;
  s.H = reinterpret_cast<double2*>(smraw);
  s.T = s.H + n;
  s.X = s.T + n;
  s.R = s.X + P;
  s.Y = s.R + P;
  s.tw = s.Y + P;
  s.W = reinterpret_cast<double*>(s.tw + P);
  s.tq = s.W + P * kTTaps;
  s.i0 = reinterpret_cast<int*>(s.tq + P);
  const double2* src = in + (int64_t)blockIdx.x * P;
  double2* dst = out + (int64_t)blockIdx.x * P;

  for (int k = threadIdx.x; k < P; k += blockDim.x) {  // n/2 = P twiddles
    double sn, cs;
    sincospi(-(double)k / (double)P, &sn, &cs);
    s.tw[k] = make_double2(cs, sn);
  }
  // node geometry and the factorised Gaussian weights (gridding.cu gauss_fast)
  for (int q = threadIdx.x; q < P; q += blockDim.x) {
    const double t = a.ts[q];
    const NodeGeo geo = node_geo(t, (double)n);
    s.tq[q] = t;
    s.i0[q] = geo.i0;
    double e1 = exp(-a.alpha * geo.f * geo.f);
    double E = exp(2.0 * a.alpha * geo.f);
    double Ei = 1.0 / E;
    double* w = s.W + q * kTTaps;
    w[kTM] = e1;
    double pp = e1, pn = e1;
#pragma unroll
    for (int k = 1; k <= kTM; k++) {
      pp *= E;
      pn *= Ei;
      w[kTM + k] = pp * a.G.g[k];
      w[kTM - k] = pn * a.G.g[k];
    }
    // solve input: type 5 -> spread amplitudes s_perm(q) c5_q; type 4 -> A_p
    s.R[q] = kind == 5 ? cmul(src[a.perm[q]], a.c5[q]) : src[q];
  }
  __syncthreads();

  if (kind == 5) {
    tiny_t5(s, a, s.R, s.X);  // x (p order)
    if (passes > 0) {
      // r_q = e^{+2 pi i K t_q} type2(x)_q - s_q  (forward.py:67-102), ascending nodes
      for (int j = threadIdx.x; j < n; j += blockDim.x) {
        const int p = (j + K) % n;
        s.T[j] = p < P ? cscale(s.X[p], deconv_weight(p, K, n, a.b)) : make_double2(0.0, 0.0);
      }
      __syncthreads();
      double2* G = tiny_fft(s.T, s.H, n, +1, s.tw, n);
      for (int q = threadIdx.x; q < P; q += blockDim.x) {
        const double2 v = cmul(tiny_gather1(s, G, q, n), cis_turns(turns_of_product((double)K, s.tq[q])));
        s.R[q] = cmul(csub(v, src[a.perm[q]]), a.c5[q]);  // the correction solve's spread amplitude
      }
      __syncthreads();
      tiny_t5(s, a, s.R, s.R);  // y = T5(r): R is consumed by the spread, then holds y
      for (int p = threadIdx.x; p < P; p += blockDim.x) dst[p] = csub(s.X[p], s.R[p]);
    } else {
      for (int p = threadIdx.x; p < P; p += blockDim.x) dst[p] = s.X[p];
    }
  } else {
    tiny_t4(s, a, s.R, s.X);  // x (ascending-node order)
    if (passes > 0) {
      // r_p = band(FFT_n(spread(x e^{-2 pi i K t}))) deconv - A_p  (forward.py:26-64)
      for (int q = threadIdx.x; q < P; q += blockDim.x)
        s.Y[q] = cmul(s.X[q], cis_turns(-turns_of_product((double)K, s.tq[q])));
      __syncthreads();
      tiny_spread(s, s.Y, P);
      double2* F = tiny_fft(s.H, s.T, n, -1, s.tw, n);
      for (int p = threadIdx.x; p < P; p += blockDim.x) {
        int bin = (p - K) % n;
        if (bin < 0) bin += n;
        s.R[p] = csub(cscale(F[bin], deconv_weight(p, K, n, a.b)), src[p]);
      }
      __syncthreads();
      tiny_t4(s, a, s.R, s.Y);  // y = T4(r) (Y is free again once the pad has consumed it)
      for (int q = threadIdx.x; q < P; q += blockDim.x) dst[a.perm[q]] = csub(s.X[q], s.Y[q]);
    } else {
      for (int q = threadIdx.x; q < P; q += blockDim.x) dst[a.perm[q]] = s.X[q];
    }
  }
}
}  // namespace

// Up to P * batch = 2^17 points the one-CTA solves win (B200, refined type-5 +
// type-4 step: P = 64 single 0.040 vs 0.120 ms, 64 x 1024 0.089 vs 0.195,
// 256 x 64 0.066 vs 0.202); at 256 x 1024 the general batched path is ahead
// (0.233 vs 0.279 ms).  NFFT45_NO_TINY=1 disables the path (A/B runs).
bool tiny_eligible(int64_t P, int m, int passes, int64_t batch) {
  static const bool off = getenv("NFFT45_NO_TINY") != nullptr;
  return !off && m == kTM && P >= 32 && P <= 256 && (P & (P - 1)) == 0 && passes <= 1 &&
         P * batch <= (int64_t(1) << 17);
}

int tiny_solve(const GridDev& g, int64_t P, double2 const* c5, double2 const* c4, const double2* decay,
               const double2* ks, const double2* coef, int kind, const double2* in, int64_t batch, int passes,
               double2* out, cudaStream_t st) {
  if (batch <= 0) return NFFT45_OK;
  Window win = Window::make(kTM);
  TinyArgs a{g.ts, g.perm, c5, c4, decay, ks, coef, (int)P, win.alpha, win.b, gauss_tab(win)};
  const size_t smem = sizeof(double2) * (2 * 2 * P + 4 * P) + sizeof(double) * P * (kTTaps + 1) + sizeof(int) * P;
  auto tiny = k_tiny_solve;  // the launched name keys the per-kernel profile
  if (smem > 48 * 1024) NFFT_CUDA(cudaFuncSetAttribute(tiny, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  LAUNCH(tiny, (unsigned)batch, kTThreads, smem, st, a, kind, passes < 0 ? 0 : passes, in, out);
  return NFFT45_OK;
}

}  // namespace nfft45
