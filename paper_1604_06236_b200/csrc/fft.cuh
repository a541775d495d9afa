// fft.cuh — batched fp64 complex FFT engine (Stockham autosort, SMEM tiles).
//
// Replaces every np.fft call site on the hot path (forward.py:23,55,
// lagrange.py:125, inverse.py:115,134): X_k = sum_j x_j e^{sign 2 pi i jk/N},
// unnormalised in both directions.
//
//  * N <= kTileMax (smooth N = 2^a 3^b 5^c): one kernel, the whole transform
//    of C signals resident in one CTA's shared memory.
//  * larger smooth N: four-step N = N1 * N2, two SMEM passes (column FFTs
//    + twiddle, row FFTs with transposed store).
//  * non-smooth N: direct O(N^2) DFT with an exact integer twiddle index.
//
// The tile routines are also used by the fused solve-chain kernels (see
// chain.cu), which is why they are header-visible device functions.
#pragma once

#include "common.cuh"

namespace nfft45 {

constexpr int kTileMax = 4096;   // max elements of one tile FFT (64 KB fp64 complex)
constexpr int kMaxPasses = 16;

// Radix schedule of one tile FFT of length N (product of R[0..np)).
struct FftSeq {
  int N;
  int np;
  int R[kMaxPasses];
};

bool fft_smooth(int64_t N);
FftSeq fft_seq(int N);

// Twiddle tables, per device and length; immutable once built.
struct FftTables {
  int64_t N;
  double2* tw;   // W_N^k = e^{-2 pi i k / N}, k < N (only when N <= kTileMax or non-smooth)
                 // powers of two up to kTileMax: [4][N], section q holds W_N^{k 2^q} (section 0 = the
                 // plain table), so warp-local passes read their 2^q-th powers as contiguous runs
  double2* lo;   // four-step twiddles: W_N^k, k < 2^s
  double2* hi;   // W_N^{k 2^s}, k < ceil(N / 2^s)
  int s;
};
const FftTables* fft_tables(int64_t N, cudaStream_t st, int* status);

// Split a large smooth N into N1 * N2 (both smooth, <= kTileMax).
bool fft_split(int64_t N, int* N1, int* N2);

// out[b] = post .* FFT_sign(pre .* in[b]); pre/post are complex tables of
// length N broadcast over the batch (nullptr = identity).  in == out allowed.
int fft_run(const double2* in, double2* out, int64_t batch, int64_t N, int sign,
            const double2* pre, const double2* post, cudaStream_t st);

// ------------------------------------------------- shared-memory tile FFT

// Padded SMEM index of element (i, c) of an [Nt][C] tile: one 16-byte slot
// of padding per 8 elements keeps Stockham strides conflict-free for
// 128-bit accesses.
__device__ __forceinline__ int tpad(int e) { return e + (e >> 3); }

template <int S>
__device__ __forceinline__ double2 mul_si(double2 v) {  // v * (S i)
  return S < 0 ? make_double2(v.y, -v.x) : make_double2(-v.y, v.x);
}

template <int S>
__device__ __forceinline__ void bfly2(double2* v) {
  double2 a = v[0], b = v[1];
  v[0] = cadd(a, b);
  v[1] = csub(a, b);
}

template <int S>
__device__ __forceinline__ void bfly4(double2& x0, double2& x1, double2& x2, double2& x3) {
  double2 t0 = cadd(x0, x2), t1 = csub(x0, x2), t2 = cadd(x1, x3), t3 = mul_si<S>(csub(x1, x3));
  x0 = cadd(t0, t2);
  x2 = csub(t0, t2);
  x1 = cadd(t1, t3);
  x3 = csub(t1, t3);
}

template <int S>
__device__ __forceinline__ void bfly4v(double2* v) { bfly4<S>(v[0], v[1], v[2], v[3]); }

template <int S>
__device__ __forceinline__ void bfly8(double2* v) {
  const double h = 0.70710678118654752440;
  double2 e0 = v[0], e1 = v[2], e2 = v[4], e3 = v[6];
  double2 o0 = v[1], o1 = v[3], o2 = v[5], o3 = v[7];
  bfly4<S>(e0, e1, e2, e3);
  bfly4<S>(o0, o1, o2, o3);
  // W8^1 = (1 + S i)/sqrt2, W8^2 = S i, W8^3 = (-1 + S i)/sqrt2
  double2 w1 = make_double2(h * (o1.x - S * o1.y), h * (o1.y + S * o1.x));
  double2 w2 = mul_si<S>(o2);
  double2 w3 = make_double2(h * (-o3.x - S * o3.y), h * (-o3.y + S * o3.x));
  v[0] = cadd(e0, o0);
  v[4] = csub(e0, o0);
  v[1] = cadd(e1, w1);
  v[5] = csub(e1, w1);
  v[2] = cadd(e2, w2);
  v[6] = csub(e2, w2);
  v[3] = cadd(e3, w3);
  v[7] = csub(e3, w3);
}

template <int S>
__device__ __forceinline__ void bfly3(double2* v) {
  const double r3 = 0.86602540378443864676;  // sqrt(3)/2
  double2 a0 = v[0], s12 = cadd(v[1], v[2]);
  double2 d = mul_si<S>(csub(v[1], v[2]));
  double2 t = make_double2(fma(-0.5, s12.x, a0.x), fma(-0.5, s12.y, a0.y));
  v[0] = cadd(a0, s12);
  v[1] = make_double2(fma(r3, d.x, t.x), fma(r3, d.y, t.y));
  v[2] = make_double2(fma(-r3, d.x, t.x), fma(-r3, d.y, t.y));
}

template <int S>
__device__ __forceinline__ void bfly5(double2* v) {
  const double c1 = 0.30901699437494742410, c2 = -0.80901699437494742410;
  const double s1 = 0.95105651629515357212, s2 = 0.58778525229247312917;
  double2 a0 = v[0];
  double2 b1 = cadd(v[1], v[4]), b2 = cadd(v[2], v[3]);
  double2 d1 = csub(v[1], v[4]), d2 = csub(v[2], v[3]);
  double2 t1 = make_double2(fma(c2, b2.x, fma(c1, b1.x, a0.x)), fma(c2, b2.y, fma(c1, b1.y, a0.y)));
  double2 t2 = make_double2(fma(c1, b2.x, fma(c2, b1.x, a0.x)), fma(c1, b2.y, fma(c2, b1.y, a0.y)));
  double2 u1 = mul_si<S>(make_double2(fma(s1, d1.x, s2 * d2.x), fma(s1, d1.y, s2 * d2.y)));
  double2 u2 = mul_si<S>(make_double2(fma(s2, d1.x, -s1 * d2.x), fma(s2, d1.y, -s1 * d2.y)));
  v[0] = cadd(a0, cadd(b1, b2));
  v[1] = cadd(t1, u1);
  v[4] = csub(t1, u1);
  v[2] = cadd(t2, u2);
  v[3] = csub(t2, u2);
}

template <int R, int S>
__device__ __forceinline__ void bfly(double2* v) {
  if (R == 2) bfly2<S>(v);
  if (R == 3) bfly3<S>(v);
  if (R == 4) bfly4v<S>(v);
  if (R == 5) bfly5<S>(v);
  if (R == 8) bfly8<S>(v);
}

// Per-thread butterfly capacity per pass; launch with
// blockDim.x >= Nt * C / 12 so that every radix fits (R * (MAXE / R) >= 12).
constexpr int kTileElemsPerThread = 16;

// One Stockham pass of radix R over all C columns of an [Nt][C] tile.
template <int R, int S>
__device__ __forceinline__ void tile_pass(double2* sm, int Nt, int C, int Ns,
                                          const double2* __restrict__ tw) {
  constexpr int MB = kTileElemsPerThread / R;
  const int stride = Nt / R;
  const int nbf = stride * C;
  const int T = blockDim.x;
  double2 v[MB][R];
#pragma unroll
  for (int u = 0; u < MB; u++) {
    int bf = threadIdx.x + u * T;
    if (bf < nbf) {
      int c = bf % C, j = bf / C;
#pragma unroll
      for (int r = 0; r < R; r++) v[u][r] = sm[tpad((j + r * stride) * C + c)];
    }
  }
  __syncthreads();
  const int tstep = Nt / (Ns * R);
#pragma unroll
  for (int u = 0; u < MB; u++) {
    int bf = threadIdx.x + u * T;
    if (bf < nbf) {
      int c = bf % C, j = bf / C;
      int k = j % Ns;
      if (Ns > 1) {
#pragma unroll
        for (int r = 1; r < R; r++) {
          double2 w = __ldg(&tw[k * r * tstep]);
          v[u][r] = S < 0 ? cmul(v[u][r], w) : cmulc(v[u][r], w);
        }
      }
      bfly<R, S>(v[u]);
      int d = (j - k) * R + k;
#pragma unroll
      for (int r = 0; r < R; r++) sm[tpad((d + r * Ns) * C + c)] = v[u][r];
    }
  }
  __syncthreads();
}

// Full FFT of every column of the [Nt][C] tile (in place, natural order out).
// Caller must __syncthreads() after filling the tile.
template <int S>
__device__ void tile_fft(double2* sm, const FftSeq& seq, int C, const double2* __restrict__ tw) {
  int Ns = 1;
  for (int ip = 0; ip < seq.np; ip++) {
    int R = seq.R[ip];
    switch (R) {
      case 8: tile_pass<8, S>(sm, seq.N, C, Ns, tw); break;
      case 4: tile_pass<4, S>(sm, seq.N, C, Ns, tw); break;
      case 2: tile_pass<2, S>(sm, seq.N, C, Ns, tw); break;
      case 3: tile_pass<3, S>(sm, seq.N, C, Ns, tw); break;
      case 5: tile_pass<5, S>(sm, seq.N, C, Ns, tw); break;
    }
    Ns *= R;
  }
}

inline int tile_threads(int Nt, int C) {
  int need = (Nt * C + 11) / 12;
  int T = ((need + 31) / 32) * 32;
  if (T < 32) T = 32;
  if (T > 256) T = 256;
  return T;
}
inline size_t tile_smem_bytes(int Nt, int C) {
  size_t e = (size_t)Nt * C;
  return (e + e / 8 + 1) * sizeof(double2);
}

}  // namespace nfft45
