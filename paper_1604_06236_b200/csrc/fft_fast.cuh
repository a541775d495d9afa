// fft_fast.cuh — compile-time-sized Stockham tile FFTs (fp64 complex).
//
// A tile is C independent length-N FFTs ("columns") done by one CTA of
// T = N*C/E threads, each thread owning E elements in registers:
//   pass 0      : loads its butterfly inputs straight from global memory
//                 through the caller's loader functor (fused prologue),
//   middle      : exchange through padded shared memory,
//   last pass   : stores straight to global memory through the caller's
//                 storer functor (fused epilogue: twiddles, tables, band
//                 selection ...).
// All index arithmetic is compile-time (shifts / masks).  Two thread
// mappings: CF (column-fast lanes, for column-contiguous global layouts)
// and JF (butterfly-fast lanes, for row-contiguous layouts).
#pragma once

#include <type_traits>

#include "fft.cuh"

namespace nfft45 {

__host__ __device__ constexpr bool is_pow2_c(int n) { return n > 0 && (n & (n - 1)) == 0; }
__host__ __device__ constexpr int log2_c(int n) { return n <= 1 ? 0 : 1 + log2_c(n >> 1); }

// elements per thread: 16 for 2^a, 24 for 3*2^a (divisible by 2,3,4,8)
template <int N>
struct FastTraits {
  static constexpr bool pow2 = is_pow2_c(N);
  static constexpr int E = pow2 ? 16 : 24;
  static constexpr int m2 = pow2 ? N : N / 3;  // power-of-two part
  static constexpr int a = log2_c(m2);
  // schedule for 2^a with radix-16 passes (pow2) or radix-8 passes (3*2^a);
  // the leftover small radix goes first (pass 0 has no twiddles).
  static constexpr int big = pow2 ? 16 : 8;
  static constexpr int bigbits = pow2 ? 4 : 3;
  static constexpr int rem = a % bigbits;
  static constexpr int nbig = a / bigbits;
  static constexpr int np = (pow2 ? 0 : 1) + (rem ? 1 : 0) + nbig;
  __host__ __device__ static constexpr int radix(int p) {
    // pass order: [3], [2^rem], big, big, ...
    return (!pow2 && p == 0) ? 3 : ((rem && p == (pow2 ? 0 : 1)) ? (1 << rem) : big);
  }
};

// 8 elements per thread, radix-8 passes (power-of-two N only): twice the
// threads of FastTraits<N> for the same tile, one more pass.  Used where a
// chain kernel's CTA is sized for a 2N-point FFT and the N-point stage
// would otherwise leave half the threads idle.
template <int N>
struct FastTraitsE8 {
  static_assert(is_pow2_c(N), "radix-8 schedule is for powers of two");
  static constexpr bool pow2 = true;
  static constexpr int E = 8;
  static constexpr int a = log2_c(N);
  static constexpr int rem = a % 3;
  static constexpr int nbig = a / 3;
  static constexpr int np = (rem ? 1 : 0) + nbig;
  __host__ __device__ static constexpr int radix(int p) { return (rem && p == 0) ? (1 << rem) : 8; }
};

// The M-point stage of a band / pad chain kernel runs in a CTA sized for the
// 2M-point FFT: with 8 elements per thread (radix-8 schedule) it uses all of
// its threads.  Signal-major and batch-minor chains use the same schedule,
// so batched and per-signal results stay bitwise identical.
template <int M>
using HalfTr = std::conditional_t<is_pow2_c(M), FastTraitsE8<M>, FastTraits<M>>;

template <int S>
__device__ __forceinline__ void bfly16(double2* v) {
  // radix-16 = 4 x radix-4 with W16 twiddles in between
  double2 a[16];
#pragma unroll
  for (int i = 0; i < 4; i++) {
    a[i] = v[i];
    a[4 + i] = v[4 + i];
    a[8 + i] = v[8 + i];
    a[12 + i] = v[12 + i];
  }
  // columns: elements {q, q+4, q+8, q+12} for q = 0..3
#pragma unroll
  for (int q = 0; q < 4; q++) bfly4<S>(a[q], a[q + 4], a[q + 8], a[q + 12]);
  // twiddle a[q + 4 p] *= W16^{q p}
  const double c1 = 0.92387953251128675613, s1 = 0.38268343236508977173, h = 0.70710678118654752440;
  const double2 w[10] = {
      make_double2(c1, S * s1), make_double2(h, S * h), make_double2(s1, S * c1),     // q=1: p=1,2,3
      make_double2(h, S * h), make_double2(0.0, S * 1.0), make_double2(-h, S * h),   // q=2
      make_double2(s1, S * c1), make_double2(-h, S * h), make_double2(-c1, -S * s1), // q=3
      make_double2(0, 0)};
#pragma unroll
  for (int q = 1; q < 4; q++)
#pragma unroll
    for (int p = 1; p < 4; p++) a[q + 4 * p] = cmul(a[q + 4 * p], w[(q - 1) * 3 + (p - 1)]);
  // rows: radix-4 over q for each p; output index p + 4 * k
#pragma unroll
  for (int p = 0; p < 4; p++) {
    double2 x0 = a[4 * p], x1 = a[4 * p + 1], x2 = a[4 * p + 2], x3 = a[4 * p + 3];
    bfly4<S>(x0, x1, x2, x3);
    v[p] = x0;
    v[p + 4] = x1;
    v[p + 8] = x2;
    v[p + 12] = x3;
  }
}

template <int R, int S>
__device__ __forceinline__ void bfly_fast(double2* v) {
  if constexpr (R == 16) bfly16<S>(v);
  else bfly<R, S>(v);
}

// Stockham twiddles w[r] = W^{r e} (r = 1..R-1) from the table W_N[.]:
// powers of two are loaded, the rest are products of at most three loaded
// values (<= 3 roundings), cutting L1 traffic from R-1 loads to log2(R).
template <int R>
__device__ __forceinline__ void twiddles(const double2* __restrict__ tw, int e, double2* w) {
  if constexpr (R == 3 || R == 5) {
#pragma unroll
    for (int r = 1; r < R; r++) w[r] = __ldg(&tw[r * e]);
  } else {
    w[1] = __ldg(&tw[e]);
    if constexpr (R >= 4) {
      w[2] = __ldg(&tw[2 * e]);
      w[3] = cmul(w[1], w[2]);
    }
    if constexpr (R >= 8) {
      w[4] = __ldg(&tw[4 * e]);
      w[5] = cmul(w[1], w[4]);
      w[6] = cmul(w[2], w[4]);
      w[7] = cmul(w[3], w[4]);
    }
    if constexpr (R >= 16) {
      w[8] = __ldg(&tw[8 * e]);
#pragma unroll
      for (int r = 1; r < 8; r++) w[8 + r] = cmul(w[r], w[8]);
    }
  }
}

// The same twiddles from the [4][N] power table of FftTables (section q =
// W_N^{k 2^q}): bitwise the values twiddles<R> loads, but lanes with
// consecutive e read consecutive words of every section.
template <int R, int N>
__device__ __forceinline__ void twiddles_pw(const double2* __restrict__ tw, int e, double2* w) {
  static_assert(R == 2 || R == 4 || R == 8 || R == 16, "power-table twiddles: radix 2/4/8/16");
  w[1] = __ldg(&tw[e]);
  if constexpr (R >= 4) {
    w[2] = __ldg(&tw[N + e]);
    w[3] = cmul(w[1], w[2]);
  }
  if constexpr (R >= 8) {
    w[4] = __ldg(&tw[2 * N + e]);
    w[5] = cmul(w[1], w[4]);
    w[6] = cmul(w[2], w[4]);
    w[7] = cmul(w[3], w[4]);
  }
  if constexpr (R >= 16) {
    w[8] = __ldg(&tw[3 * N + e]);
#pragma unroll
    for (int r = 1; r < 8; r++) w[8 + r] = cmul(w[r], w[8]);
  }
}

// For column-fast tiles the padding term is split so the index stays linear
// in i (c < C, C a power of two): tpad(i C + c) = i C + (i C >> 3) + c + (c >> 3)
// when 8 | C, and i C + c + i / (8 / C) when C < 8 — the same slots, but the
// per-element offsets of a butterfly fold into immediate offsets.
template <int N, int C, bool CF>
__device__ __forceinline__ int sidx(int i, int c) {
  if constexpr (CF && is_pow2_c(C) && C >= 8) return i * (C + C / 8) + c + (c >> 3);
  if constexpr (CF && is_pow2_c(C) && C < 8) return i * C + c + i / (8 / C);
  return CF ? tpad(i * C + c) : tpad(c * N + i);
}

// No post-twiddle (default for fast_tile_fft).
struct NoPostTw {
  template <int R, int STRIDE>
  __device__ __forceinline__ void apply(int, int, double2*) const {}
};

// Four-step inter-pass twiddle applied in the last pass: output index
// k = j + r*STRIDE of column `col` is multiplied by W_N^{S col k} with
//   W_N^{col j}           (two-level table lo/hi of N: 2 loads),
//   W_N^{col STRIDE 2^i}  (= W_Q^{col 2^i}, Q = N/STRIDE, 4 exact loads),
// and products for the other powers (<= 4 roundings) — 6 loads per
// butterfly instead of 2 per output element.
template <int S>
struct FourStepTw {
  const double2* lo;
  const double2* hi;
  int sh;
  const double2* twQ;  // W_Q^k, k < Q
  int Q;
  int col0;
  int cmask;  // tile column c maps to FFT column col0 + (c & cmask)
  template <int R, int STRIDE>
  __device__ __forceinline__ void apply(int c, int j, double2* v) const {
    const int64_t col = col0 + (c & cmask);
    const int64_t e = col * j;
    double2 base = cmul(__ldg(&hi[e >> sh]), __ldg(&lo[e & ((int64_t(1) << sh) - 1)]));
    double2 w[R];
    w[0] = base;
    if constexpr (R > 1) {
      double2 p[R];
      p[1] = __ldg(&twQ[col]);  // col * 8 < Q for every chain size (no reduction)
      if constexpr (R >= 4) {
        p[2] = __ldg(&twQ[2 * col]);
        p[3] = cmul(p[1], p[2]);
      }
      if constexpr (R >= 8) {
        p[4] = __ldg(&twQ[4 * col]);
        p[5] = cmul(p[1], p[4]);
        p[6] = cmul(p[2], p[4]);
        p[7] = cmul(p[3], p[4]);
      }
      if constexpr (R >= 16) {
        p[8] = __ldg(&twQ[8 * col]);
#pragma unroll
        for (int r = 1; r < 8; r++) p[8 + r] = cmul(p[r], p[8]);
      }
      if constexpr (R == 3) p[2] = __ldg(&twQ[2 * col]);
#pragma unroll
      for (int r = 1; r < R; r++) w[r] = cmul(base, p[r]);
    }
#pragma unroll
    for (int r = 0; r < R; r++) v[r] = S < 0 ? cmul(v[r], w[r]) : cmulc(v[r], w[r]);
  }
};

// Hook run by every thread at the end of the first pass, just before its
// barrier: kernels that stage per-tile tables with cp.async at entry wait for
// them here, so the copies overlap the first pass and are visible to the
// last pass's storer.
// `after()` runs once more right after the first pass's barrier (every thread
// has read its first-pass inputs): the TMA-staged kernels refill their input
// buffer with the next tile there.
// kOpaque: the tile FFT runs inside a persistent tile loop — every pass
// launders the thread index through an empty asm, so nvcc cannot hoist the
// per-pass thread-derived addresses out of the loop (live across tiles, they
// spill).
template <bool OPQ>
struct NoHookT {
  static constexpr bool kActive = false;
  static constexpr bool kOpaque = OPQ;
  __device__ __forceinline__ void operator()() const {}
  __device__ __forceinline__ void after() const {}
};
using NoHook = NoHookT<false>;
struct CpAsyncWaitHook {
  static constexpr bool kActive = true;
  static constexpr bool kOpaque = false;
  __device__ __forceinline__ void operator()() const { asm volatile("cp.async.wait_all;\n" ::); }
  __device__ __forceinline__ void after() const {}
};

// Synchronisation policy of a tile FFT: the whole CTA (default), or one
// GROUP of T threads of a persistent CTA whose groups work on different tiles
// (named barrier 1 + group id; thread index within the group).
struct CtaSync {
  __device__ __forceinline__ int tid() const { return threadIdx.x; }
  __device__ __forceinline__ void sync() const { __syncthreads(); }
};
template <int T>
struct GroupSync {
  int id;  // group index (named barrier id - 1)
  int t;   // thread index within the group
  __device__ __forceinline__ int tid() const { return t; }
  __device__ __forceinline__ void sync() const { asm volatile("bar.sync %0, %1;\n" ::"r"(id + 1), "n"(T) : "memory"); }
};

// One pass; FIRST reads through `ld`, LAST writes through `st`.  Threads
// with threadIdx.x >= T (a CTA sized for a bigger FFT of a chain) idle but
// still meet every barrier.  SYNC0: the first pass reads shared memory that
// its own stores overwrite (chain kernels), so it needs a barrier too.
template <int N, int C, int S, bool CF, bool SYNC0, int P, int Ns, class Tr, class Ld, class St, class PT,
          class Hk = NoHook, class Sy = CtaSync>
__device__ __forceinline__ void fast_passes(double2* sm, const Ld& ld, const St& st, const double2* __restrict__ tw,
                                            const PT& pt, const Hk& hook = Hk(), const Sy& sy = Sy()) {
  constexpr int E = Tr::E;
  constexpr int R = Tr::radix(P);
  constexpr int T = N * C / E;
  constexpr int MB = E / R;
  constexpr int stride = N / R;
  constexpr bool FIRST = (P == 0);
  constexpr bool LAST = (P == Tr::np - 1);
  int tid = sy.tid();
  if constexpr (Hk::kOpaque) asm volatile("" : "+r"(tid));
  const bool active = tid < T;
  double2 v[MB][R];
  if (active) {
#pragma unroll
  for (int u = 0; u < MB; u++) {
    const int bf = tid + u * T;
    const int c = CF ? (bf % C) : (bf / (N / R));
    const int j = CF ? (bf / C) : (bf % (N / R));
#pragma unroll
    for (int r = 0; r < R; r++) {
      const int i = j + r * stride;
      if constexpr (FIRST) v[u][r] = ld(i, c);
      else v[u][r] = sm[sidx<N, C, CF>(i, c)];
    }
  }
  }
  if constexpr (FIRST && LAST && Hk::kActive) hook();
  if constexpr (!FIRST || SYNC0 || (LAST && Hk::kActive)) sy.sync();  // everyone has read before anyone overwrites
  if (active) {
#pragma unroll
  for (int u = 0; u < MB; u++) {
    const int bf = tid + u * T;
    const int c = CF ? (bf % C) : (bf / (N / R));
    const int j = CF ? (bf / C) : (bf % (N / R));
    const int k = j % Ns;
    if constexpr (Ns > 1) {
      constexpr int tstep = N / (Ns * R);
      double2 w[R];
      twiddles<R>(tw, k * tstep, w);
#pragma unroll
      for (int r = 1; r < R; r++) v[u][r] = S < 0 ? cmul(v[u][r], w[r]) : cmulc(v[u][r], w[r]);
    }
    bfly_fast<R, S>(v[u]);
    if constexpr (LAST) pt.template apply<R, stride>(c, j, v[u]);  // outputs k = j + r*stride
    const int d = (j - k) * R + k;
#pragma unroll
    for (int r = 0; r < R; r++) {
      if constexpr (LAST) st(d + r * Ns, c, v[u][r]);
      else sm[sidx<N, C, CF>(d + r * Ns, c)] = v[u][r];
    }
  }
  }
  if constexpr (!LAST) {
    if constexpr (FIRST && Hk::kActive) hook();
    sy.sync();
    if constexpr (FIRST && Hk::kActive) hook.after();
    fast_passes<N, C, S, CF, SYNC0, P + 1, Ns * R, Tr>(sm, ld, st, tw, pt, NoHookT<Hk::kOpaque>(), sy);
  }
}

template <int N, int C, int S, bool CF, class Tr = FastTraits<N>, class Ld, class St, class PT = NoPostTw,
          class Hk = NoHook, class Sy = CtaSync>
__device__ __forceinline__ void fast_tile_fft(double2* sm, const Ld& ld, const St& st, const double2* __restrict__ tw,
                                              const PT& pt = PT(), const Hk& hook = Hk(), const Sy& sy = Sy()) {
  fast_passes<N, C, S, CF, false, 0, 1, Tr>(sm, ld, st, tw, pt, hook, sy);
}

// Variant whose first pass reads the tile from shared memory (via `ld`)
// that later passes overwrite.
template <int N, int C, int S, bool CF, class Tr = FastTraits<N>, class Ld, class St, class PT = NoPostTw,
          class Hk = NoHook, class Sy = CtaSync>
__device__ __forceinline__ void fast_tile_fft_smem(double2* sm, const Ld& ld, const St& st,
                                                   const double2* __restrict__ tw, const PT& pt = PT(),
                                                   const Hk& hook = Hk(), const Sy& sy = Sy()) {
  fast_passes<N, C, S, CF, true, 0, 1, Tr>(sm, ld, st, tw, pt, hook, sy);
}

// Run passes P0.. of a tile FFT whose earlier passes were produced directly
// in shared memory (Stockham layout after pass P0-1, Ns = NS0).
template <int N, int C, int S, bool CF, int P0, int NS0, class St, class PT = NoPostTw, class Hk = NoHook,
          class Sy = CtaSync>
__device__ __forceinline__ void fast_tile_fft_from(double2* sm, const St& st, const double2* __restrict__ tw,
                                                   const PT& pt = PT(), const Hk& hook = Hk(), const Sy& sy = Sy()) {
  auto no_ld = [](int, int) -> double2 { return make_double2(0.0, 0.0); };
  fast_passes<N, C, S, CF, false, P0, NS0, FastTraits<N>>(sm, no_ld, st, tw, pt, hook, sy);
}


// ------------------------------------------------------------------------
// Hybrid tile FFT for batch-minor tiles of 8 signals ([N][8] in shared
// memory).  The passes that touch global memory (first / last) keep the
// column-fast mapping (a warp = 4 consecutive indices x 8 signals: 128-byte
// global runs); the passes in between use a WARP-LOCAL mapping: the N / E
// threads that own one signal sit in one warp (E = 16, N = 512: warp w is
// signal w), so their exchanges through shared memory need only __syncwarp.
// A two-FFT chain kernel then has 2 CTA barriers per tile instead of 9-10,
// and its 8 warps drift apart between them: one warp's shared-memory phase
// overlaps another's fp64 phase instead of every warp of the CTA hitting the
// same pipe at once.  Every element sees the same butterflies and twiddles as
// in fast_passes (same radix schedule): results are bitwise identical.
//
// Layout: unpadded, XOR-swizzled.  Element (i, c) lives in 16-byte slot
// 8 i + (c ^ h(i)), h(i) = XOR of the base-8 digits of i: a row's 8 signals
// are 8 different bank groups (column-fast accesses), and so are 8 aligned
// consecutive indices of one signal, also at any power-of-two stride
// (warp-local accesses).  h is linear over disjoint bit fields, so for
// i = j + r * stride the per-element part is a compile-time XOR constant.
//
// h is a GF(2)-linear map of the index bits onto 3 bank-group bits, chosen so
// that every access pattern of the warp-local passes (8 aligned consecutive
// indices; strides 2 ... 256; the mixed patterns of the Stockham stores with
// Ns = 2 and 4) touches 8 distinct bank groups — checked exhaustively over
// all radix schedules of N = 64 ... 512:
//   h0 = i0 ^ i3 ^ i4 ^ i7,  h1 = i1 ^ i4 ^ i6 ^ i8,  h2 = i2 ^ i5 ^ i6.
__host__ __device__ constexpr int hsw8(int i) {
  return ((i & 7) ^ ((i >> 3) & 1) ^ ((i >> 4) & 1) * 3 ^ ((i >> 5) & 1) * 4 ^ ((i >> 6) & 1) * 6 ^ ((i >> 7) & 1) ^
          ((i >> 8) & 1) * 2);
}
__device__ __forceinline__ int hidx(int i, int c) { return (i << 3) + ((c ^ hsw8(i)) & 7); }

// lanes per signal of the warp-local mapping
template <int N, class Tr>
__host__ __device__ constexpr int hyb_lps() { return N / Tr::E; }
// a tile FFT can run hybrid: power of two, at most 32 threads per signal
template <int N, class Tr = FastTraits<N>>
__host__ __device__ constexpr bool hyb_ok() {
  return is_pow2_c(N) && N <= 512 && Tr::np >= 2 && hyb_lps<N, Tr>() <= 32 && hyb_lps<N, Tr>() >= 1;
}

// Passes P.. of the hybrid schedule.  WLMASK bit p: pass p is warp-local.
// SRC_SMEM: the first pass's `ld` reads this tile's shared memory (in-place
// hazard); DST_SMEM: the last pass's `st` writes shared memory.
//
// ROWST: the last pass's `st` writes row d (all 8 signals) of THIS tile's
// shared memory in some other slot order (the dense rows a TMA store reads).
// The last pass of a Stockham schedule writes exactly the indices it read
// (Ns = stride: d + r Ns = j + r stride), and the 8 threads of a row are
// adjacent lanes of one warp, so the in-place hazard needs only __syncwarp.
template <int N, int S, int P, int Ns, class Tr, unsigned WLMASK, bool SRC_SMEM, bool DST_SMEM, int P0, class Ld,
          class St, class PT, class Hk, int PEND = Tr::np, class Sy = CtaSync, bool ROWST = false>
__device__ __forceinline__ void hyb_passes(double2* sm, const Ld& ld, const St& st, const double2* __restrict__ tw,
                                           const PT& pt, const Hk& hook, const Sy& sy = Sy()) {
  constexpr int C = 8;
  constexpr int E = Tr::E;
  constexpr int R = Tr::radix(P);
  constexpr int T = N * C / E;
  constexpr int MB = E / R;
  constexpr int stride = N / R;
  constexpr int LPS = N / E;
  constexpr bool FIRST = (P == P0);
  constexpr bool LAST = (P == Tr::np - 1);
  constexpr bool WL = (WLMASK >> P) & 1u;
  constexpr bool LD_FN = FIRST && P0 == 0;  // the very first pass reads through `ld`
  const int tid = sy.tid();
  double2 v[MB][R];
#pragma unroll
  for (int u = 0; u < MB; u++) {
    const int c = WL ? tid / LPS : tid % C;
    const int j = WL ? (tid % LPS) + u * LPS : tid / C + u * (T / C);
    const int hj = (c ^ hsw8(j)) & 7;
#pragma unroll
    for (int r = 0; r < R; r++) {
      if constexpr (LD_FN) v[u][r] = ld(j + r * stride, c);
      else v[u][r] = sm[((j + r * stride) << 3) + (hj ^ hsw8(r * stride))];
    }
  }
  // in place: every read of the pass precedes every write of its sync domain
  if constexpr ((!LD_FN || SRC_SMEM) && (!LAST || DST_SMEM)) {
    if constexpr (WL) __syncwarp();
    else sy.sync();
  } else if constexpr (LAST && ROWST) {
    static_assert(!WL && Ns * R == N, "row-local in-place store: column-fast last pass");
    __syncwarp();
  }
#pragma unroll
  for (int u = 0; u < MB; u++) {
    const int c = WL ? tid / LPS : tid % C;
    const int j = WL ? (tid % LPS) + u * LPS : tid / C + u * (T / C);
    const int k = j % Ns;
    if constexpr (Ns > 1) {
      constexpr int tstep = N / (Ns * R);
      double2 w[R];
      if constexpr (WL) twiddles_pw<R, N>(tw, k * tstep, w);  // lanes = consecutive k: contiguous runs
      else twiddles<R>(tw, k * tstep, w);
#pragma unroll
      for (int r = 1; r < R; r++) v[u][r] = S < 0 ? cmul(v[u][r], w[r]) : cmulc(v[u][r], w[r]);
    }
    bfly_fast<R, S>(v[u]);
    if constexpr (LAST) pt.template apply<R, stride>(c, j, v[u]);  // outputs k = j + r*stride
    const int d = (j - k) * R + k;
    if constexpr (LAST) {
#pragma unroll
      for (int r = 0; r < R; r++) st(d + r * Ns, c, v[u][r]);
    } else {
      const int hd = (c ^ hsw8(d)) & 7;
#pragma unroll
      for (int r = 0; r < R; r++) sm[((d + r * Ns) << 3) + (hd ^ hsw8(r * Ns))] = v[u][r];
    }
  }
  if constexpr (!LAST) {
    constexpr bool WLN = (WLMASK >> (P + 1)) & 1u;
    if constexpr (FIRST && Hk::kActive) hook();
    if constexpr (WL && WLN) __syncwarp();
    else sy.sync();
    if constexpr (FIRST && Hk::kActive) hook.after();
    // PEND < np: the caller runs the remaining passes itself (fused handoff
    // to the next transform in registers); the boundary sync above is done
    if constexpr (P + 1 < PEND)
      hyb_passes<N, S, P + 1, Ns * R, Tr, WLMASK, SRC_SMEM, DST_SMEM, P0, Ld, St, PT, NoHook, PEND, Sy, ROWST>(
          sm, ld, st, tw, pt, NoHook(), sy);
  }
}

// passes 0 .. PEND-1 of a tile FFT (all of them write shared memory); ends
// with the sync that pass PEND's mapping (WLMASK bit PEND) needs
template <int N, int S, class Tr, unsigned WLMASK, int PEND, bool SRC_SMEM = false, class Ld, class Hk = NoHook,
          class Sy = CtaSync>
__device__ __forceinline__ void hyb_tile_fft_head(double2* sm, const Ld& ld, const double2* __restrict__ tw,
                                                  const Hk& hook = Hk(), const Sy& sy = Sy()) {
  auto no_st = [](int, int, double2) {};
  hyb_passes<N, S, 0, 1, Tr, WLMASK, SRC_SMEM, true, 0, Ld, decltype(no_st), NoPostTw, Hk, PEND, Sy>(
      sm, ld, no_st, tw, NoPostTw(), hook, sy);
}

// whole tile FFT, first pass through `ld`
template <int N, int S, class Tr, unsigned WLMASK, bool SRC_SMEM, bool DST_SMEM, class Ld, class St,
          class PT = NoPostTw, class Hk = NoHook>
__device__ __forceinline__ void hyb_tile_fft(double2* sm, const Ld& ld, const St& st, const double2* __restrict__ tw,
                                             const PT& pt = PT(), const Hk& hook = Hk()) {
  hyb_passes<N, S, 0, 1, Tr, WLMASK, SRC_SMEM, DST_SMEM, 0>(sm, ld, st, tw, pt, hook);
}
// passes P0.. of a tile FFT whose earlier passes were produced directly in
// shared memory (swizzled Stockham layout after pass P0 - 1, Ns = NS0)
template <int N, int S, class Tr, unsigned WLMASK, int P0, int NS0, class St, class PT = NoPostTw, class Sy = CtaSync,
          bool ROWST = false>
__device__ __forceinline__ void hyb_tile_fft_from(double2* sm, const St& st, const double2* __restrict__ tw,
                                                  const PT& pt = PT(), const Sy& sy = Sy()) {
  auto no_ld = [](int, int) -> double2 { return make_double2(0.0, 0.0); };
  hyb_passes<N, S, P0, NS0, Tr, WLMASK, true, false, P0, decltype(no_ld), St, PT, NoHook, Tr::np, Sy, ROWST>(
      sm, no_ld, st, tw, pt, NoHook(), sy);
}
// warp-local mask: every pass but the first (when it reads global memory)
// and the last (when it writes global memory)
template <class Tr>
__host__ __device__ constexpr unsigned hyb_mask(bool first_global, bool last_global) {
  unsigned m = (1u << Tr::np) - 1u;
  if (first_global) m &= ~1u;
  if (last_global) m &= ~(1u << (Tr::np - 1));
  return m;
}

// the last-pass stride (= N / radix of the last pass) of a fast tile FFT
template <int N, class Tr = FastTraits<N>>
__host__ __device__ constexpr int last_stride() { return N / Tr::radix(Tr::np - 1); }

template <int N, int C>
__host__ __device__ constexpr int fast_threads() { return N * C / FastTraits<N>::E; }

template <int N, int C>
__host__ __device__ constexpr size_t fast_smem() {
  return FastTraits<N>::np > 1 ? ((size_t)N * C + (size_t)N * C / 8 + 1) * sizeof(double2) : 16;
}

}  // namespace nfft45
