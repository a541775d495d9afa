// chain_bm.cu — the fused FFT chains of chain.cu for BATCHES, on a
// batch-minor internal layout X[index][signal] (signal stride 1, padded
// batch Bp = multiple of 8).
//
// P = R * C (R = C = M for even powers of two, R = 2C for odd ones, R = 3 * 2^a
// and C = 4R/3 for P = 3 * 2^k).  The
// P-point vectors use the layout p = k + R m (k < R, m < C); the fine grid
// n = 2P is split R x 2C for the FFT_2P / IFFT_2P four-steps, so with
// K = P/2 = R (C/2) the band (p - K) mod n of FFT_2P row k is exactly column
// k of the P layout (and, in the other direction, the zero-padded IFFT_2P
// column of P-layout row k).  Kernel tile lengths: col R, band 2C + C, mid
// R + R, pad C + 2C, row R, colin / rowout C.
//
// Every tile is one row (or column) of the four-step layout for 8 signals,
// so (i) global loads/stores are contiguous 128-byte runs over signals,
// (ii) the per-index tables (ks, deconv*decay, coef*deconv) and the
// four-step twiddles are warp-uniform broadcasts instead of per-element
// loads — the L1 data pipe, which limits the signal-major tiles, carries
// little more than the data itself.  The user's signal-major operands are
// converted in two boundary kernels with 2-D tiles (4 rows x 4 signals):
// kbm_colin (type-4 input) and kbm_rowout (type-5 output); the gridding
// kernels transpose through shared memory (gridding_b.cu).
//
// Stage semantics are those of chain.cu (inverse.py:101-143, forward.py:26-102).
#include <algorithm>
#include <cstdlib>
#include <type_traits>

#include "fft_fast.cuh"
#include "ops.cuh"
#include "tma.cuh"

// The file is compiled as TWO translation units (Makefile: -DNFFT45_BM_PART=1 / 2) so that the
// per-size instantiations of the chains build in parallel: part 1 holds the R = C sizes, the host
// helpers and the dispatch; part 2 the R = 2C and 3 * 2^k sizes.  Undefined: one unit with everything.
#ifndef NFFT45_BM_PART
#define NFFT45_BM_PART 0
#endif

namespace nfft45 {

namespace {
constexpr int kSig = 8;  // signals per tile (batch-minor kernels)

// CTAs per SM to request for a T-thread tile kernel: enough that every thread
// keeps ~128 registers (a 16-element tile FFT spills below that).
__host__ __device__ constexpr int bm_minb(int T) { return T >= 512 ? 1 : (T >= 256 ? 2 : 4); }
// signals per tile of the two-FFT kernels (tile lengths 2C and C): 8, or 4
// when 8 would need a CTA above 512 threads (C = 1024)
template <int C>
__host__ __device__ constexpr int bm_sg() { return fast_threads<2 * C, kSig>() > 512 ? kSig / 2 : kSig; }
// rows per tile of the boundary kernels (length C, 4 signals each): 4, or 2 for C = 1024
template <int C>
__host__ __device__ constexpr int bm_rw() { return fast_threads<C, 16>() > 512 ? 2 : 4; }

__device__ __forceinline__ double2 rsc(double2 v, double s) { return make_double2(v.x * s, v.y * s); }

__device__ __forceinline__ void cpa16(void* sdst, const void* gsrc) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(sdst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gsrc));
}
__device__ __forceinline__ void cpa_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cpa8(void* sdst, const void* gsrc) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(sdst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gsrc));
}

// L2 prefetch of the input tile of the CTA `pf` launch slots ahead (about one
// wave of resident CTAs): its DRAM reads then run while this wave computes,
// and that CTA's first pass hits L2 instead of waiting on DRAM.  No registers
// or shared memory are held for it (bulk prefetch, fire and forget).
__device__ __forceinline__ void pf_l2(const void* p, unsigned bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(p), "r"(bytes) : "memory");
}
// block coordinates (x, y) of the launch slot `pf` ahead, false past the grid
__device__ __forceinline__ bool ahead_block(int pf, unsigned& x, unsigned& y) {
  if (pf <= 0) return false;
  const unsigned long long nx =
      blockIdx.x + (unsigned long long)gridDim.x * blockIdx.y + (unsigned long long)pf;
  if (nx >= (unsigned long long)gridDim.x * gridDim.y) return false;
  x = (unsigned)(nx % gridDim.x);
  y = (unsigned)(nx / gridDim.x);
  return true;
}
// prefetch `rows` rows of `bytes` each, `stride` elements apart, from p
__device__ __forceinline__ void pf_rows(const double2* p, int64_t stride, int rows, unsigned bytes) {
  for (int i = threadIdx.x; i < rows; i += blockDim.x) pf_l2(p + (int64_t)i * stride, bytes);
}
}  // namespace

// column pass: columns n2 = blockIdx.x of x[i * L2 + n2] (length L), optional
// real pre-table, twiddle W_N^{S n2 k1}, in place-layout.
template <int L, int S>
__global__ void __launch_bounds__(fast_threads<L, kSig>(), bm_minb(fast_threads<L, kSig>())) kbm_col(
    const double2* __restrict__ in, double2* __restrict__ out, int L2, int64_t Bp, const double2* __restrict__ tw,
    const double2* __restrict__ lo, const double2* __restrict__ hi, int sh, const double2* __restrict__ twQ, int Q,
    const double* __restrict__ pre, int sw, int pf, int perm) {
  pdl_enter();  // programmatic dependent launch: wait for the producer grid
  extern __shared__ double2 sm[];
  const int n2 = sw ? blockIdx.y : blockIdx.x;
  const int64_t b0 = (int64_t)(sw ? blockIdx.x : blockIdx.y) * kSig;
  {
    unsigned ax, ay;
    if (ahead_block(pf, ax, ay))
      pf_rows(in + (int64_t)(sw ? ay : ax) * Bp + (int64_t)(sw ? ax : ay) * kSig, (int64_t)L2 * Bp, L,
              kSig * sizeof(double2));
  }
  // tile base pointers + 32-bit in-tile offsets (n * Bp < 2^31, guarded on the
  // host): the per-element address math stays out of 64-bit registers
  const unsigned ub = (unsigned)Bp;
  // perm: the producer (spreading) stored cell i L2 + n2 at row n2 L + i, so this column is one
  // contiguous range of L rows (DRAM reads like the row pass's instead of L scattered 128-byte runs)
  // (perm = block size cblk of the producer's row permutation, 0: natural order)
  const double2* __restrict__ it =
      in + (perm ? (int64_t)(n2 / perm) * L * perm + n2 % perm : (int64_t)n2) * Bp + b0;
  double2* __restrict__ ot = out + (int64_t)n2 * Bp + b0;
  const int istep = perm ? perm : L2;
  auto ld = [&](int i, int c) -> double2 {
    double2 v = it[(unsigned)(i * istep) * ub + c];
    if (pre) v = rsc(v, __ldg(&pre[(int64_t)i * L2 + n2]));
    return v;
  };
  auto st = [&](int k1, int c, double2 v) { ot[(unsigned)(k1 * L2) * ub + c] = v; };
  const FourStepTw<S> pt{lo, hi, sh, twQ, Q, n2, 0};
  fast_tile_fft<L, kSig, S, true>(sm, ld, st, tw, pt);
}

// kbm_col on the unpadded swizzled tile of the hybrid kernels (all passes column-fast: same
// butterflies and twiddles, bitwise identical) with the output leaving through the TMA unit: the
// last pass writes dense rows in place (ROWST), one thread stores L <= 256 rows k1 L2 + n2.
template <int L, int S>
__global__ void __launch_bounds__(fast_threads<L, kSig>(), bm_minb(fast_threads<L, kSig>())) kbm_col_s(
    const __grid_constant__ CUtensorMap tmO, const double2* __restrict__ in, int L2, int64_t Bp,
    const double2* __restrict__ tw, const double2* __restrict__ lo, const double2* __restrict__ hi, int sh,
    const double2* __restrict__ twQ, int Q, int perm) {
  pdl_enter();  // programmatic dependent launch: wait for the producer grid
  static_assert(L <= 512 && hyb_ok<L>(), "at most two TMA boxes, hybrid tile");
  extern __shared__ __align__(128) double2 sm_hs[];
  double2* sm = sm_hs;
  const int n2 = blockIdx.y;
  const int64_t b0 = (int64_t)blockIdx.x * kSig;
  const unsigned ub = (unsigned)Bp;
  const double2* __restrict__ it =
      in + (perm ? (int64_t)(n2 / perm) * L * perm + n2 % perm : (int64_t)n2) * Bp + b0;
  const int istep = perm ? perm : L2;
  auto ld = [&](int i, int c) -> double2 { return it[(unsigned)(i * istep) * ub + c]; };
  auto st = [&](int k1, int c, double2 v) { sm[(k1 << 3) + c] = v; };
  const FourStepTw<S> pt{lo, hi, sh, twQ, Q, n2, 0};
  using Tr = FastTraits<L>;
  hyb_passes<L, S, 0, 1, Tr, 0x0u, false, false, 0, decltype(ld), decltype(st), FourStepTw<S>, NoHook, Tr::np, CtaSync,
             true>(sm, ld, st, tw, pt, NoHook());
  fence_proxy_async();
  __syncthreads();
  if (threadIdx.x == 0) {
    constexpr int BOX = L < 256 ? L : 256;
#pragma unroll
    for (int k0 = 0; k0 < L; k0 += BOX) tma_store_3d(&tmO, (int)(2 * b0), n2, k0, sm + k0 * kSig);
    tma_store_commit();
    tma_store_wait_read();
  }
}

// row FFT_2P (row k1 < R, length 2C) -> band p = k1 + R m1 (m1 < C) with
// deconv*decay (or (X deconv - sub) decay) -> column IFFT_P (length C) ->
// W_P^{+k1 k1'} -> U[(k1' R + k1)][b].
// Per-tile tables (deconv*decay, or deconv and decay plus the subtrahend
// tile) are staged into shared memory with cp.async at entry; the copies fly
// during the first FFT pass (CpAsyncWaitHook) instead of stalling the band
// epilogue on L2 latency.
template <int R, int C, int SG>
__global__ void __launch_bounds__(fast_threads<2 * C, SG>(), bm_minb(fast_threads<2 * C, SG>())) kbm_band(
    const double2* __restrict__ T, double2* __restrict__ U, int64_t Bp, const double2* __restrict__ twR,
    const double2* __restrict__ twC, const double2* __restrict__ loP, const double2* __restrict__ hiP, int sP,
    const double2* __restrict__ twQ, int Q, const double* __restrict__ deconv, const double* __restrict__ decay,
    const double* __restrict__ dd, const double2* __restrict__ sub, int sw, int pf, double2* __restrict__ rsave) {
  pdl_enter();  // programmatic dependent launch: wait for the producer grid
  constexpr int NR = 2 * C;
  extern __shared__ double2 sm[];
  double* s_t0 = reinterpret_cast<double*>(reinterpret_cast<char*>(sm) + fast_smem<NR, SG>());
  double* s_t1 = s_t0 + C;
  double2* s_sb = reinterpret_cast<double2*>(s_t1 + C);
  const int k1 = sw ? blockIdx.y : blockIdx.x;
  const int64_t b0 = (int64_t)(sw ? blockIdx.x : blockIdx.y) * SG;
  {
    unsigned ax, ay;
    if (ahead_block(pf, ax, ay)) {
      const int64_t k = sw ? ay : ax, bb = (int64_t)(sw ? ax : ay) * SG;
      pf_rows(T + k * NR * Bp + bb, Bp, NR, SG * sizeof(double2));
      if (sub) pf_rows(sub + k * Bp + bb, (int64_t)R * Bp, C, SG * sizeof(double2));
    }
  }
  for (int m1 = threadIdx.x; m1 < C; m1 += blockDim.x) {
    const int64_t p = (int64_t)k1 + (int64_t)R * m1;
    if (sub) {
      cpa8(&s_t0[m1], &deconv[p]);
      cpa8(&s_t1[m1], &decay[p]);
    } else {
      cpa8(&s_t0[m1], &dd[p]);
    }
  }
  if (sub)
    for (int e = threadIdx.x; e < C * SG; e += blockDim.x)
      cpa16(&s_sb[e], &sub[((int64_t)k1 + (int64_t)R * (e / SG)) * Bp + b0 + e % SG]);
  cpa_commit();
  const unsigned ub = (unsigned)Bp;  // 32-bit in-tile offsets (see kbm_col)
  const double2* __restrict__ Tt = T + (int64_t)k1 * NR * Bp + b0;
  double2* __restrict__ Ut = U + (int64_t)k1 * Bp + b0;
  auto ld1 = [&](int i, int c) -> double2 { return Tt[(unsigned)i * ub + c]; };
  auto st1 = [&](int k2, int c, double2 v) {
    const int m1 = (k2 + C / 2) & (NR - 1);  // (k2 + K/R) mod 2C, K/R = C/2
    if (m1 < C) {
      if (sub) {
        v = rsc(v, s_t0[m1]);
        v = csub(v, s_sb[m1 * SG + c]);
        if (rsave) rsave[((int64_t)k1 + (int64_t)R * m1) * Bp + b0 + c] = v;  // r itself (norms, passes >= 2)
        v = rsc(v, s_t1[m1]);
      } else {
        v = rsc(v, s_t0[m1]);
      }
      sm[sidx<C, SG, true>(m1, c)] = v;
    }
  };
  fast_tile_fft<NR, SG, -1, true>(sm, ld1, st1, twR, NoPostTw(), CpAsyncWaitHook());
  __syncthreads();
  auto ld2 = [&](int i, int c) -> double2 { return sm[sidx<C, SG, true>(i, c)]; };
  auto st2 = [&](int k1p, int c, double2 v) { Ut[(unsigned)(k1p * R) * ub + c] = v; };
  const FourStepTw<+1> pt{loP, hiP, sP, twQ, Q, k1, 0};
  fast_tile_fft_smem<C, SG, +1, true, HalfTr<C>>(sm, ld2, st2, twC, pt);
}

// row IFFT_P (row r < C of U, length R) -> * ks[r + C k2] -> column FFT_P
// (length R, column r of the layout q = r + C k2) -> W_P^{-r k} -> Z[(k C + r)].
template <int R, int C>
__global__ void __launch_bounds__(fast_threads<R, kSig>(), bm_minb(fast_threads<R, kSig>())) kbm_mid(
    const double2* __restrict__ U, double2* __restrict__ Z, int64_t Bp, const double2* __restrict__ tw,
    const double2* __restrict__ loP, const double2* __restrict__ hiP, int sP, const double2* __restrict__ twQ, int Q,
    const double2* __restrict__ ks, int sw, int pf) {
  pdl_enter();  // programmatic dependent launch: wait for the producer grid
  extern __shared__ double2 sm[];
  double2* s_ks = reinterpret_cast<double2*>(reinterpret_cast<char*>(sm) + fast_smem<R, kSig>());
  const int r = sw ? blockIdx.y : blockIdx.x;
  const int64_t b0 = (int64_t)(sw ? blockIdx.x : blockIdx.y) * kSig;
  {
    unsigned ax, ay;
    if (ahead_block(pf, ax, ay))
      pf_rows(U + (int64_t)(sw ? ay : ax) * R * Bp + (int64_t)(sw ? ax : ay) * kSig, Bp, R, kSig * sizeof(double2));
  }
  for (int k2 = threadIdx.x; k2 < R; k2 += blockDim.x) cpa16(&s_ks[k2], &ks[(int64_t)r + (int64_t)C * k2]);
  cpa_commit();
  const unsigned ub = (unsigned)Bp;  // 32-bit in-tile offsets (see kbm_col)
  const double2* __restrict__ Ut = U + (int64_t)r * R * Bp + b0;
  double2* __restrict__ Zt = Z + (int64_t)r * Bp + b0;
  auto ld1 = [&](int i, int c) -> double2 { return Ut[(unsigned)i * ub + c]; };
  auto st1 = [&](int k2, int c, double2 v) { sm[sidx<R, kSig, true>(k2, c)] = cmul(v, s_ks[k2]); };
  fast_tile_fft<R, kSig, +1, true>(sm, ld1, st1, tw, NoPostTw(), CpAsyncWaitHook());
  __syncthreads();
  auto ld2 = [&](int i, int c) -> double2 { return sm[sidx<R, kSig, true>(i, c)]; };
  auto st2 = [&](int k, int c, double2 v) { Zt[(unsigned)(k * C) * ub + c] = v; };
  const FourStepTw<-1> pt{loP, hiP, sP, twQ, Q, r, 0};
  fast_tile_fft_smem<R, kSig, -1, true>(sm, ld2, st2, tw, pt);
}

// row FFT_P (row r < R of Z, length C) -> * coef (x = [xsub -] S coef stored
// when xout) * deconv -> zero-padded column IFFT_2P (length 2C, column r of
// the n = R x 2C layout) -> W_n^{+r k} -> Y[(k R + r)].
template <int R, int C, int SG>
__global__ void __launch_bounds__(fast_threads<2 * C, SG>(), bm_minb(fast_threads<2 * C, SG>())) kbm_pad(
    const double2* __restrict__ Z, double2* __restrict__ Y, int64_t Bp, const double2* __restrict__ twR,
    const double2* __restrict__ twC, const double2* __restrict__ loN, const double2* __restrict__ hiN, int sN,
    const double2* __restrict__ twQ, int Q, const double* __restrict__ coef, const double* __restrict__ deconv,
    const double* __restrict__ cd, const double2* __restrict__ xsub, double2* __restrict__ xout, int sw, int pf) {
  pdl_enter();  // programmatic dependent launch: wait for the producer grid
  constexpr int NC = 2 * C;
  constexpr bool kLead2 = FastTraits<NC>::radix(0) == 2;
  extern __shared__ double2 sm[];
  double* s_t0 = reinterpret_cast<double*>(reinterpret_cast<char*>(sm) + fast_smem<NC, SG>());
  double* s_t1 = s_t0 + C;
  double2* s_xs = reinterpret_cast<double2*>(s_t1 + C);
  const int r = sw ? blockIdx.y : blockIdx.x;
  const int64_t b0 = (int64_t)(sw ? blockIdx.x : blockIdx.y) * SG;
  // tile base pointers + 32-bit in-tile offsets (2C * Bp and R * C * Bp fit in
  // 31 bits, checked on the host): keeps the epilogue's address arithmetic out
  // of 64-bit registers (no spills at the 128-register budget)
  const unsigned ub = (unsigned)Bp;
  const double2* __restrict__ Zt = Z + (int64_t)r * C * Bp + b0;
  double2* __restrict__ Yt = Y + (int64_t)r * Bp + b0;
  double2* __restrict__ Xt = xout ? xout + (int64_t)r * Bp + b0 : nullptr;
  const double2* __restrict__ XSt = xsub ? xsub + (int64_t)r * Bp + b0 : nullptr;
  {
    unsigned ax, ay;
    if (ahead_block(pf, ax, ay)) {
      const int64_t k = sw ? ay : ax, bb = (int64_t)(sw ? ax : ay) * SG;
      pf_rows(Z + k * C * Bp + bb, Bp, C, SG * sizeof(double2));
      if (xout && xsub) pf_rows(xsub + k * Bp + bb, (int64_t)R * Bp, C, SG * sizeof(double2));
    }
  }
  // per-tile tables (and the xsub tile) staged with cp.async, waited for at
  // the end of the first FFT pass
  for (int k2 = threadIdx.x; k2 < C; k2 += blockDim.x) {
    const int64_t p = (int64_t)r + (int64_t)R * k2;
    if (xout) {
      cpa8(&s_t0[k2], &coef[p]);
      cpa8(&s_t1[k2], &deconv[p]);
    } else {
      cpa8(&s_t0[k2], &cd[p]);
    }
  }
  if (xout && xsub)
    for (int e = threadIdx.x; e < C * SG; e += blockDim.x)
      cpa16(&s_xs[e], &XSt[(unsigned)(R * (e / SG)) * ub + e % SG]);
  cpa_commit();
  auto ld1 = [&](int i, int c) -> double2 { return Zt[(unsigned)i * ub + c]; };
  auto st1 = [&](int k2, int c, double2 v) {
    if (xout) {
      v = rsc(v, s_t0[k2]);
      if (xsub) v = csub(s_xs[k2 * SG + c], v);
      Xt[(unsigned)(R * k2) * ub + c] = v;
      v = rsc(v, s_t1[k2]);
    } else {
      v = rsc(v, s_t0[k2]);
    }
    const int n1 = (k2 - C / 2) & (NC - 1);
    if constexpr (kLead2) {
      // The IFFT_2P column is zero outside the band, so its first Stockham
      // pass (radix 2, pairs n1 and n1 + C) is a copy: write its outputs
      // directly.  n1 in [0, C/2): partner zero -> (v, v); n1 in
      // [3C/2, 2C): partner zero on the other side -> (v, -v).
      if (n1 < C) {
        sm[sidx<NC, SG, true>(2 * n1, c)] = v;
        sm[sidx<NC, SG, true>(2 * n1 + 1, c)] = v;
      } else {
        const int j = n1 - C;
        sm[sidx<NC, SG, true>(2 * j, c)] = v;
        sm[sidx<NC, SG, true>(2 * j + 1, c)] = make_double2(-v.x, -v.y);
      }
    } else {
      sm[sidx<NC, SG, true>(n1, c)] = v;
      sm[sidx<NC, SG, true>((n1 + C) & (NC - 1), c)] = make_double2(0.0, 0.0);
    }
  };
  fast_tile_fft<C, SG, -1, true, HalfTr<C>>(sm, ld1, st1, twR, NoPostTw(), CpAsyncWaitHook());
  __syncthreads();
  auto st2 = [&](int k, int c, double2 v) { Yt[(unsigned)(k * R) * ub + c] = v; };
  const FourStepTw<+1> pt{loN, hiN, sN, twQ, Q, r, 0};
  if constexpr (kLead2) {
    fast_tile_fft_from<NC, SG, +1, true, 1, 2>(sm, st2, twC, pt);
  } else {
    auto ld2 = [&](int i, int c) -> double2 { return sm[sidx<NC, SG, true>(i, c)]; };
    fast_tile_fft_smem<NC, SG, +1, true>(sm, ld2, st2, twC, pt);
  }
}

// ------------------------------------------------------------------------
// Hybrid variants of the two-FFT kernels (see hyb_passes in fft_fast.cuh):
// the first pass (from global memory) and the last pass (to global memory)
// keep the column-fast mapping, every pass in between is warp-local on an
// unpadded XOR-swizzled tile, so a tile costs 2 CTA barriers instead of 9-10.
// Same arithmetic per element as kbm_band / kbm_mid / kbm_pad (bitwise
// identical results).  Used when both tile FFTs satisfy hyb_ok (powers of two
// with at most 32 threads per signal: every R = C and R = 2C chain up to
// P = 2^17).
template <int R, int C>
__host__ __device__ constexpr bool bm_hyb() {
  return bm_sg<C>() == kSig && hyb_ok<2 * C>() && hyb_ok<C, HalfTr<C>>() && hyb_ok<R>();
}

template <int R, int C>
__global__ void __launch_bounds__(fast_threads<2 * C, kSig>(), bm_minb(fast_threads<2 * C, kSig>())) kbm_band_h(
    const double2* __restrict__ T, double2* __restrict__ U, int64_t Bp, const double2* __restrict__ twR,
    const double2* __restrict__ twC, const double2* __restrict__ loP, const double2* __restrict__ hiP, int sP,
    const double2* __restrict__ twQ, int Q, const double* __restrict__ deconv, const double* __restrict__ decay,
    const double* __restrict__ dd, const double2* __restrict__ sub, double2* __restrict__ rsave) {
  pdl_enter();  // programmatic dependent launch: wait for the producer grid
  constexpr int NR = 2 * C;
  constexpr int SG = kSig;
  using TrA = FastTraits<NR>;
  using TrB = HalfTr<C>;
  extern __shared__ double2 sm[];
  double* s_t0 = reinterpret_cast<double*>(sm + NR * SG);
  double* s_t1 = s_t0 + C;
  double2* s_sb = reinterpret_cast<double2*>(s_t1 + C);
  const int k1 = blockIdx.y;
  const int64_t b0 = (int64_t)blockIdx.x * SG;
  for (int i = threadIdx.x; i < C / 2; i += blockDim.x) {  // tile-major tables: contiguous slices
    const int64_t o = (int64_t)k1 * C + 2 * i;
    if (sub) {
      cpa16(&s_t0[2 * i], &deconv[o]);
      cpa16(&s_t1[2 * i], &decay[o]);
    } else {
      cpa16(&s_t0[2 * i], &dd[o]);
    }
  }
  if (sub)  // subtrahend tile, swizzled like the data tile (it is read by warp-local lanes)
    for (int e = threadIdx.x; e < C * SG; e += blockDim.x)
      cpa16(&s_sb[hidx(e / SG, e % SG)], &sub[((int64_t)k1 + (int64_t)R * (e / SG)) * Bp + b0 + e % SG]);
  cpa_commit();
  const unsigned ub = (unsigned)Bp;  // 32-bit in-tile offsets (see kbm_col)
  const double2* __restrict__ Tt = T + (int64_t)k1 * NR * Bp + b0;
  double2* __restrict__ Ut = U + (int64_t)k1 * Bp + b0;
  auto ld1 = [&](int i, int c) -> double2 { return Tt[(unsigned)i * ub + c]; };
  auto st1 = [&](int k2, int c, double2 v) {
    const int m1 = (k2 + C / 2) & (NR - 1);  // (k2 + K/R) mod 2C, K/R = C/2
    if (m1 < C) {
      if (sub) {
        v = rsc(v, s_t0[m1]);
        v = csub(v, s_sb[hidx(m1, c)]);
        if (rsave) rsave[((int64_t)k1 + (int64_t)R * m1) * Bp + b0 + c] = v;  // r itself (norms, passes >= 2)
        v = rsc(v, s_t1[m1]);
      } else {
        v = rsc(v, s_t0[m1]);
      }
      sm[hidx(m1, c)] = v;
    }
  };
  hyb_tile_fft<NR, -1, TrA, hyb_mask<TrA>(true, false), false, true>(sm, ld1, st1, twR, NoPostTw(),
                                                                     CpAsyncWaitHook());
  __syncwarp();  // the band of signal c was written by the warp that transforms it next
  auto ld2 = [&](int i, int c) -> double2 { return sm[hidx(i, c)]; };
  auto st2 = [&](int k1p, int c, double2 v) { Ut[(unsigned)(k1p * R) * ub + c] = v; };
  const FourStepTw<+1> pt{loP, hiP, sP, twQ, Q, k1, 0};
  hyb_tile_fft<C, +1, TrB, hyb_mask<TrB>(false, true), true, false>(sm, ld2, st2, twC, pt);
}

template <int R, int C>
__global__ void __launch_bounds__(fast_threads<R, kSig>(), bm_minb(fast_threads<R, kSig>())) kbm_mid_h(
    const double2* __restrict__ U, double2* __restrict__ Z, int64_t Bp, const double2* __restrict__ tw,
    const double2* __restrict__ loP, const double2* __restrict__ hiP, int sP, const double2* __restrict__ twQ, int Q,
    const double2* __restrict__ ks) {
  pdl_enter();  // programmatic dependent launch: wait for the producer grid
  using Tr = FastTraits<R>;
  extern __shared__ double2 sm[];
  double2* s_ks = sm + R * kSig;
  const int r = blockIdx.y;
  const int64_t b0 = (int64_t)blockIdx.x * kSig;
  for (int k2 = threadIdx.x; k2 < R; k2 += blockDim.x) cpa16(&s_ks[k2], &ks[(int64_t)r * R + k2]);  // tile-major ks
  cpa_commit();
  const unsigned ub = (unsigned)Bp;  // 32-bit in-tile offsets (see kbm_col)
  const double2* __restrict__ Ut = U + (int64_t)r * R * Bp + b0;
  double2* __restrict__ Zt = Z + (int64_t)r * Bp + b0;
  auto ld1 = [&](int i, int c) -> double2 { return Ut[(unsigned)i * ub + c]; };
  auto st1 = [&](int k2, int c, double2 v) { sm[hidx(k2, c)] = cmul(v, s_ks[k2]); };
  hyb_tile_fft<R, +1, Tr, hyb_mask<Tr>(true, false), false, true>(sm, ld1, st1, tw, NoPostTw(), CpAsyncWaitHook());
  __syncwarp();
  auto ld2 = [&](int i, int c) -> double2 { return sm[hidx(i, c)]; };
  auto st2 = [&](int k, int c, double2 v) { Zt[(unsigned)(k * C) * ub + c] = v; };
  const FourStepTw<-1> pt{loP, hiP, sP, twQ, Q, r, 0};
  hyb_tile_fft<R, -1, Tr, hyb_mask<Tr>(false, true), true, false>(sm, ld2, st2, tw, pt);
}

// kbm_mid_h with the handoff between the two transforms kept in REGISTERS:
// for an all-radix-16 schedule (R = 256) the last pass of the IFFT leaves
// thread (signal c, j) with X[j + 16 r], r < 16 -- exactly the inputs of
// butterfly j of the FFT's first pass -- so IFFT pass 1, the ks product and
// FFT pass 0 run back to back on one register tile: 2 shared-memory round
// trips per tile instead of 3, same arithmetic per element (bitwise identical).
template <int R, int C>
__host__ __device__ constexpr bool bm_mid_fused() {
  return bm_hyb<R, C>() && FastTraits<R>::rem == 0 && FastTraits<R>::np == 2;
}

// TST: the last pass leaves dense rows [k][8] in the tile's shared memory and
// one thread stores them with the TMA unit (see kbm_pad_hs)
template <int R, int C, bool TST>
__device__ __forceinline__ void mid_hf_body(double2* sm, const CUtensorMap* tmZ,
    const double2* __restrict__ U, double2* __restrict__ Z, int64_t Bp, const double2* __restrict__ tw,
    const double2* __restrict__ loP, const double2* __restrict__ hiP, int sP, const double2* __restrict__ twQ, int Q,
    const double2* __restrict__ ks) {
  pdl_enter();  // programmatic dependent launch: wait for the producer grid
  using Tr = FastTraits<R>;
  static_assert(Tr::np == 2 && Tr::rem == 0, "fused handoff: schedule 16 x 16");
  constexpr int LPS = R / 16;  // lanes per signal = stride of the radix-16 passes
  double2* s_ks = sm + R * kSig;
  const int r = blockIdx.y;
  const int64_t b0 = (int64_t)blockIdx.x * kSig;
  for (int k2 = threadIdx.x; k2 < R; k2 += blockDim.x) cpa16(&s_ks[k2], &ks[(int64_t)r * R + k2]);  // tile-major ks
  cpa_commit();
  const unsigned ub = (unsigned)Bp;  // 32-bit in-tile offsets (see kbm_col)
  const double2* __restrict__ Ut = U + (int64_t)r * R * Bp + b0;
  double2* __restrict__ Zt = Z + (int64_t)r * Bp + b0;
  auto ld1 = [&](int i, int c) -> double2 { return Ut[(unsigned)i * ub + c]; };
  constexpr unsigned mask = 0x2u;  // pass 0 column-fast (global), pass 1 warp-local
  hyb_tile_fft_head<R, +1, Tr, mask, 1>(sm, ld1, tw, CpAsyncWaitHook());  // ends with a CTA barrier
  {
    const int tid = threadIdx.x;
    const int c = tid / LPS, j = tid % LPS;
    const int hj = (c ^ hsw8(j)) & 7;
    double2 v[16];
#pragma unroll
    for (int q = 0; q < 16; q++) v[q] = sm[((j + q * LPS) << 3) + (hj ^ hsw8(q * LPS))];
    __syncwarp();  // the signal's lanes have read before any of them overwrites
    {  // IFFT pass 1: Ns = R / 16 (k = j), twiddle step 1
      double2 w[16];
      twiddles_pw<16, R>(tw, j, w);
#pragma unroll
      for (int q = 1; q < 16; q++) v[q] = cmulc(v[q], w[q]);
    }
    bfly_fast<16, +1>(v);  // v[q] = X[j + q LPS]
#pragma unroll
    for (int q = 0; q < 16; q++) v[q] = cmul(v[q], s_ks[j + q * LPS]);
    bfly_fast<16, -1>(v);  // FFT pass 0 (no twiddles): outputs at 16 j + q
    const int d = j * 16;
    const int hd = (c ^ hsw8(d)) & 7;
#pragma unroll
    for (int q = 0; q < 16; q++) sm[((d + q) << 3) + (hd ^ hsw8(q))] = v[q];
  }
  __syncthreads();  // the last pass is column-fast
  const FourStepTw<-1> pt{loP, hiP, sP, twQ, Q, r, 0};
  if constexpr (TST) {
    static_assert(R <= 256, "one TMA box");
    auto st2 = [&](int k, int c, double2 v) { sm[(k << 3) + c] = v; };
    hyb_tile_fft_from<R, -1, Tr, 0x0u, 1, 16, decltype(st2), FourStepTw<-1>, CtaSync, true>(sm, st2, tw, pt);
    fence_proxy_async();
    __syncthreads();
    if (threadIdx.x == 0) {
      tma_store_3d(tmZ, (int)(2 * b0), r, 0, sm);
      tma_store_commit();
      tma_store_wait_read();
    }
  } else {
    auto st2 = [&](int k, int c, double2 v) { Zt[(unsigned)(k * C) * ub + c] = v; };
    hyb_tile_fft_from<R, -1, Tr, 0x0u, 1, 16>(sm, st2, tw, pt);
  }
}

template <int R, int C>
__global__ void __launch_bounds__(fast_threads<R, kSig>(), bm_minb(fast_threads<R, kSig>())) kbm_mid_hf(
    const double2* __restrict__ U, double2* __restrict__ Z, int64_t Bp, const double2* __restrict__ tw,
    const double2* __restrict__ loP, const double2* __restrict__ hiP, int sP, const double2* __restrict__ twQ, int Q,
    const double2* __restrict__ ks) {
  extern __shared__ double2 sm[];
  mid_hf_body<R, C, false>(sm, nullptr, U, Z, Bp, tw, loP, hiP, sP, twQ, Q, ks);
}
template <int R, int C>
__global__ void __launch_bounds__(fast_threads<R, kSig>(), bm_minb(fast_threads<R, kSig>())) kbm_mid_hs(
    const __grid_constant__ CUtensorMap tmZ, const double2* __restrict__ U, double2* __restrict__ Z, int64_t Bp,
    const double2* __restrict__ tw, const double2* __restrict__ loP, const double2* __restrict__ hiP, int sP,
    const double2* __restrict__ twQ, int Q, const double2* __restrict__ ks) {
  extern __shared__ __align__(128) double2 sm_hs[];
  mid_hf_body<R, C, true>(sm_hs, &tmZ, U, Z, Bp, tw, loP, hiP, sP, twQ, Q, ks);
}

// kbm_band_h with the band handoff in registers: after the last (radix-16)
// pass of the row FFT_2P (2C = 512) thread (signal c, j < 32) holds
// X[j + 32 r]; the in-band half, m1 = j + 32 s (s < 8), is exactly the input
// of butterflies j and j + 32 of the column IFFT_P's first (radix-4) pass.
template <int R, int C>
__host__ __device__ constexpr bool bm_band_fused() {
  return bm_hyb<R, C>() && C == 256;  // FFT_512 = 2 x 16 x 16, IFFT_256 = 4 x 8 x 8
}

template <int R, int C, bool TST>
__device__ __forceinline__ void band_hf_body(double2* sm, const CUtensorMap* tmU,
    const double2* __restrict__ T, double2* __restrict__ U, int64_t Bp, const double2* __restrict__ twR,
    const double2* __restrict__ twC, const double2* __restrict__ loP, const double2* __restrict__ hiP, int sP,
    const double2* __restrict__ twQ, int Q, const double* __restrict__ deconv, const double* __restrict__ decay,
    const double* __restrict__ dd, const double2* __restrict__ sub, double2* __restrict__ rsave) {
  pdl_enter();  // programmatic dependent launch: wait for the producer grid
  constexpr int NR = 2 * C;
  constexpr int SG = kSig;
  using TrA = FastTraits<NR>;
  using TrB = HalfTr<C>;
  static_assert(NR == 512 && TrA::np == 3 && TrB::np == 3 && TrB::radix(0) == 4, "fused band handoff: 512 / 256");
  double* s_t0 = reinterpret_cast<double*>(sm + NR * SG);
  double* s_t1 = s_t0 + C;
  double2* s_sb = reinterpret_cast<double2*>(s_t1 + C);
  const int k1 = blockIdx.y;
  const int64_t b0 = (int64_t)blockIdx.x * SG;
  for (int i = threadIdx.x; i < C / 2; i += blockDim.x) {  // tile-major tables: contiguous slices
    const int64_t o = (int64_t)k1 * C + 2 * i;
    if (sub) {
      cpa16(&s_t0[2 * i], &deconv[o]);
      cpa16(&s_t1[2 * i], &decay[o]);
    } else {
      cpa16(&s_t0[2 * i], &dd[o]);
    }
  }
  if (sub)  // subtrahend tile, swizzled like the data tile (it is read by warp-local lanes)
    for (int e = threadIdx.x; e < C * SG; e += blockDim.x)
      cpa16(&s_sb[hidx(e / SG, e % SG)], &sub[((int64_t)k1 + (int64_t)R * (e / SG)) * Bp + b0 + e % SG]);
  cpa_commit();
  const unsigned ub = (unsigned)Bp;  // 32-bit in-tile offsets (see kbm_col)
  const double2* __restrict__ Tt = T + (int64_t)k1 * NR * Bp + b0;
  double2* __restrict__ Ut = U + (int64_t)k1 * Bp + b0;
  auto ld1 = [&](int i, int c) -> double2 { return Tt[(unsigned)i * ub + c]; };
  constexpr unsigned maskA = 0x6u;  // pass 0 column-fast (global), passes 1, 2 warp-local
  hyb_tile_fft_head<NR, -1, TrA, maskA, 2>(sm, ld1, twR, CpAsyncWaitHook());  // passes 0, 1 (+ warp sync)
  {
    const int tid = threadIdx.x;
    const int c = tid >> 5, j = tid & 31;  // warp = signal
    const int hj = (c ^ hsw8(j)) & 7;
    double2 v[16];
#pragma unroll
    for (int q = 0; q < 16; q++) v[q] = sm[((j + q * 32) << 3) + (hj ^ hsw8(q * 32))];
    __syncwarp();
    {  // FFT_512 pass 2: Ns = 32 (k = j), twiddle step 1
      double2 w[16];
      twiddles_pw<16, NR>(twR, j, w);
#pragma unroll
      for (int q = 1; q < 16; q++) v[q] = cmul(v[q], w[q]);
    }
    bfly_fast<16, -1>(v);  // v[q] = X[k2 = j + 32 q]
    // band: m1 = (k2 + C/2) mod 2C = j + 32 s with s = (q + 4) mod 16 < 8
    double2 u[8];
#pragma unroll
    for (int s8 = 0; s8 < 8; s8++) {
      const int m1 = j + 32 * s8;
      double2 x = v[(s8 + 12) & 15];
      if (sub) {
        x = rsc(x, s_t0[m1]);
        x = csub(x, s_sb[hidx(m1, c)]);
        if (rsave) rsave[((int64_t)k1 + (int64_t)R * m1) * Bp + b0 + c] = x;  // r itself (norms, passes >= 2)
        x = rsc(x, s_t1[m1]);
      } else {
        x = rsc(x, s_t0[m1]);
      }
      u[s8] = x;
    }
    // column IFFT_P pass 0 (radix 4, stride 64): butterflies j (s = 0, 2, 4, 6) and j + 32 (s = 1, 3, 5, 7)
#pragma unroll
    for (int h = 0; h < 2; h++) {
      double2 x0 = u[h], x1 = u[2 + h], x2 = u[4 + h], x3 = u[6 + h];
      bfly4<+1>(x0, x1, x2, x3);
      const int d = (j + 32 * h) * 4;
      const int hd = (c ^ hsw8(d)) & 7;
      sm[((d + 0) << 3) + (hd ^ hsw8(0))] = x0;
      sm[((d + 1) << 3) + (hd ^ hsw8(1))] = x1;
      sm[((d + 2) << 3) + (hd ^ hsw8(2))] = x2;
      sm[((d + 3) << 3) + (hd ^ hsw8(3))] = x3;
    }
  }
  __syncwarp();  // pass 1 of the IFFT is warp-local
  const FourStepTw<+1> pt{loP, hiP, sP, twQ, Q, k1, 0};
  if constexpr (TST) {  // dense rows [k1'][8] in the first half of the tile buffer, stored by the TMA unit
    auto st2 = [&](int k1p, int c, double2 v) { sm[(k1p << 3) + c] = v; };
    hyb_tile_fft_from<C, +1, TrB, 0x2u, 1, 4, decltype(st2), FourStepTw<+1>, CtaSync, true>(sm, st2, twC, pt);
    fence_proxy_async();
    __syncthreads();
    if (threadIdx.x == 0) {
      tma_store_3d(tmU, (int)(2 * b0), k1, 0, sm);
      tma_store_commit();
      tma_store_wait_read();
    }
  } else {
    auto st2 = [&](int k1p, int c, double2 v) { Ut[(unsigned)(k1p * R) * ub + c] = v; };
    hyb_tile_fft_from<C, +1, TrB, 0x2u, 1, 4>(sm, st2, twC, pt);  // pass 1 warp-local, pass 2 column-fast
  }
}

template <int R, int C>
__global__ void __launch_bounds__(fast_threads<2 * C, kSig>(), bm_minb(fast_threads<2 * C, kSig>())) kbm_band_hf(
    const double2* __restrict__ T, double2* __restrict__ U, int64_t Bp, const double2* __restrict__ twR,
    const double2* __restrict__ twC, const double2* __restrict__ loP, const double2* __restrict__ hiP, int sP,
    const double2* __restrict__ twQ, int Q, const double* __restrict__ deconv, const double* __restrict__ decay,
    const double* __restrict__ dd, const double2* __restrict__ sub, double2* __restrict__ rsave) {
  extern __shared__ double2 sm[];
  band_hf_body<R, C, false>(sm, nullptr, T, U, Bp, twR, twC, loP, hiP, sP, twQ, Q, deconv, decay, dd, sub, rsave);
}
template <int R, int C>
__global__ void __launch_bounds__(fast_threads<2 * C, kSig>(), bm_minb(fast_threads<2 * C, kSig>())) kbm_band_hs(
    const __grid_constant__ CUtensorMap tmU, const double2* __restrict__ T, double2* __restrict__ U, int64_t Bp,
    const double2* __restrict__ twR, const double2* __restrict__ twC, const double2* __restrict__ loP,
    const double2* __restrict__ hiP, int sP, const double2* __restrict__ twQ, int Q,
    const double* __restrict__ deconv, const double* __restrict__ decay, const double* __restrict__ dd,
    const double2* __restrict__ sub, double2* __restrict__ rsave) {
  extern __shared__ __align__(128) double2 sm_hs[];
  band_hf_body<R, C, true>(sm_hs, &tmU, T, U, Bp, twR, twC, loP, hiP, sP, twQ, Q, deconv, decay, dd, sub, rsave);
}

// kbm_pad_h (no x output) with the zero-padding handoff done by ONE warp
// shuffle exchange: after the last (radix-8) pass of the row FFT_P (C = 256)
// lane j of the signal's warp holds S[k2 = j + 32 r]; butterfly j' = 2a + b of
// the first computed pass (radix 16, Ns = 2) of the zero-padded IFFT_2P needs
// V[s] = S[a + 16 s], s < 16 -- the values of lanes a (even s) and a + 16
// (odd s) -- as inputs q -> V[(q + 8) & 15] (times (-1)^b for q >= 8: the
// radix-2 first pass over the zero half is a copy, see kbm_pad).  Lanes a and
// a + 16 swap their eight values (__shfl_xor 16) and run butterflies b = 0 and
// b = 1: the padded tile is never written and re-read (8 instead of 12
// half-tile shared-memory transfers per tile).  Same arithmetic per element.
template <int R, int C>
__host__ __device__ constexpr bool bm_pad_fused() {
  return bm_hyb<R, C>() && C == 256;  // FFT_256 = 4 x 8 x 8, IFFT_512 = (2) x 16 x 16
}

__device__ __forceinline__ double2 shfl_xor16(double2 v) {
  return make_double2(__shfl_xor_sync(0xffffffffu, v.x, 16), __shfl_xor_sync(0xffffffffu, v.y, 16));
}

struct PadHfArgs {
  double2* Y;
  int64_t Bp;
  const double2 *twR, *twC, *loN, *hiN;
  int sN;
  const double2* twQ;
  int Q;
  const double* cd;
  int ntiles, groups;
};

// one tile (row r, signals b0 ..) of the fused pad; `ld1` reads the tile's Z
// rows (global memory, or a TMA-staged dense copy), `sy` is the CTA or one
// tile group of a persistent CTA
template <int R, int C, bool TST = false, class Ld, class Hk, class Sy>
__device__ __forceinline__ void pad_hf_tile(const PadHfArgs& a, double2* sm, double* s_t0, const Ld& ld1,
                                            const Hk& hook, int r, int64_t b0, const Sy& sy) {
  constexpr int NC = 2 * C;
  using TrA = HalfTr<C>;
  using TrB = FastTraits<NC>;
  static_assert(NC == 512 && TrA::np == 3 && TrA::radix(2) == 8 && TrB::np == 3 && TrB::radix(0) == 2,
                "fused pad handoff: 256 / 512");
  const unsigned ub = (unsigned)a.Bp;
  double2* __restrict__ Yt = a.Y + (int64_t)r * a.Bp + b0;
  hyb_tile_fft_head<C, -1, TrA, 0x6u, 2>(sm, ld1, a.twR, hook, sy);  // passes 0 (global / staged), 1 (+ warp sync)
  {
    const int tid = sy.tid();
    const int c = tid >> 5, j = tid & 31;  // warp = signal
    const int hj = (c ^ hsw8(j)) & 7;
    double2 v[8];
#pragma unroll
    for (int q = 0; q < 8; q++) v[q] = sm[((j + q * 32) << 3) + (hj ^ hsw8(q * 32))];
    __syncwarp();
    {  // FFT_256 pass 2 (radix 8): Ns = 32 (k = j), twiddle step 1
      double2 w[8];
      twiddles_pw<8, C>(a.twR, j, w);
#pragma unroll
      for (int q = 1; q < 8; q++) v[q] = cmul(v[q], w[q]);
    }
    bfly_fast<8, -1>(v);  // v[q] = S[k2 = j + 32 q]
#pragma unroll
    for (int q = 0; q < 8; q++) v[q] = rsc(v[q], s_t0[j + 32 * q]);
    // V[s] = S[a + 16 s]: even s from lane a, odd s from lane a + 16
    const int la = j & 15, b = j >> 4;
    double2 in[16];
#pragma unroll
    for (int q = 0; q < 8; q++) {
      const double2 o = shfl_xor16(v[q]);
      const double2 ev = b ? o : v[q];  // V[2 q]
      const double2 od = b ? v[q] : o;  // V[2 q + 1]
      // input q' of the butterfly = V[(q' + 8) & 15], negated for q' >= 8 when b = 1
      const int qe = (2 * q + 8) & 15, qo = (2 * q + 1 + 8) & 15;
      in[qe] = (qe >= 8 && b) ? make_double2(-ev.x, -ev.y) : ev;
      in[qo] = (qo >= 8 && b) ? make_double2(-od.x, -od.y) : od;
    }
    {  // IFFT_512 pass 1 (radix 16): Ns = 2 (k = b), twiddle step 16
      double2 w[16];
      twiddles_pw<16, NC>(a.twC, b * 16, w);
#pragma unroll
      for (int q = 1; q < 16; q++) in[q] = cmulc(in[q], w[q]);
    }
    bfly_fast<16, +1>(in);
    const int d = 32 * la + b;  // (j' - k) * 16 + k with j' = 2 a + b
    const int hd = (c ^ hsw8(d)) & 7;
#pragma unroll
    for (int q = 0; q < 16; q++) sm[((d + 2 * q) << 3) + (hd ^ hsw8(2 * q))] = in[q];
  }
  sy.sync();  // the last pass is column-fast
  const FourStepTw<+1> pt{a.loN, a.hiN, a.sN, a.twQ, a.Q, r, 0};
  if constexpr (TST) {  // dense rows [k][8] in place; the caller stores them with the TMA unit
    auto st2 = [&](int k, int c, double2 v) { sm[(k << 3) + c] = v; };
    hyb_tile_fft_from<NC, +1, TrB, 0x0u, 2, 32, decltype(st2), FourStepTw<+1>, Sy, true>(sm, st2, a.twC, pt, sy);
  } else {
    auto st2 = [&](int k, int c, double2 v) { Yt[(unsigned)(k * R) * ub + c] = v; };
    hyb_tile_fft_from<NC, +1, TrB, 0x0u, 2, 32>(sm, st2, a.twC, pt, sy);
  }
}

template <int R, int C>
__global__ void __launch_bounds__(fast_threads<2 * C, kSig>(), bm_minb(fast_threads<2 * C, kSig>())) kbm_pad_hf(
    const double2* __restrict__ Z, const __grid_constant__ PadHfArgs a) {
  pdl_enter();  // programmatic dependent launch: wait for the producer grid
  constexpr int NC = 2 * C;
  extern __shared__ double2 sm[];
  double* s_t0 = reinterpret_cast<double*>(sm + NC * kSig);
  const int r = blockIdx.y;
  const int64_t b0 = (int64_t)blockIdx.x * kSig;
  const unsigned ub = (unsigned)a.Bp;
  const double2* __restrict__ Zt = Z + (int64_t)r * C * a.Bp + b0;
  for (int i = threadIdx.x; i < C / 2; i += blockDim.x) cpa16(&s_t0[2 * i], &a.cd[(int64_t)r * C + 2 * i]);  // tile-major
  cpa_commit();
  auto ld1 = [&](int i, int c) -> double2 { return Zt[(unsigned)i * ub + c]; };
  pad_hf_tile<R, C>(a, sm, s_t0, ld1, CpAsyncWaitHook(), r, b0, CtaSync());
}

// kbm_pad_hf whose output leaves through the TMA unit: the last pass writes
// its rows back into the tile's shared memory (dense [k][8], in place — see
// ROWST in fft_fast.cuh), then one thread issues two bulk tensor stores (SASS
// UTMASTG) of 256 rows each to rows k R + r of Y.  The 2 units of output of
// the zero-padded first IFFT_2P pass cost STS wavefronts instead of STG ones
// (about half the L1 data-pipe cycles per byte).
template <int R, int C>
__global__ void __launch_bounds__(fast_threads<2 * C, kSig>(), bm_minb(fast_threads<2 * C, kSig>())) kbm_pad_hs(
    const double2* __restrict__ Z, const __grid_constant__ CUtensorMap tmY, const __grid_constant__ PadHfArgs a) {
  pdl_enter();  // programmatic dependent launch: wait for the producer grid
  constexpr int NC = 2 * C;
  extern __shared__ __align__(128) double2 sm_hs[];
  double2* sm = sm_hs;
  double* s_t0 = reinterpret_cast<double*>(sm + NC * kSig);
  const int r = blockIdx.y;
  const int64_t b0 = (int64_t)blockIdx.x * kSig;
  const unsigned ub = (unsigned)a.Bp;
  const double2* __restrict__ Zt = Z + (int64_t)r * C * a.Bp + b0;
  for (int i = threadIdx.x; i < C / 2; i += blockDim.x) cpa16(&s_t0[2 * i], &a.cd[(int64_t)r * C + 2 * i]);  // tile-major
  cpa_commit();
  auto ld1 = [&](int i, int c) -> double2 { return Zt[(unsigned)i * ub + c]; };
  pad_hf_tile<R, C, true>(a, sm, s_t0, ld1, CpAsyncWaitHook(), r, b0, CtaSync());
  fence_proxy_async();  // this thread's rows become visible to the async proxy
  __syncthreads();
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k0 = 0; k0 < NC; k0 += 256) tma_store_3d(&tmY, (int)(2 * b0), r, k0, sm + k0 * kSig);
    tma_store_commit();
    tma_store_wait_read();
  }
}

// Persistent form of kbm_pad_hf: ONE CTA per SM made of two tile groups of
// 256 threads (named barriers), each with its own work tile, table slot, TMA
// staging buffer and mbarrier.  A group's next Z tile is requested (one bulk
// tensor copy, SASS UTMALDG) right after its first pass has consumed the
// staged one, so the tile's DRAM latency hides under the current tile's
// remaining passes and no registers idle behind a load.  The tile body is a
// real call: inlined into the loop, ptxas keeps ~30 more registers live across
// the barriers and spills > 1 KB per thread.
// First-pass hook of the persistent kernels: wait for this thread's cp.async
// table copies before the group barrier; after it (every thread of the group
// has pulled the staged tile into registers) thread 0 refills the staging
// buffer with the group's next tile of ROWS rows.
template <int ROWS>
struct TmaRefill {
  static constexpr bool kActive = true;
  static constexpr bool kOpaque = false;
  const CUtensorMap* map;
  double2* dst;
  uint64_t* bar;
  int tn, ntiles, groups;
  int tid;
  __device__ __forceinline__ void operator()() const { asm volatile("cp.async.wait_all;\n" ::); }
  __device__ __forceinline__ void after() const {
    if (tid == 0 && tn < ntiles) {
      fence_proxy_async();  // the group's generic reads of the buffer precede the async refill
      mbar_expect_tx(bar, (unsigned)(ROWS * kSig * sizeof(double2)));
      tma_load_2d(dst, map, 2 * kSig * (tn % groups), ROWS * (tn / groups), bar);
    }
  }
};

template <int R, int C>
struct PadHpLayout {
  static constexpr size_t kWork = sizeof(double2) * 2 * C * kSig + sizeof(double) * C;  // tile + cd slot
  static constexpr size_t kStage = sizeof(double2) * C * kSig;                          // dense TMA box
  static constexpr size_t kGroup = (kWork + kStage + 127) / 128 * 128;
  static constexpr size_t kBytes = 2 * kGroup + 16;
};

template <int R, int C>
__device__ __noinline__ bool pad_hp_body(const CUtensorMap* tmZ, const PadHfArgs* ap, unsigned char* smraw, int it) {
  constexpr int T = fast_threads<2 * C, kSig>();
  using L = PadHpLayout<R, C>;
  const PadHfArgs& a = *ap;
  const int g = threadIdx.x / T;
  const GroupSync<T> sy{g, (int)threadIdx.x - g * T};
  const int stride = 2 * gridDim.x;
  const int t = 2 * blockIdx.x + g + it * stride;
  if (t >= a.ntiles) return false;
  double2* inb = reinterpret_cast<double2*>(smraw + g * L::kGroup);  // [C][8] dense (TMA box), 128-byte aligned
  double2* sm = reinterpret_cast<double2*>(smraw + g * L::kGroup + L::kStage);
  double* s_t0 = reinterpret_cast<double*>(sm + 2 * C * kSig);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smraw + 2 * L::kGroup) + g;
  const int r = t / a.groups;
  const int64_t b0 = (int64_t)(t % a.groups) * kSig;
  sy.sync();  // the group's previous tile is done with `sm` and the table slot
  for (int i = sy.t; i < C / 2; i += T) cpa16(&s_t0[2 * i], &a.cd[(int64_t)r * C + 2 * i]);  // tile-major
  cpa_commit();
  mbar_wait(bar, it & 1);
  const TmaRefill<C> hook{tmZ, inb, bar, t + stride, a.ntiles, a.groups, sy.t};
  auto ld1 = [&](int i, int c) -> double2 { return inb[i * kSig + c]; };
  pad_hf_tile<R, C>(a, sm, s_t0, ld1, hook, r, b0, sy);
  return true;
}

template <int R, int C>
__global__ void __launch_bounds__(2 * fast_threads<2 * C, kSig>(), 1) kbm_pad_hp(
    const __grid_constant__ CUtensorMap tmZ, const __grid_constant__ PadHfArgs a) {
  constexpr int T = fast_threads<2 * C, kSig>();
  using L = PadHpLayout<R, C>;
  extern __shared__ __align__(128) unsigned char smraw_hp[];
  {
    const int g = threadIdx.x / T;
    uint64_t* bar = reinterpret_cast<uint64_t*>(smraw_hp + 2 * L::kGroup) + g;
    if ((int)threadIdx.x - g * T == 0) {
      if (g == 0) tma_prefetch_desc(&tmZ);
      mbar_init(bar, 1);
      mbar_fence_init();
    }
  }
  __syncthreads();
  pdl_enter();  // programmatic dependent launch: Z is the producer's output
  {
    const int g = threadIdx.x / T;
    const int t = 2 * blockIdx.x + g;
    if ((int)threadIdx.x - g * T == 0 && t < a.ntiles) {
      uint64_t* bar = reinterpret_cast<uint64_t*>(smraw_hp + 2 * L::kGroup) + g;
      mbar_expect_tx(bar, (unsigned)L::kStage);
      tma_load_2d(smraw_hp + g * L::kGroup, &tmZ, 2 * kSig * (t % a.groups), C * (t / a.groups), bar);
    }
  }
#pragma unroll 1
  for (int it = 0; pad_hp_body<R, C>(&tmZ, &a, smraw_hp, it); it++) {
  }
}

// XOUT: the tile also stores x (coalesced rows), so the last pass of the
// C-point FFT keeps the column-fast mapping and is followed by a CTA barrier.
// TST: the padded grid Y leaves through the TMA unit (dense rows written in
// place by the last pass, bulk tensor stores of <= 256 rows; see kbm_pad_hs).
template <int R, int C, bool XOUT, bool TST>
__device__ __forceinline__ void pad_h_body(double2* sm, const CUtensorMap* tmY,
    const double2* __restrict__ Z, double2* __restrict__ Y, int64_t Bp, const double2* __restrict__ twR,
    const double2* __restrict__ twC, const double2* __restrict__ loN, const double2* __restrict__ hiN, int sN,
    const double2* __restrict__ twQ, int Q, const double* __restrict__ coef, const double* __restrict__ deconv,
    const double* __restrict__ cd, const double2* __restrict__ xsub, double2* __restrict__ xout) {
  pdl_enter();  // programmatic dependent launch: wait for the producer grid
  constexpr int NC = 2 * C;
  constexpr int SG = kSig;
  using TrA = HalfTr<C>;
  using TrB = FastTraits<NC>;
  constexpr bool kLead2 = TrB::radix(0) == 2;
  static_assert(!TST || kLead2, "TMA-store form: power-of-two tiles");
  double* s_t0 = reinterpret_cast<double*>(sm + NC * SG);
  double* s_t1 = s_t0 + C;
  double2* s_xs = reinterpret_cast<double2*>(s_t1 + C);
  const int r = blockIdx.y;
  const int64_t b0 = (int64_t)blockIdx.x * SG;
  const unsigned ub = (unsigned)Bp;
  const double2* __restrict__ Zt = Z + (int64_t)r * C * Bp + b0;
  double2* __restrict__ Yt = Y + (int64_t)r * Bp + b0;
  double2* __restrict__ Xt = XOUT ? xout + (int64_t)r * Bp + b0 : nullptr;
  const double2* __restrict__ XSt = (XOUT && xsub) ? xsub + (int64_t)r * Bp + b0 : nullptr;
  for (int i = threadIdx.x; i < C / 2; i += blockDim.x) {  // tile-major tables: contiguous slices
    const int64_t o = (int64_t)r * C + 2 * i;
    if (XOUT) {
      cpa16(&s_t0[2 * i], &coef[o]);
      cpa16(&s_t1[2 * i], &deconv[o]);
    } else {
      cpa16(&s_t0[2 * i], &cd[o]);
    }
  }
  if (XOUT && xsub)
    for (int e = threadIdx.x; e < C * SG; e += blockDim.x)
      cpa16(&s_xs[e], &XSt[(unsigned)(R * (e / SG)) * ub + e % SG]);
  cpa_commit();
  auto ld1 = [&](int i, int c) -> double2 { return Zt[(unsigned)i * ub + c]; };
  auto st1 = [&](int k2, int c, double2 v) {
    if (XOUT) {
      v = rsc(v, s_t0[k2]);
      if (xsub) v = csub(s_xs[k2 * SG + c], v);
      Xt[(unsigned)(R * k2) * ub + c] = v;
      v = rsc(v, s_t1[k2]);
    } else {
      v = rsc(v, s_t0[k2]);
    }
    const int n1 = (k2 - C / 2) & (NC - 1);
    if constexpr (kLead2) {
      // first Stockham pass (radix 2) of the zero-padded column: a copy (see kbm_pad)
      if (n1 < C) {
        sm[hidx(2 * n1, c)] = v;
        sm[hidx(2 * n1 + 1, c)] = v;
      } else {
        const int j = n1 - C;
        sm[hidx(2 * j, c)] = v;
        sm[hidx(2 * j + 1, c)] = make_double2(-v.x, -v.y);
      }
    } else {
      sm[hidx(n1, c)] = v;
      sm[hidx((n1 + C) & (NC - 1), c)] = make_double2(0.0, 0.0);
    }
  };
  constexpr unsigned maskA = hyb_mask<TrA>(true, XOUT);
  hyb_tile_fft<C, -1, TrA, maskA, false, true>(sm, ld1, st1, twR, NoPostTw(), CpAsyncWaitHook());
  if constexpr (XOUT) __syncthreads();
  else __syncwarp();
  auto st2 = [&](int k, int c, double2 v) { Yt[(unsigned)(k * R) * ub + c] = v; };
  const FourStepTw<+1> pt{loN, hiN, sN, twQ, Q, r, 0};
  if constexpr (TST) {
    auto st3 = [&](int k, int c, double2 v) { sm[(k << 3) + c] = v; };
    hyb_tile_fft_from<NC, +1, TrB, hyb_mask<TrB>(false, true), 1, 2, decltype(st3), FourStepTw<+1>, CtaSync, true>(
        sm, st3, twC, pt);
    fence_proxy_async();
    __syncthreads();
    if (threadIdx.x == 0) {
      constexpr int BOX = NC < 256 ? NC : 256;
#pragma unroll
      for (int k0 = 0; k0 < NC; k0 += BOX) tma_store_3d(tmY, (int)(2 * b0), r, k0, sm + k0 * kSig);
      tma_store_commit();
      tma_store_wait_read();
    }
  } else if constexpr (kLead2) {
    hyb_tile_fft_from<NC, +1, TrB, hyb_mask<TrB>(false, true), 1, 2>(sm, st2, twC, pt);
  } else {
    auto ld2 = [&](int i, int c) -> double2 { return sm[hidx(i, c)]; };
    hyb_tile_fft<NC, +1, TrB, hyb_mask<TrB>(false, true), true, false>(sm, ld2, st2, twC, pt);
  }
}

template <int R, int C, bool XOUT>
__global__ void __launch_bounds__(fast_threads<2 * C, kSig>(), bm_minb(fast_threads<2 * C, kSig>())) kbm_pad_h(
    const double2* __restrict__ Z, double2* __restrict__ Y, int64_t Bp, const double2* __restrict__ twR,
    const double2* __restrict__ twC, const double2* __restrict__ loN, const double2* __restrict__ hiN, int sN,
    const double2* __restrict__ twQ, int Q, const double* __restrict__ coef, const double* __restrict__ deconv,
    const double* __restrict__ cd, const double2* __restrict__ xsub, double2* __restrict__ xout) {
  extern __shared__ double2 sm[];
  pad_h_body<R, C, XOUT, false>(sm, nullptr, Z, Y, Bp, twR, twC, loN, hiN, sN, twQ, Q, coef, deconv, cd, xsub, xout);
}
template <int R, int C, bool XOUT>
__global__ void __launch_bounds__(fast_threads<2 * C, kSig>(), bm_minb(fast_threads<2 * C, kSig>())) kbm_pad_hst(
    const __grid_constant__ CUtensorMap tmY, const double2* __restrict__ Z, double2* __restrict__ Y, int64_t Bp,
    const double2* __restrict__ twR, const double2* __restrict__ twC, const double2* __restrict__ loN,
    const double2* __restrict__ hiN, int sN, const double2* __restrict__ twQ, int Q, const double* __restrict__ coef,
    const double* __restrict__ deconv, const double* __restrict__ cd, const double2* __restrict__ xsub,
    double2* __restrict__ xout) {
  extern __shared__ __align__(128) double2 sm_hs[];
  if constexpr (FastTraits<2 * C>::radix(0) == 2)
    pad_h_body<R, C, XOUT, true>(sm_hs, &tmY, Z, Y, Bp, twR, twC, loN, hiN, sN, twQ, Q, coef, deconv, cd, xsub, xout);
}

// First-pass hook of the TMA-staged kernels: wait for the cp.async table
// copies before the barrier; after it (every thread has read the tile) thread
// 0 refills the buffer with the CTA's next tile of ROWS rows.
template <int ROWS, int SG, bool OPQ = false>
struct TmaNextTile {
  static constexpr bool kActive = true;
  static constexpr bool kOpaque = OPQ;
  const CUtensorMap* map;
  double2* dst;
  uint64_t* bar;
  int tn, ntiles, groups;
  int tid;  // thread index within the CTA (or the CTA's tile group)
  __device__ __forceinline__ void operator()() const { asm volatile("cp.async.wait_all;\n" ::); }
  __device__ __forceinline__ void after() const {
    if (tid == 0 && tn < ntiles) {
      fence_proxy_async();  // the first pass's generic reads of the buffer precede the async refill
      mbar_expect_tx(bar, (unsigned)(ROWS * SG * sizeof(double2)));
      tma_load_2d(dst, map, 2 * SG * (tn % groups), ROWS * (tn / groups), bar);
    }
  }
};

// kbm_pad with a TMA-staged input tile: the tile's Z rows (C rows x 8
// signals, 32 KB at C = 256) are brought into shared memory by ONE
// cp.async.bulk.tensor issued by thread 0 (SASS UTMALDG, mbarrier
// transaction count) instead of 16 LDGs per thread into registers; the
// per-tile tables are staged with cp.async meanwhile.  Tile order as the
// one-shot kernels (signal groups fastest).  Arithmetic and store order are
// those of kbm_pad (bitwise identical results).
//
// A persistent variant that refills the buffer with the CTA's next tile
// right after the first pass (so its DRAM latency hides under the current
// tile) is possible with the TmaNextTile hook, but nvcc then spills
// 1.2 KB/thread at the 128-register budget (the second tile's FFT keeps
// values of the first live: measured with a runtime loop, `#pragma unroll 1`,
// a two-tile unroll, laundered pointers and thread indices alike), so each
// CTA handles one tile.
struct PadTileArgs {
  double2* Y;
  int64_t Bp;
  const double2 *twR, *twC, *loN, *hiN;
  int sN;
  const double2* twQ;
  int Q;
  const double *coef, *deconv, *cd;
  double2* xout;
  int ntiles, groups;
};

template <int R, int C, int SG, bool OPQ = false, class Sy = CtaSync>
__device__ __forceinline__ void pad_tile(const PadTileArgs& a, const CUtensorMap* tmZ, double2* sm, double2* inb,
                                      uint64_t* bar, int t, int tn, const Sy& sy = Sy()) {
  constexpr int NC = 2 * C;
  constexpr bool kLead2 = FastTraits<NC>::radix(0) == 2;
  double* s_t0 = reinterpret_cast<double*>(reinterpret_cast<char*>(sm) + fast_smem<NC, SG>());
  double* s_t1 = s_t0 + C;
  const int r = t / a.groups;
  const int64_t b0 = (int64_t)(t % a.groups) * SG;
  const unsigned ub = (unsigned)a.Bp;
  double2* __restrict__ Yt = a.Y + (int64_t)r * a.Bp + b0;
  double2* __restrict__ Xt = a.xout ? a.xout + (int64_t)r * a.Bp + b0 : nullptr;
  const bool xo = a.xout != nullptr;
  int tid0 = sy.tid();
  asm volatile("" : "+r"(tid0));
  for (int k2 = tid0; k2 < C; k2 += fast_threads<NC, SG>()) {
    const int64_t p = (int64_t)r + (int64_t)R * k2;
    if (xo) {
      cpa8(&s_t0[k2], &a.coef[p]);
      cpa8(&s_t1[k2], &a.deconv[p]);
    } else {
      cpa8(&s_t0[k2], &a.cd[p]);
    }
  }
  cpa_commit();
  const TmaNextTile<C, SG, OPQ> hook{tmZ, inb, bar, tn, a.ntiles, a.groups, sy.tid()};  // refill with tile tn
  auto ld1 = [&](int i, int c) -> double2 { return inb[i * SG + c]; };
  auto st1 = [&](int k2, int c, double2 v) {
    if (xo) {
      v = rsc(v, s_t0[k2]);
      Xt[(unsigned)(R * k2) * ub + c] = v;
      v = rsc(v, s_t1[k2]);
    } else {
      v = rsc(v, s_t0[k2]);
    }
    const int n1 = (k2 - C / 2) & (NC - 1);
    if constexpr (kLead2) {
      if (n1 < C) {
        sm[sidx<NC, SG, true>(2 * n1, c)] = v;
        sm[sidx<NC, SG, true>(2 * n1 + 1, c)] = v;
      } else {
        const int j = n1 - C;
        sm[sidx<NC, SG, true>(2 * j, c)] = v;
        sm[sidx<NC, SG, true>(2 * j + 1, c)] = make_double2(-v.x, -v.y);
      }
    } else {
      sm[sidx<NC, SG, true>(n1, c)] = v;
      sm[sidx<NC, SG, true>((n1 + C) & (NC - 1), c)] = make_double2(0.0, 0.0);
    }
  };
  fast_tile_fft<C, SG, -1, true, HalfTr<C>>(sm, ld1, st1, a.twR, NoPostTw(), hook, sy);
  sy.sync();
  auto st2 = [&](int k, int c, double2 v) { Yt[(unsigned)(k * R) * ub + c] = v; };
  const FourStepTw<+1> pt{a.loN, a.hiN, a.sN, a.twQ, a.Q, r, 0};
  if constexpr (kLead2) {
    fast_tile_fft_from<NC, SG, +1, true, 1, 2>(sm, st2, a.twC, pt, NoHookT<OPQ>(), sy);
  } else {
    auto ld2 = [&](int i, int c) -> double2 { return sm[sidx<NC, SG, true>(i, c)]; };
    fast_tile_fft_smem<NC, SG, +1, true>(sm, ld2, st2, a.twC, pt, NoHookT<OPQ>(), sy);
  }
}

template <int R, int C, int SG>
__global__ void __launch_bounds__(fast_threads<2 * C, SG>(), bm_minb(fast_threads<2 * C, SG>())) kbm_pad_t(
    const __grid_constant__ CUtensorMap tmZ, const __grid_constant__ PadTileArgs a) {
  constexpr int NC = 2 * C;
  constexpr unsigned kTileBytes = (unsigned)(C * SG * sizeof(double2));
  extern __shared__ __align__(128) unsigned char smraw_t[];
  double2* sm = reinterpret_cast<double2*>(smraw_t);
  double* s_t1 = reinterpret_cast<double*>(smraw_t + fast_smem<NC, SG>()) + C;
  double2* inb = reinterpret_cast<double2*>(
      (reinterpret_cast<uintptr_t>(s_t1 + C) + 127) & ~uintptr_t(127));  // [C][SG] dense (TMA box)
  uint64_t* bar = reinterpret_cast<uint64_t*>(inb + C * SG);
  int t = blockIdx.x;
  if (threadIdx.x == 0) {
    tma_prefetch_desc(&tmZ);
    mbar_init(bar, 1);
    mbar_fence_init();
  }
  __syncthreads();
  pdl_enter();  // programmatic dependent launch: Z is the producer's output
  if (threadIdx.x == 0 && t < a.ntiles) {
    mbar_expect_tx(bar, kTileBytes);
    tma_load_2d(inb, &tmZ, 2 * SG * (t % a.groups), C * (t / a.groups), bar);
  }
  if (t < a.ntiles) {
    mbar_wait(bar, 0);
    pad_tile<R, C, SG>(a, &tmZ, sm, inb, bar, t, a.ntiles);  // no refill (one tile per CTA)
  }
}

// row pass: row r = blockIdx.x (length L), output index r + R1 k.
template <int L, int S>
__global__ void __launch_bounds__(fast_threads<L, kSig>(), bm_minb(fast_threads<L, kSig>())) kbm_row(const double2* __restrict__ in,
                                                                  double2* __restrict__ out, int64_t Bp, int64_t R1,
                                                                  const double2* __restrict__ tw, int sw, int pf) {
  pdl_enter();  // programmatic dependent launch: wait for the producer grid
  extern __shared__ double2 sm[];
  const int r = sw ? blockIdx.y : blockIdx.x;
  const int64_t b0 = (int64_t)(sw ? blockIdx.x : blockIdx.y) * kSig;
  {
    unsigned ax, ay;
    if (ahead_block(pf, ax, ay))
      pf_rows(in + (int64_t)(sw ? ay : ax) * L * Bp + (int64_t)(sw ? ax : ay) * kSig, Bp, L, kSig * sizeof(double2));
  }
  auto ld = [&](int i, int c) -> double2 { return in[((int64_t)r * L + i) * Bp + b0 + c]; };
  auto st = [&](int k, int c, double2 v) { out[((int64_t)r + R1 * k) * Bp + b0 + c] = v; };
  fast_tile_fft<L, kSig, S, true>(sm, ld, st, tw);
}

// kbm_row on the unpadded swizzled tile with the output through the TMA unit (see kbm_col_s).
template <int L, int S>
__global__ void __launch_bounds__(fast_threads<L, kSig>(), bm_minb(fast_threads<L, kSig>())) kbm_row_s(
    const __grid_constant__ CUtensorMap tmO, const double2* __restrict__ in, int64_t Bp,
    const double2* __restrict__ tw) {
  pdl_enter();  // programmatic dependent launch: wait for the producer grid
  static_assert(L <= 256 && hyb_ok<L>(), "one TMA box, hybrid tile");
  extern __shared__ __align__(128) double2 sm_hs[];
  double2* sm = sm_hs;
  const int r = blockIdx.y;
  const int64_t b0 = (int64_t)blockIdx.x * kSig;
  const unsigned ub = (unsigned)Bp;
  const double2* __restrict__ it = in + (int64_t)r * L * Bp + b0;
  auto ld = [&](int i, int c) -> double2 { return it[(unsigned)i * ub + c]; };
  auto st = [&](int k, int c, double2 v) { sm[(k << 3) + c] = v; };
  using Tr = FastTraits<L>;
  hyb_passes<L, S, 0, 1, Tr, 0x0u, false, false, 0, decltype(ld), decltype(st), NoPostTw, NoHook, Tr::np, CtaSync, true>(
      sm, ld, st, tw, NoPostTw(), NoHook());
  fence_proxy_async();
  __syncthreads();
  if (threadIdx.x == 0) {
    tma_store_3d(&tmO, (int)(2 * b0), r, 0, sm);
    tma_store_commit();
    tma_store_wait_read();
  }
}

// Boundary, type-4 input: signal-major A[b][P] -> column IFFT_P (length C,
// columns k = RW blockIdx.x + (c % RW) of the p = k + R m layout, signals
// b = 4 blockIdx.y + c / RW) * decay -> batch-minor U; optionally also a
// batch-minor copy AT of A.
template <int R, int C, int RW>
__global__ void __launch_bounds__(fast_threads<C, 4 * RW>(), bm_minb(fast_threads<C, 4 * RW>())) kbm_colin(
    const double2* __restrict__ A, int64_t batch, double2* __restrict__ U, int64_t Bp, const double2* __restrict__ tw,
    const double2* __restrict__ loP, const double2* __restrict__ hiP, int sP, const double2* __restrict__ twQ, int Q,
    const double* __restrict__ decay, double2* __restrict__ AT, int sw) {
  pdl_enter();  // programmatic dependent launch: wait for the producer grid
  constexpr int64_t P = (int64_t)R * C;
  extern __shared__ double2 sm[];
  const int m20 = (sw ? blockIdx.y : blockIdx.x) * RW;
  const int64_t bb = (int64_t)(sw ? blockIdx.x : blockIdx.y) * 4;
  auto ld = [&](int i, int c) -> double2 {
    const int64_t idx = (int64_t)i * R + m20 + (c % RW);
    const int64_t b = bb + c / RW;
    double2 v = b < batch ? A[b * P + idx] : make_double2(0.0, 0.0);
    if (AT) AT[idx * Bp + b] = v;
    return rsc(v, __ldg(&decay[idx]));
  };
  auto st = [&](int k1, int c, double2 v) {
    U[((int64_t)k1 * R + m20 + (c % RW)) * Bp + bb + c / RW] = v;
  };
  const FourStepTw<+1> pt{loP, hiP, sP, twQ, Q, m20, RW - 1};
  fast_tile_fft<C, 4 * RW, +1, true>(sm, ld, st, tw, pt);
}

// Boundary, type-5 output: batch-minor Z rows r = RW blockIdx.x + (c % RW)
// (length C) -> row FFT_P * coef [xsub (batch-minor) - .] -> signal-major
// out[b][P] at p = r + R k.
template <int R, int C, int RW>
__global__ void __launch_bounds__(fast_threads<C, 4 * RW>(), bm_minb(fast_threads<C, 4 * RW>())) kbm_rowout(
    const double2* __restrict__ Z, double2* __restrict__ out, int64_t batch, int64_t Bp,
    const double2* __restrict__ tw, const double* __restrict__ coef, const double2* __restrict__ xsub, int sw) {
  pdl_enter();  // programmatic dependent launch: wait for the producer grid
  constexpr int64_t P = (int64_t)R * C;
  extern __shared__ double2 sm[];
  const int r0 = (sw ? blockIdx.y : blockIdx.x) * RW;
  const int64_t bb = (int64_t)(sw ? blockIdx.x : blockIdx.y) * 4;
  auto ld = [&](int i, int c) -> double2 {
    return Z[((int64_t)(r0 + (c % RW)) * C + i) * Bp + bb + c / RW];
  };
  auto st = [&](int k, int c, double2 v) {
    const int64_t p = (int64_t)(r0 + (c % RW)) + (int64_t)R * k;
    const int64_t b = bb + c / RW;
    v = rsc(v, __ldg(&coef[p]));
    if (xsub) v = csub(xsub[p * Bp + b], v);
    if (b < batch) out[b * P + p] = v;
  };
  fast_tile_fft<C, 4 * RW, -1, true>(sm, ld, st, tw);
}

// ------------------------------------------------------------------------
// Batched FORWARD transforms (nfft_type1 / nfft_type2 with R = P = Q, forward.py:26-102) on
// the batch-minor passes: the user's signal-major operand meets the batch-minor grid in ONE
// boundary kernel per direction, on 2-D tiles of KK adjacent indices x 8 / KK signals of length
// 2C (KK = 2: 32-byte runs on the signal-major side, 64-byte runs on the batch-minor side).
//
// deconvolution weights of the band p < P of the n = 2P grid (gridding.py:90), once per call
static __global__ void k_fwd_deconv(double* __restrict__ d, int64_t P, double wb) {
  const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (p < P) d[p] = deconv_weight(p, P / 2, 2 * P, wb);
}

// Launch order (1-D grid): W index blocks x all G signal groups, then the next W index blocks.
// The ~150 resident CTAs then cover W x 64 bytes of every signal-major row AND ~150 / W x 64
// bytes of every batch-minor row (index blocks fastest alone leaves the batch-minor side with
// isolated 64-byte runs, signal groups fastest alone the signal-major side).
__device__ __forceinline__ void fwd_block(int W, int G, int& kb, int& sg) {
  const unsigned L = blockIdx.x;
  const unsigned per = (unsigned)W * (unsigned)G;
  kb = (int)((L / per) * W + L % W);
  sg = (int)((L % per) / W);
}

// type-2 front: S[b][p] (signal-major) * deconv(p) -> zero-padded column IFFT_2P (columns
// k = KK kb + c % KK of the n = R x 2C layout: input position (m1 - C/2) mod 2C holds
// p = k + R m1, m1 < C) -> W_n^{+k n2} -> Y[(n2 R + k)][b]; kbm_row + the gather finish it.
// 8-column tiles (KK indices x 8 / KK signals, 256 threads for 2C = 512, two CTAs per SM) on
// the hybrid schedule: the passes between the global-memory ones are warp-local (hyb_passes),
// 2 CTA barriers per tile (a 16-column, 512-thread tile with a barrier per pass measured
// 1.43 ms for this kernel at C4 size against 1.00 ms, 1.04 against 0.80 ms for kbm_fwd_out_h).
template <int R, int C, int KK>
__global__ void __launch_bounds__(fast_threads<2 * C, kSig>(), bm_minb(fast_threads<2 * C, kSig>())) kbm_fwd_in_h(
    const double2* __restrict__ S, int64_t batch, double2* __restrict__ Y, int64_t Bp, const double2* __restrict__ tw,
    const double2* __restrict__ loN, const double2* __restrict__ hiN, int sN, const double2* __restrict__ twQ, int Q,
    const double* __restrict__ deconv, int W, int G) {
  pdl_enter();  // programmatic dependent launch: wait for the producer grid
  constexpr int64_t P = (int64_t)R * C;
  constexpr int NC = 2 * C;
  constexpr int BB = 8 / KK;
  using Tr = FastTraits<NC>;
  extern __shared__ double2 sm[];
  int kb, sg;
  fwd_block(W, G, kb, sg);
  const int k0 = kb * KK;
  const int64_t bb = (int64_t)sg * BB;
  auto ld = [&](int i, int c) -> double2 {
    const int m1 = (i + C / 2) & (NC - 1);
    const int64_t b = bb + c / KK;
    if (m1 >= C || b >= batch) return make_double2(0.0, 0.0);
    const int64_t p = (int64_t)(k0 + (c % KK)) + (int64_t)R * m1;
    return rsc(S[b * P + p], __ldg(&deconv[p]));
  };
  auto st = [&](int n2, int c, double2 v) { Y[((int64_t)n2 * R + k0 + (c % KK)) * Bp + bb + c / KK] = v; };
  const FourStepTw<+1> pt{loN, hiN, sN, twQ, Q, k0, KK - 1};
  hyb_tile_fft<NC, +1, Tr, hyb_mask<Tr>(true, true), false, false>(sm, ld, st, tw, pt);
}

// type-1 back: rows k1 = KK kb + c % KK of the column pass's output T[(k1 2C + n2)][b]
// -> row FFT_2P -> band m1 = (k2 + C/2) mod 2C < C -> * deconv(p), p = k1 + R m1 [- sub]
// -> out[b][p] (signal-major).
template <int R, int C, int KK>
__global__ void __launch_bounds__(fast_threads<2 * C, kSig>(), bm_minb(fast_threads<2 * C, kSig>())) kbm_fwd_out_h(
    const double2* __restrict__ T, double2* __restrict__ out, int64_t batch, int64_t Bp, const double2* __restrict__ tw,
    const double2* __restrict__ sub, const double* __restrict__ deconv, int W, int G) {
  pdl_enter();  // programmatic dependent launch: wait for the producer grid
  constexpr int64_t P = (int64_t)R * C;
  constexpr int NC = 2 * C;
  constexpr int BB = 8 / KK;
  using Tr = FastTraits<NC>;
  extern __shared__ double2 sm[];
  int kb, sg;
  fwd_block(W, G, kb, sg);
  const int k0 = kb * KK;
  const int64_t bb = (int64_t)sg * BB;
  auto ld = [&](int i, int c) -> double2 { return T[((int64_t)(k0 + (c % KK)) * NC + i) * Bp + bb + c / KK]; };
  auto st = [&](int k2, int c, double2 v) {
    const int m1 = (k2 + C / 2) & (NC - 1);
    const int64_t b = bb + c / KK;
    if (m1 >= C || b >= batch) return;
    const int64_t p = (int64_t)(k0 + (c % KK)) + (int64_t)R * m1;
    v = rsc(v, __ldg(&deconv[p]));
    if (sub) v = csub(v, sub[b * P + p]);
    out[b * P + p] = v;
  };
  hyb_tile_fft<NC, -1, Tr, hyb_mask<Tr>(true, true), false, false>(sm, ld, st, tw);
}

// Kernel-only build for register / SASS experiments:
//   nvcc ... -DNFFT45_EXP_ONLY -Xptxas -v -c csrc/chain_bm.cu
#ifdef NFFT45_EXP_ONLY
#define NFFT45_EXP_RC 256, 256
template __global__ void kbm_band_h<NFFT45_EXP_RC>(const double2*, double2*, int64_t, const double2*, const double2*, const double2*,
                                              const double2*, int, const double2*, int, const double*, const double*,
                                              const double*, const double2*, double2*);
template __global__ void kbm_mid_h<NFFT45_EXP_RC>(const double2*, double2*, int64_t, const double2*, const double2*, const double2*,
                                             int, const double2*, int, const double2*);
template __global__ void kbm_band_hf<NFFT45_EXP_RC>(const double2*, double2*, int64_t, const double2*, const double2*, const double2*,
                                               const double2*, int, const double2*, int, const double*, const double*,
                                               const double*, const double2*, double2*);
template __global__ void kbm_mid_hf<NFFT45_EXP_RC>(const double2*, double2*, int64_t, const double2*, const double2*, const double2*,
                                              int, const double2*, int, const double2*);
template __global__ void kbm_pad_hf<NFFT45_EXP_RC>(const double2*, const __grid_constant__ PadHfArgs);
template __global__ void kbm_pad_hs<NFFT45_EXP_RC>(const double2*, const __grid_constant__ CUtensorMap,
                                              const __grid_constant__ PadHfArgs);
template __global__ void kbm_pad_hp<NFFT45_EXP_RC>(const __grid_constant__ CUtensorMap, const __grid_constant__ PadHfArgs);
template __global__ void kbm_pad_h<NFFT45_EXP_RC, false>(const double2*, double2*, int64_t, const double2*, const double2*,
                                                    const double2*, const double2*, int, const double2*, int,
                                                    const double*, const double*, const double*, const double2*, double2*);
template __global__ void kbm_pad_h<NFFT45_EXP_RC, true>(const double2*, double2*, int64_t, const double2*, const double2*,
                                                   const double2*, const double2*, int, const double2*, int,
                                                   const double*, const double*, const double*, const double2*, double2*);
#else
// ------------------------------------------------------------ host side

#if NFFT45_BM_PART != 2
using TmaEncode = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                 const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                 CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static TmaEncode tma_encoder() {
  static TmaEncode encode = [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      fn = nullptr;
    return reinterpret_cast<TmaEncode>(fn);
  }();
  if (!encode) set_error(NFFT45_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  return encode;
}

int tma_map_strided(CUtensorMap* map, const void* base, int64_t outer_n, int64_t inner_n, int64_t Bp, int box_outer,
                    int box_sig) {
  TmaEncode encode = tma_encoder();
  if (!encode) return NFFT45_ERR_CUDA;
  const cuuint64_t gdim[3] = {(cuuint64_t)(2 * Bp), (cuuint64_t)inner_n, (cuuint64_t)outer_n};
  const cuuint64_t gstride[2] = {(cuuint64_t)(Bp * sizeof(double2)), (cuuint64_t)(inner_n * Bp * sizeof(double2))};
  const cuuint32_t box[3] = {(cuuint32_t)(2 * box_sig), 1u, (cuuint32_t)box_outer};
  const cuuint32_t estride[3] = {1, 1, 1};
  CUresult r = encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<void*>(base), gdim, gstride, box, estride,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error(NFFT45_ERR_CUDA, "cuTensorMapEncodeTiled (3-D) failed (" + std::to_string((int)r) + ")");
    return NFFT45_ERR_CUDA;
  }
  return NFFT45_OK;
}

int tma_map_rows(CUtensorMap* map, const void* base, int64_t rows, int64_t Bp, int box_rows, int box_sig) {
  TmaEncode encode = tma_encoder();
  if (!encode) return NFFT45_ERR_CUDA;
  const cuuint64_t gdim[2] = {(cuuint64_t)(2 * Bp), (cuuint64_t)rows};
  const cuuint64_t gstride[1] = {(cuuint64_t)(Bp * sizeof(double2))};
  const cuuint32_t box[2] = {(cuuint32_t)(2 * box_sig), (cuuint32_t)box_rows};
  const cuuint32_t estride[2] = {1, 1};
  CUresult r = encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<void*>(base), gdim, gstride, box, estride,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error(NFFT45_ERR_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
    return NFFT45_ERR_CUDA;
  }
  return NFFT45_OK;
}

#endif  // NFFT45_BM_PART != 2

template <typename K>
static int bm_attr(K kernel, size_t bytes) {
  if (bytes > 48 * 1024) NFFT_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
  return NFFT45_OK;
}

struct BmTabs {
  const double2 *twR, *twC, *tw2C;  // tile twiddles for lengths R, C, 2C
  const FftTables *tP, *tN;
};

template <int R, int C>
struct ChainBM {
  static constexpr int64_t P = (int64_t)R * C, n = 2 * P;
  static constexpr int SG = bm_sg<C>();
  BmTabs t;
  int64_t Bp, batch;
  unsigned groups;  // Bp / 8
  cudaStream_t st;
  bool small_tiles = false;  // 4-signal tiles for the two-FFT kernels (A/B experiment)
  bool sw = false;           // grid order: signal groups fastest (blockIdx.x) instead of tile index
  int pf = 0;                // L2 prefetch distance in launch slots (0: off)
  bool hyb = false;          // hybrid two-FFT kernels (warp-local middle passes), when bm_hyb<R, C>()
  bool fuse = true;          // register handoff between the two transforms of band / mid (NFFT45_FUSE=0: off)
  // FFT_2P / IFFT_2P passes on the hybrid tile with TMA-stored output: bit 0 column pass, bit 1 row
  // pass (NFFT45_PASS_TMAST; A/B and the variant test)
  static int pass_tma() {
    static const int on = getenv("NFFT45_PASS_TMAST") ? atoi(getenv("NFFT45_PASS_TMAST")) : 1;
    return on;
  }
  // outputs of the fused hybrid kernels through bulk tensor stores: 1 (default) pad and mid, 2 also
  // band, 0 off (NFFT45_TMAST; A/B and the variant test)
  static int tma_st() {
    static const int on = getenv("NFFT45_TMAST") ? atoi(getenv("NFFT45_TMAST")) : 1;
    return on;
  }
  // grid of (tiles x groups*mult); with sw the signal groups run fastest
  dim3 gdim(int tiles, int mult = 1) const {
    return sw ? dim3(groups * mult, (unsigned)tiles) : dim3((unsigned)tiles, groups * mult);
  }

  int qtab(int64_t Q, const double2** out) {
    int status = NFFT45_OK;
    const FftTables* tq = fft_tables(Q, st, &status);
    if (!tq) return status;
    *out = tq->tw;
    return NFFT45_OK;
  }

  // FFT_2P column pass: R-point columns over the 2C columns of H
  int col(const double2* in, double2* out, int perm = 0) {
    auto bm_col = kbm_col<R, -1>;
    constexpr size_t smem = fast_smem<R, kSig>();
    NFFT_CHECK(bm_attr(bm_col, smem));
    constexpr int T = fast_threads<R, kSig>();
    const int64_t Q = n / last_stride<R>();
    const double2* twQ = nullptr;
    NFFT_CHECK(qtab(Q, &twQ));
    if constexpr (R <= 512 && hyb_ok<R>()) {
      if ((pass_tma() & 1) && sw && pf == 0) {  // signal groups fastest (the default order), output through the TMA unit
        auto bm_col = kbm_col_s<R, -1>;
        constexpr size_t smem_s = sizeof(double2) * R * kSig;
        NFFT_CHECK(bm_attr(bm_col, smem_s));
        CUtensorMap tm;
        NFFT_CHECK(tma_map_strided(&tm, out, R, 2 * C, Bp, R < 256 ? R : 256, kSig));
        LAUNCH_PDL(bm_col, dim3(groups, (unsigned)(2 * C)), T, smem_s, st, tm, in, 2 * C, Bp, t.twR, t.tN->lo, t.tN->hi,
                   t.tN->s, twQ, (int)Q, perm);
        return NFFT45_OK;
      }
    }
    LAUNCH_PDL(bm_col, gdim(2 * C), T, smem, st, in, out, 2 * C, Bp, t.twR, t.tN->lo, t.tN->hi, t.tN->s, twQ, (int)Q,
           nullptr, (int)sw, pf, perm);
    return NFFT45_OK;
  }

  template <int G>
  int band_g(const double2* T_, double2* U, const ChainPlanView& pv, const double2* sub, double2* rsave) {
    auto bm_band = kbm_band<R, C, G>;
    const size_t smem = fast_smem<2 * C, G>() + 2 * sizeof(double) * C + (sub ? sizeof(double2) * C * G : 0);
    NFFT_CHECK(bm_attr(bm_band, smem));
    constexpr int T = fast_threads<2 * C, G>();
    const int64_t Q = P / last_stride<C, HalfTr<C>>();  // the column IFFT_P runs the HalfTr schedule
    const double2* twQ = nullptr;
    NFFT_CHECK(qtab(Q, &twQ));
    LAUNCH_PDL(bm_band, gdim(R, kSig / G), T, smem, st, T_, U, Bp, t.tw2C, t.twC, t.tP->lo, t.tP->hi, t.tP->s, twQ,
           (int)Q, pv.deconv, pv.decay, pv.dd, sub, (int)sw, pf, rsave);
    return NFFT45_OK;
  }
  int band_h(const double2* T_, double2* U, const ChainPlanView& pv, const double2* sub, double2* rsave) {
    if constexpr (bm_hyb<R, C>()) {
      auto bm_band = kbm_band_h<R, C>;
      if constexpr (bm_band_fused<R, C>())
        if (fuse) bm_band = kbm_band_hf<R, C>;  // band handoff in registers
      const size_t smem = sizeof(double2) * 2 * C * kSig + 2 * sizeof(double) * C + (sub ? sizeof(double2) * C * kSig : 0);
      NFFT_CHECK(bm_attr(bm_band, smem));
      constexpr int T = fast_threads<2 * C, kSig>();
      const int64_t Q = P / last_stride<C, HalfTr<C>>();
      const double2* twQ = nullptr;
      NFFT_CHECK(qtab(Q, &twQ));
      if constexpr (bm_band_fused<R, C>()) {
        if (fuse && tma_st() >= 2) {  // output through a bulk tensor store (measured neutral: opt-in)
          auto bm_band = kbm_band_hs<R, C>;
          NFFT_CHECK(bm_attr(bm_band, smem));
          CUtensorMap tm;
          NFFT_CHECK(tma_map_strided(&tm, U, C, R, Bp, C, kSig));
          LAUNCH_PDL(bm_band, dim3(groups, (unsigned)R), T, smem, st, tm, T_, U, Bp, t.tw2C, t.twC, t.tP->lo, t.tP->hi,
                     t.tP->s, twQ, (int)Q, pv.tdeconv, pv.tdecay, pv.tdd, sub, rsave);
          return NFFT45_OK;
        }
      }
      LAUNCH_PDL(bm_band, dim3(groups, (unsigned)R), T, smem, st, T_, U, Bp, t.tw2C, t.twC, t.tP->lo, t.tP->hi, t.tP->s,
                 twQ, (int)Q, pv.tdeconv, pv.tdecay, pv.tdd, sub, rsave);
    }
    return NFFT45_OK;
  }
  int band(const double2* T_, double2* U, const ChainPlanView& pv, const double2* sub, double2* rsave = nullptr) {
    if (hyb && !small_tiles) return band_h(T_, U, pv, sub, rsave);
    if (small_tiles || SG < kSig) return band_g<kSig / 2>(T_, U, pv, sub, rsave);  // always for C = 1024
    return band_g<kSig>(T_, U, pv, sub, rsave);
  }

  int mid_h(const double2* U, double2* Z, const ChainPlanView& pv) {
    if constexpr (bm_hyb<R, C>()) {
      auto bm_mid = kbm_mid_h<R, C>;
      if constexpr (bm_mid_fused<R, C>())
        if (fuse) bm_mid = kbm_mid_hf<R, C>;  // IFFT -> ks -> FFT handoff in registers
      constexpr size_t smem = sizeof(double2) * R * kSig + sizeof(double2) * R;
      NFFT_CHECK(bm_attr(bm_mid, smem));
      constexpr int T = fast_threads<R, kSig>();
      const int64_t Q = P / last_stride<R>();
      const double2* twQ = nullptr;
      NFFT_CHECK(qtab(Q, &twQ));
      if constexpr (bm_mid_fused<R, C>() && R <= 256) {
        if (fuse && tma_st()) {
          auto bm_mid = kbm_mid_hs<R, C>;
          NFFT_CHECK(bm_attr(bm_mid, smem));
          CUtensorMap tm;
          NFFT_CHECK(tma_map_strided(&tm, Z, R, C, Bp, R, kSig));
          LAUNCH_PDL(bm_mid, dim3(groups, (unsigned)C), T, smem, st, tm, U, Z, Bp, t.twR, t.tP->lo, t.tP->hi, t.tP->s,
                     twQ, (int)Q, pv.tks);
          return NFFT45_OK;
        }
      }
      LAUNCH_PDL(bm_mid, dim3(groups, (unsigned)C), T, smem, st, U, Z, Bp, t.twR, t.tP->lo, t.tP->hi, t.tP->s, twQ, (int)Q,
                 pv.tks);
    }
    return NFFT45_OK;
  }
  int mid(const double2* U, double2* Z, const ChainPlanView& pv) {
    if (hyb) return mid_h(U, Z, pv);
    auto bm_mid = kbm_mid<R, C>;
    constexpr size_t smem = fast_smem<R, kSig>() + sizeof(double2) * R;
    NFFT_CHECK(bm_attr(bm_mid, smem));
    constexpr int T = fast_threads<R, kSig>();
    const int64_t Q = P / last_stride<R>();
    const double2* twQ = nullptr;
    NFFT_CHECK(qtab(Q, &twQ));
    LAUNCH_PDL(bm_mid, gdim(C), T, smem, st, U, Z, Bp, t.twR, t.tP->lo, t.tP->hi, t.tP->s, twQ, (int)Q, pv.ks, (int)sw, pf);
    return NFFT45_OK;
  }

  template <int G>
  int pad_g(const double2* Z, double2* Y, const ChainPlanView& pv, const double2* xsub, double2* xout) {
    auto bm_pad = kbm_pad<R, C, G>;
    const size_t smem =
        fast_smem<2 * C, G>() + 2 * sizeof(double) * C + (xout && xsub ? sizeof(double2) * C * G : 0);
    NFFT_CHECK(bm_attr(bm_pad, smem));
    constexpr int T = fast_threads<2 * C, G>();
    const int64_t Q = n / last_stride<2 * C>();
    const double2* twQ = nullptr;
    NFFT_CHECK(qtab(Q, &twQ));
    LAUNCH_PDL(bm_pad, gdim(R, kSig / G), T, smem, st, Z, Y, Bp, t.twC, t.tw2C, t.tN->lo, t.tN->hi, t.tN->s, twQ,
           (int)Q, pv.coef, pv.deconv, pv.cd, xsub, xout, (int)sw, pf);
    return NFFT45_OK;
  }
  // TMA-staged pad (C <= 256 with 8-signal tiles, no subtrahend tile: two
  // CTAs per SM fit).  Opt-in (NFFT45_TMA=1): bitwise identical to kbm_pad
  // but measured 1.5-2 % slower on the C4 step (bm_pad 3.82 -> 3.88 ms per
  // step): one CTA per tile still waits for its own tile, and the persistent
  // form that would hide that wait spills (see kbm_pad_t).
  int pad_tma(const double2* Z, double2* Y, const ChainPlanView& pv, double2* xout) {
    auto bm_pad = kbm_pad_t<R, C, kSig>;
    const size_t smem = fast_smem<2 * C, kSig>() + 2 * sizeof(double) * C + 128 + sizeof(double2) * C * kSig + 16;
    NFFT_CHECK(bm_attr(bm_pad, smem));
    constexpr int T = fast_threads<2 * C, kSig>();
    const int64_t Q = n / last_stride<2 * C>();
    const double2* twQ = nullptr;
    NFFT_CHECK(qtab(Q, &twQ));
    CUtensorMap tm;
    NFFT_CHECK(tma_map_rows(&tm, Z, P, Bp, C, kSig));
    const int ntiles = (int)(R * groups);
    static const int sms = [] {
      int dev = 0, v = 148;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
      return v;
    }();
    const int grid = ntiles;
    (void)sms;
    const PadTileArgs args{Y, Bp, t.twC, t.tw2C, t.tN->lo, t.tN->hi, t.tN->s, twQ, (int)Q,
                           pv.coef, pv.deconv, pv.cd, xout, ntiles, (int)groups};
    LAUNCH_PDL(bm_pad, grid, T, smem, st, tm, args);
    return NFFT45_OK;
  }
  template <bool XOUT>
  int pad_h(const double2* Z, double2* Y, const ChainPlanView& pv, const double2* xsub, double2* xout) {
    if constexpr (bm_pad_fused<R, C>() && !XOUT) {
      if (fuse) {  // zero-padding handoff by warp shuffle
        constexpr int T = fast_threads<2 * C, kSig>();
        const int64_t Q = n / last_stride<2 * C>();
        const double2* twQ = nullptr;
        NFFT_CHECK(qtab(Q, &twQ));
        const int ntiles = (int)(R * groups);
        const PadHfArgs args{Y, Bp, t.twC, t.tw2C, t.tN->lo, t.tN->hi, t.tN->s, twQ, (int)Q, pv.tcd, ntiles, (int)groups};
        static const bool persist = getenv("NFFT45_PAD_PERSIST") != nullptr;
        if (persist) {  // one CTA per SM, two tile groups, TMA-prefetched tiles
          auto bm_pad = kbm_pad_hp<R, C>;
          constexpr size_t smem = PadHpLayout<R, C>::kBytes;
          NFFT_CHECK(bm_attr(bm_pad, smem));
          CUtensorMap tm;
          NFFT_CHECK(tma_map_rows(&tm, Z, P, Bp, C, kSig));
          static const int sms = [] {
            int dev = 0, v = 148;
            cudaGetDevice(&dev);
            cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
            return v;
          }();
          LAUNCH_PDL(bm_pad, std::min(sms, (ntiles + 1) / 2), 2 * T, smem, st, tm, args);
          return NFFT45_OK;
        }
        const size_t smem = sizeof(double2) * 2 * C * kSig + 2 * sizeof(double) * C;
        if (tma_st()) {  // output through bulk tensor stores
          auto bm_pad = kbm_pad_hs<R, C>;
          NFFT_CHECK(bm_attr(bm_pad, smem));
          CUtensorMap tm;
          NFFT_CHECK(tma_map_strided(&tm, Y, 2 * C, R, Bp, 256, kSig));
          LAUNCH_PDL(bm_pad, dim3(groups, (unsigned)R), T, smem, st, Z, tm, args);
          return NFFT45_OK;
        }
        auto bm_pad = kbm_pad_hf<R, C>;
        NFFT_CHECK(bm_attr(bm_pad, smem));
        LAUNCH_PDL(bm_pad, dim3(groups, (unsigned)R), T, smem, st, Z, args);
        return NFFT45_OK;
      }
    }
    if constexpr (bm_hyb<R, C>()) {
      auto bm_pad = kbm_pad_h<R, C, XOUT>;
      const size_t smem =
          sizeof(double2) * 2 * C * kSig + 2 * sizeof(double) * C + (XOUT && xsub ? sizeof(double2) * C * kSig : 0);
      NFFT_CHECK(bm_attr(bm_pad, smem));
      constexpr int T = fast_threads<2 * C, kSig>();
      const int64_t Q = n / last_stride<2 * C>();
      const double2* twQ = nullptr;
      NFFT_CHECK(qtab(Q, &twQ));
      if constexpr (FastTraits<2 * C>::radix(0) == 2) {
        if (tma_st()) {  // the padded grid through bulk tensor stores
          auto bm_pad = kbm_pad_hst<R, C, XOUT>;
          NFFT_CHECK(bm_attr(bm_pad, smem));
          CUtensorMap tm;
          NFFT_CHECK(tma_map_strided(&tm, Y, 2 * C, R, Bp, 2 * C < 256 ? 2 * C : 256, kSig));
          LAUNCH_PDL(bm_pad, dim3(groups, (unsigned)R), T, smem, st, tm, Z, Y, Bp, t.twC, t.tw2C, t.tN->lo, t.tN->hi,
                     t.tN->s, twQ, (int)Q, pv.tcoef, pv.tdeconv, pv.tcd, xsub, xout);
          return NFFT45_OK;
        }
      }
      LAUNCH_PDL(bm_pad, dim3(groups, (unsigned)R), T, smem, st, Z, Y, Bp, t.twC, t.tw2C, t.tN->lo, t.tN->hi, t.tN->s,
                 twQ, (int)Q, pv.tcoef, pv.tdeconv, pv.tcd, xsub, xout);
    }
    return NFFT45_OK;
  }
  int pad(const double2* Z, double2* Y, const ChainPlanView& pv, const double2* xsub, double2* xout) {
    static const bool tma = getenv("NFFT45_TMA") != nullptr;
    if (hyb && !small_tiles && !tma)
      return xout ? pad_h<true>(Z, Y, pv, xsub, xout) : pad_h<false>(Z, Y, pv, xsub, xout);
    if constexpr (C <= 256 && SG == kSig)
      if (tma && !small_tiles && !(xout && xsub)) return pad_tma(Z, Y, pv, xout);
    if (small_tiles || SG < kSig) return pad_g<kSig / 2>(Z, Y, pv, xsub, xout);  // always for C = 1024
    return pad_g<kSig>(Z, Y, pv, xsub, xout);
  }

  // IFFT_2P row pass: 2C rows of length R -> natural-order grid
  int row_grid(const double2* Y, double2* H) {
    auto bm_row = kbm_row<R, +1>;
    constexpr size_t smem = fast_smem<R, kSig>();
    NFFT_CHECK(bm_attr(bm_row, smem));
    constexpr int T = fast_threads<R, kSig>();
    if constexpr (R <= 256 && hyb_ok<R>()) {
      if ((pass_tma() & 2) && sw && pf == 0) {
        auto bm_row = kbm_row_s<R, +1>;
        constexpr size_t smem_s = sizeof(double2) * R * kSig;
        NFFT_CHECK(bm_attr(bm_row, smem_s));
        CUtensorMap tm;
        NFFT_CHECK(tma_map_strided(&tm, H, R, 2 * C, Bp, R, kSig));
        LAUNCH_PDL(bm_row, dim3(groups, (unsigned)(2 * C)), T, smem_s, st, tm, Y, Bp, t.twR);
        return NFFT45_OK;
      }
    }
    LAUNCH_PDL(bm_row, gdim(2 * C), T, smem, st, Y, H, Bp, (int64_t)(2 * C), t.twR, (int)sw, pf);
    return NFFT45_OK;
  }

  // forward type-2 front / type-1 back boundary kernels (KK indices x 8 / KK signals, length 2C)
  static int fwd_w(int nkb) {  // index blocks per launch-order group (a divisor of nkb; NFFT45_FWD_W for A/B runs)
    static const int env = getenv("NFFT45_FWD_W") ? atoi(getenv("NFFT45_FWD_W")) : 8;
    int w = env < 1 ? 1 : env;
    while (nkb % w) w--;
    return w;
  }
  template <int KK>
  int fwd_in_h(const double2* S, double2* Y, const double* deconv) {
    if constexpr (hyb_ok<2 * C>()) {
      auto bm_fwd_in = kbm_fwd_in_h<R, C, KK>;
      constexpr size_t smem = sizeof(double2) * 2 * C * kSig;
      NFFT_CHECK(bm_attr(bm_fwd_in, smem));
      constexpr int T = fast_threads<2 * C, kSig>();
      const int64_t Q = n / last_stride<2 * C>();
      const double2* twQ = nullptr;
      NFFT_CHECK(qtab(Q, &twQ));
      const int G = (int)ceil_div(Bp, 8 / KK);
      LAUNCH_PDL(bm_fwd_in, dim3((unsigned)((R / KK) * G)), T, smem, st, S, batch, Y, Bp, t.tw2C, t.tN->lo, t.tN->hi,
                 t.tN->s, twQ, (int)Q, deconv, fwd_w(R / KK), G);
    }
    return NFFT45_OK;
  }
  template <int KK>
  int fwd_out_h(const double2* T_, double2* out, const double2* sub, const double* deconv) {
    if constexpr (hyb_ok<2 * C>()) {
      auto bm_fwd_out = kbm_fwd_out_h<R, C, KK>;
      constexpr size_t smem = sizeof(double2) * 2 * C * kSig;
      NFFT_CHECK(bm_attr(bm_fwd_out, smem));
      constexpr int T = fast_threads<2 * C, kSig>();
      const int G = (int)ceil_div(Bp, 8 / KK);
      LAUNCH_PDL(bm_fwd_out, dim3((unsigned)((R / KK) * G)), T, smem, st, T_, out, batch, Bp, t.tw2C, sub, deconv,
                 fwd_w(R / KK), G);
    }
    return NFFT45_OK;
  }
  static int fwd_kk() {  // tile shape (NFFT45_FWD_KK = 2 | 4 for A/B runs)
    static const int kk = getenv("NFFT45_FWD_KK") ? atoi(getenv("NFFT45_FWD_KK")) : 2;
    return kk == 4 ? 4 : 2;
  }
  int fwd_in(const double2* S, double2* Y, const double* deconv) {
    return fwd_kk() == 2 ? fwd_in_h<2>(S, Y, deconv) : fwd_in_h<4>(S, Y, deconv);
  }
  int fwd_out(const double2* T_, double2* out, const double2* sub, const double* deconv) {
    return fwd_kk() == 2 ? fwd_out_h<2>(T_, out, sub, deconv) : fwd_out_h<4>(T_, out, sub, deconv);
  }

  int colin(const double2* A, double2* U, const ChainPlanView& pv, double2* AT) {
    constexpr int RW = bm_rw<C>();
    auto bm_colin = kbm_colin<R, C, RW>;
    constexpr size_t smem = fast_smem<C, 4 * RW>();
    NFFT_CHECK(bm_attr(bm_colin, smem));
    constexpr int T = fast_threads<C, 4 * RW>();
    const int64_t Q = P / last_stride<C>();
    const double2* twQ = nullptr;
    NFFT_CHECK(qtab(Q, &twQ));
    static const int bsw = getenv("NFFT45_BOUNDARY_SWAP") != nullptr;  // A/B switch (measured slower)
    const dim3 grid = bsw ? dim3((unsigned)(Bp / 4), (unsigned)(R / RW)) : dim3((unsigned)(R / RW), (unsigned)(Bp / 4));
    LAUNCH_PDL(bm_colin, grid, T, smem, st, A, batch, U, Bp, t.twC, t.tP->lo, t.tP->hi, t.tP->s, twQ, (int)Q, pv.decay,
           AT, bsw);
    return NFFT45_OK;
  }

  int rowout(const double2* Z, double2* out, const ChainPlanView& pv, const double2* xsub) {
    constexpr int RW = bm_rw<C>();
    auto bm_rowout = kbm_rowout<R, C, RW>;
    constexpr size_t smem = fast_smem<C, 4 * RW>();
    NFFT_CHECK(bm_attr(bm_rowout, smem));
    constexpr int T = fast_threads<C, 4 * RW>();
    static const int bsw = getenv("NFFT45_BOUNDARY_SWAP") != nullptr;
    const dim3 grid = bsw ? dim3((unsigned)(Bp / 4), (unsigned)(R / RW)) : dim3((unsigned)(R / RW), (unsigned)(Bp / 4));
    LAUNCH_PDL(bm_rowout, grid, T, smem, st, Z, out, batch, Bp, t.twC, pv.coef, xsub, bsw);
    return NFFT45_OK;
  }
};

template <int R, int C>
static int chain_solve_bm(const ChainPlanView& pv, int kind, const double2* data, int64_t batch, int passes,
                          double2* out, double* norms, cudaStream_t st) {
  using Ch = ChainBM<R, C>;
  constexpr int64_t P = Ch::P, n = Ch::n;
  Ch ch;
  ch.st = st;
  ch.batch = batch;
  ch.Bp = ceil_div(batch, kSig) * kSig;
  ch.groups = (unsigned)(ch.Bp / kSig);
  {
    static const bool small = getenv("NFFT45_TILE4") != nullptr;  // A/B experiment
    ch.small_tiles = small;
    // signal groups fastest in the grid: concurrently resident tiles then
    // cover whole 16-KB rows of the batch-minor layout (DRAM locality; row
    // pass -22 %, column pass -8 % on B200).  NFFT45_GRID_TILES_FIRST restores
    // the tile-major order for A/B runs.
    static const bool tiles_first = getenv("NFFT45_GRID_TILES_FIRST") != nullptr;
    ch.sw = !tiles_first;
    // L2 prefetch of the tile one wave ahead (NFFT45_PREFETCH=<launch slots>):
    // measured slower on B200 (C4: band +0.6 ms, col +0.5 ms at 296 slots),
    // kept as an opt-in A/B switch, off by default
    static const int pf_env = getenv("NFFT45_PREFETCH") ? atoi(getenv("NFFT45_PREFETCH")) : 0;
    ch.pf = pf_env;
    // hybrid two-FFT kernels (2 CTA barriers per tile, warp-local middle
    // passes); NFFT45_HYB=0 restores the all-column-fast kernels for A/B runs
    static const bool hyb_on = !(getenv("NFFT45_HYB") && atoi(getenv("NFFT45_HYB")) == 0);
    ch.hyb = hyb_on && bm_hyb<R, C>() && !ch.small_tiles && pv.tdd != nullptr;  // needs the tile-major tables
    static const bool fuse_on = !(getenv("NFFT45_FUSE") && atoi(getenv("NFFT45_FUSE")) == 0);
    ch.fuse = fuse_on;
  }
  int status = NFFT45_OK;
  {
    const FftTables* a = fft_tables(R, st, &status);
    if (!a) return status;
    const FftTables* b = fft_tables(C, st, &status);
    if (!b) return status;
    const FftTables* c = fft_tables(2 * C, st, &status);
    if (!c) return status;
    ch.t.twR = a->tw;
    ch.t.twC = b->tw;
    ch.t.tw2C = c->tw;
    ch.t.tP = fft_tables(P, st, &status);
    if (!ch.t.tP) return status;
    ch.t.tN = fft_tables(n, st, &status);
    if (!ch.t.tN) return status;
  }
  const int64_t Bp = ch.Bp;
  const GridDev& g = *pv.g;
  Window win = Window::make(kFastM);
  double2* base = nullptr;
  // H [n], Y [n], U [P], Z [P], X [P] (refinement x), R [P] (residual / A transposed)
  const size_t need = sizeof(double2) * Bp * (2 * n + 4 * P);
  NFFT_CUDA(cudaMallocAsync(&base, need, st));
  double2* H = base;
  double2* Y = H + Bp * n;  // padded IFFT_2P column-pass output
  double2* U = Y + Bp * n;
  double2* Z = U + Bp * P;
  double2* X = Z + Bp * P;
  double2* Rs = X + Bp * P;
  // Spreading stores cell j of the fine grid at row (j % 2C) R + j / 2C, so the column pass of
  // FFT_2P reads each column as one contiguous range (it wrote and read 128-byte runs 2C rows apart
  // before: 78 % of the copy rate against the row pass's 98 %) and runs H -> Y instead of in place.
  // NFFT45_COL_PERM=0 restores the natural order (A/B switch).
  static const bool perm_on = !(getenv("NFFT45_COL_PERM") && atoi(getenv("NFFT45_COL_PERM")) == 0);
  // block size of the permutation (NFFT45_COL_BLK, a divisor of 2C)
  static const int cblk_env = getenv("NFFT45_COL_BLK") ? atoi(getenv("NFFT45_COL_BLK")) : 1;
  const int cblk = (cblk_env >= 1 && (2 * C) % cblk_env == 0) ? cblk_env : 1;
  const bool perm = perm_on && spread_layout_pipelined(n, kFastM, Bp);
  auto run = [&]() -> int {
    if (kind == 5) {
      NodeFactor fc5{pv.c5, 0.0, 0};
      // r (or s) -> spread -> colFFT_2P -> band -> mid -> Z
      auto front = [&](const double2* src, bool src_bm) -> int {
        if (perm) {  // grid rows permuted by the spreading kernel: contiguous columns, column pass H -> Y
          NFFT_CHECK(spread_layout(g, n, win, src, batch, src_bm ? Bp : 0, fc5, H, Bp, st, 2 * C, cblk));
          NFFT_CHECK(ch.col(H, Y, cblk));
          NFFT_CHECK(ch.band(Y, U, pv, nullptr));
        } else {
          NFFT_CHECK(spread_layout(g, n, win, src, batch, src_bm ? Bp : 0, fc5, H, Bp, st));
          NFFT_CHECK(ch.col(H, H));
          NFFT_CHECK(ch.band(H, U, pv, nullptr));
        }
        NFFT_CHECK(ch.mid(U, Z, pv));
        return NFFT45_OK;
      };
      NFFT_CHECK(front(data, false));
      for (int pass = 0; pass <= passes; pass++) {
        if (pass == passes) {
          NFFT_CHECK(ch.rowout(Z, out, pv, pass > 0 ? X : nullptr));
        } else {
          NFFT_CHECK(ch.pad(Z, Y, pv, pass > 0 ? X : nullptr, X));
          NFFT_CHECK(ch.row_grid(Y, H));
          NodeFactor ph{nullptr, (double)(P / 2), +1};
          // r = type2(x) - s  (s signal-major, r batch-minor)
          NFFT_CHECK(gather_layout(g, n, win, H, Bp, batch, ph, data, 0, 1, Rs, Bp, st));
          if (norms) NFFT_CHECK(norms_bm(Rs, P, batch, Bp, norms + (int64_t)pass * batch, st));
          NFFT_CHECK(front(Rs, true));
        }
      }
    } else {
      double2* AT = passes > 0 ? Rs : nullptr;
      NFFT_CHECK(ch.colin(data, U, pv, AT));
      auto back = [&](double2* dst, int64_t dst_ld, const double2* xsub, int64_t xsub_ld) -> int {
        NFFT_CHECK(ch.mid(U, Z, pv));
        NFFT_CHECK(ch.pad(Z, Y, pv, nullptr, nullptr));
        NFFT_CHECK(ch.row_grid(Y, H));
        NodeFactor fc4{pv.c4, 0.0, 0};
        return gather_layout(g, n, win, H, Bp, batch, fc4, xsub, xsub_ld, xsub ? 2 : 0, dst, dst_ld, st);
      };
      if (passes == 0) return back(out, 0, nullptr, 0);
      NFFT_CHECK(back(X, Bp, nullptr, 0));
      for (int pass = 0; pass < passes; pass++) {
        const bool last = pass == passes - 1;
        NodeFactor ph{nullptr, (double)(P / 2), -1};
        // passes >= 2: the band epilogue also stores r itself into the free grid buffer (Y, or H
        // when the column pass ran H -> Y), whose norms feed the NonConvergence check
        // (inverse.py:154-159)
        double2* rbuf = perm ? H : Y;
        if (perm) {
          NFFT_CHECK(spread_layout(g, n, win, X, batch, Bp, ph, H, Bp, st, 2 * C, cblk));
          NFFT_CHECK(ch.col(H, Y, cblk));
          NFFT_CHECK(ch.band(Y, U, pv, AT, norms ? rbuf : nullptr));
        } else {
          NFFT_CHECK(spread_layout(g, n, win, X, batch, Bp, ph, H, Bp, st));
          NFFT_CHECK(ch.col(H, H));
          NFFT_CHECK(ch.band(H, U, pv, AT, norms ? rbuf : nullptr));
        }
        if (norms) NFFT_CHECK(norms_bm(rbuf, P, batch, Bp, norms + (int64_t)pass * batch, st));
        NFFT_CHECK(back(last ? out : X, last ? 0 : Bp, X, Bp));
      }
    }
    return NFFT45_OK;
  };
  status = run();
  cudaFreeAsync(base, st);
  return status;
}

// Batched forward transform on the batch-minor passes (kind 1: out[b][p] = sum_q a[b][q]
// e^{-2 pi i p t_q} [- sub]; kind 2: out[b][q] = sum_p S[b][p] e^{+2 pi i p t_q} [- sub]), R = P = Q.
template <int R, int C>
static int forward_solve_bm(const GridDev& g, int kind, const double2* in, int64_t batch, const double2* sub,
                            double2* out, cudaStream_t st) {
  using Ch = ChainBM<R, C>;
  constexpr int64_t P = Ch::P, n = Ch::n;
  Ch ch;
  ch.st = st;
  ch.batch = batch;
  ch.Bp = ceil_div(batch, kSig) * kSig;
  ch.groups = (unsigned)(ch.Bp / kSig);
  ch.sw = true;
  int status = NFFT45_OK;
  {
    const FftTables* a = fft_tables(R, st, &status);
    if (!a) return status;
    const FftTables* c = fft_tables(2 * C, st, &status);
    if (!c) return status;
    ch.t.twR = a->tw;
    ch.t.twC = nullptr;
    ch.t.tw2C = c->tw;
    ch.t.tP = nullptr;
    ch.t.tN = fft_tables(n, st, &status);
    if (!ch.t.tN) return status;
  }
  const int64_t Bp = ch.Bp;
  const Window win = Window::make(kFastM);
  double2* base = nullptr;
  NFFT_CUDA(cudaMallocAsync(&base, sizeof(double2) * Bp * 2 * n + sizeof(double) * P, st));
  double2* H = base;
  double2* Y = H + Bp * n;
  double* dtab = reinterpret_cast<double*>(Y + Bp * n);
  auto run = [&]() -> int {
    LAUNCH(k_fwd_deconv, (unsigned)ceil_div(P, 256), 256, 0, st, dtab, P, win.b);
    if (kind == 1) {
      const NodeFactor f{nullptr, (double)(P / 2), -1};
      if (spread_layout_pipelined(n, kFastM, Bp)) {  // row-permuted grid: contiguous columns
        NFFT_CHECK(spread_layout(g, n, win, in, batch, 0, f, H, Bp, st, 2 * C, 1));
        NFFT_CHECK(ch.col(H, Y, 1));
        NFFT_CHECK(ch.fwd_out(Y, out, sub, dtab));
      } else {
        NFFT_CHECK(spread_layout(g, n, win, in, batch, 0, f, H, Bp, st));
        NFFT_CHECK(ch.col(H, H));
        NFFT_CHECK(ch.fwd_out(H, out, sub, dtab));
      }
    } else {
      NFFT_CHECK(ch.fwd_in(in, Y, dtab));
      NFFT_CHECK(ch.row_grid(Y, H));
      const NodeFactor f{nullptr, (double)(P / 2), +1};
      NFFT_CHECK(gather_layout(g, n, win, H, Bp, batch, f, sub, 0, sub ? 1 : 0, out, 0, st));
    }
    return NFFT45_OK;
  };
  status = run();
  cudaFreeAsync(base, st);
  return status;
}

// ---- part 2: the R = 2C and 3 * 2^k sizes (their own translation unit when NFFT45_BM_PART is set)
int forward_solve_bm_part2(const GridDev& g, int kind, const double2* in, int64_t batch, const double2* sub,
                           double2* out, cudaStream_t st);
int chain_solve_bm_part2(const ChainPlanView& pv, int kind, const double2* data, int64_t batch, int passes,
                         double2* out, double* norms, cudaStream_t st);
#if NFFT45_BM_PART != 1
int forward_solve_bm_part2(const GridDev& g, int kind, const double2* in, int64_t batch, const double2* sub,
                           double2* out, cudaStream_t st) {
  switch (g.Q) {
    case 2048: return forward_solve_bm<64, 32>(g, kind, in, batch, sub, out, st);
    case 8192: return forward_solve_bm<128, 64>(g, kind, in, batch, sub, out, st);
    case 32768: return forward_solve_bm<256, 128>(g, kind, in, batch, sub, out, st);
    case 131072: return forward_solve_bm<512, 256>(g, kind, in, batch, sub, out, st);
  }
  return NFFT45_ERR_INVALID_ARGUMENT;
}
int chain_solve_bm_part2(const ChainPlanView& pv, int kind, const double2* data, int64_t batch, int passes,
                         double2* out, double* norms, cudaStream_t st) {
  switch (pv.P) {
    case 2048: return chain_solve_bm<64, 32>(pv, kind, data, batch, passes, out, norms, st);
    case 8192: return chain_solve_bm<128, 64>(pv, kind, data, batch, passes, out, norms, st);
    case 32768: return chain_solve_bm<256, 128>(pv, kind, data, batch, passes, out, norms, st);
    case 131072: return chain_solve_bm<512, 256>(pv, kind, data, batch, passes, out, norms, st);
    case 524288: return chain_solve_bm<1024, 512>(pv, kind, data, batch, passes, out, norms, st);
    case 3072: return chain_solve_bm<48, 64>(pv, kind, data, batch, passes, out, norms, st);
    case 12288: return chain_solve_bm<96, 128>(pv, kind, data, batch, passes, out, norms, st);
    case 49152: return chain_solve_bm<192, 256>(pv, kind, data, batch, passes, out, norms, st);
    case 196608: return chain_solve_bm<384, 512>(pv, kind, data, batch, passes, out, norms, st);
    case 786432: return chain_solve_bm<768, 1024>(pv, kind, data, batch, passes, out, norms, st);
  }
  return NFFT45_ERR_INVALID_ARGUMENT;
}
#endif  // NFFT45_BM_PART != 1

#if NFFT45_BM_PART != 2
bool forward_bm_usable(int64_t Q, int64_t P, int m, int64_t batch) {
  static const bool off = getenv("NFFT45_NO_FORWARD_BM") != nullptr;  // A/B switch: generic batched forward path
  int r = 0, c = 0;
  return !off && m == kFastM && Q == P && batch >= 16 && chain_bm_hybrid_factors(P, &r, &c);
}

int forward_run_bm(const GridDev& g, int kind, const double2* in, int64_t batch, const double2* sub, double2* out,
                   cudaStream_t st) {
  // kbm_col addresses a tile's rows with 32-bit offsets (n * Bp < 2^31): large batches run in
  // independent slices of rows, like chain_run_bm
  const int64_t max_rows = ((int64_t(1) << 31) / (2 * g.Q)) / kSig * kSig;
  if (batch > max_rows && max_rows >= 16) {
    for (int64_t b0 = 0; b0 < batch; b0 += max_rows) {
      const int64_t nb = std::min(max_rows, batch - b0);
      NFFT_CHECK(forward_run_bm(g, kind, in + b0 * g.Q, nb, sub ? sub + b0 * g.Q : nullptr, out + b0 * g.Q, st));
    }
    return NFFT45_OK;
  }
  switch (g.Q) {
    case 1024: return forward_solve_bm<32, 32>(g, kind, in, batch, sub, out, st);
    case 4096: return forward_solve_bm<64, 64>(g, kind, in, batch, sub, out, st);
    case 16384: return forward_solve_bm<128, 128>(g, kind, in, batch, sub, out, st);
    case 65536: return forward_solve_bm<256, 256>(g, kind, in, batch, sub, out, st);
  }
  return forward_solve_bm_part2(g, kind, in, batch, sub, out, st);
}

bool chain_bm_hybrid_factors(int64_t P, int* R, int* C) {
  auto set = [&](int r, int c) {
    *R = r;
    *C = c;
    return true;
  };
  switch (P) {  // the sizes whose ChainBM<R, C> satisfies bm_hyb (chain_run_bm's table)
    case 1024: return bm_hyb<32, 32>() && set(32, 32);
    case 2048: return bm_hyb<64, 32>() && set(64, 32);
    case 4096: return bm_hyb<64, 64>() && set(64, 64);
    case 8192: return bm_hyb<128, 64>() && set(128, 64);
    case 16384: return bm_hyb<128, 128>() && set(128, 128);
    case 32768: return bm_hyb<256, 128>() && set(256, 128);
    case 65536: return bm_hyb<256, 256>() && set(256, 256);
    case 131072: return bm_hyb<512, 256>() && set(512, 256);
  }
  return false;
}

bool chain_bm_supported(int64_t P) {
  switch (P) {
    case 1024: case 4096: case 16384: case 65536: case 262144: case 1048576:  // R = C
    case 2048: case 8192: case 32768: case 131072: case 524288:               // R = 2C
    case 3072: case 12288: case 49152: case 196608: case 786432:              // R = 3 * 2^a
      return true;
  }
  return false;
}

int chain_run_bm(const ChainPlanView& pv, int kind, const double2* data, int64_t batch, int passes, double2* out,
                 double* norms, cudaStream_t st) {
  // the kernels address a tile's rows with 32-bit offsets: keep n * Bp below
  // 2^31 by solving large batches in independent slices (rows are independent)
  const int64_t max_rows = ((int64_t(1) << 31) / (2 * pv.P)) / kSig * kSig;
  if (batch > max_rows && max_rows >= 16) {
    double* sn = nullptr;  // per-slice [passes][nb] norms, scattered into [passes][batch]
    if (norms && passes > 0) NFFT_CUDA(cudaMallocAsync(&sn, sizeof(double) * passes * max_rows, st));
    int status = NFFT45_OK;
    for (int64_t b0 = 0; b0 < batch && status == NFFT45_OK; b0 += max_rows) {
      const int64_t nb = std::min(max_rows, batch - b0);
      status = chain_run_bm(pv, kind, data + b0 * pv.P, nb, passes, out + b0 * pv.P, sn, st);
      if (status == NFFT45_OK && sn) {
        const cudaError_t e = cudaMemcpy2DAsync(norms + b0, sizeof(double) * batch, sn, sizeof(double) * nb,
                                                sizeof(double) * nb, passes, cudaMemcpyDeviceToDevice, st);
        if (e != cudaSuccess) status = cuda_fail(e, "norms slice copy");
      }
    }
    if (sn) cudaFreeAsync(sn, st);
    return status;
  }
  switch (pv.P) {
    case 1024: return chain_solve_bm<32, 32>(pv, kind, data, batch, passes, out, norms, st);
    case 4096: return chain_solve_bm<64, 64>(pv, kind, data, batch, passes, out, norms, st);
    case 16384: return chain_solve_bm<128, 128>(pv, kind, data, batch, passes, out, norms, st);
    case 65536: return chain_solve_bm<256, 256>(pv, kind, data, batch, passes, out, norms, st);
    case 262144: return chain_solve_bm<512, 512>(pv, kind, data, batch, passes, out, norms, st);
    case 1048576: return chain_solve_bm<1024, 1024>(pv, kind, data, batch, passes, out, norms, st);
  }
  return chain_solve_bm_part2(pv, kind, data, batch, passes, out, norms, st);
}
#endif  // NFFT45_BM_PART != 2
#endif  // NFFT45_EXP_ONLY

}  // namespace nfft45
