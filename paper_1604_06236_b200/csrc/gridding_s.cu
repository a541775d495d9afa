// gridding_s.cu — Gaussian spreading / interpolation for ONE or a few signals
// (batch < 32), half-width m = 14: the single-transform configurations (P up
// to 2^20, plan builds) where nothing can be amortised over a batch.
//
// Spreading (gridding.py:57-72, forward.py:47-54), output-stationary:
//   CTA = 128 (or 256) consecutive fine-grid cells x SB signals.  The nodes that reach
//   the tile (all periodic images, a contiguous ascending range per image,
//   from per-tile ranges cached in the node set) are staged in chunks:
//   phase 1, one thread per node: unwrapped centre, the 29 factorised Gaussian
//   weights, the node's amplitude x factor for every signal; then one thread
//   per tile cell finds its first contributing node by binary search;
//   phase 2, one thread per cell: sum over its contributing nodes in
//   ascending order (caxpy, the same fma sequence as every other spreading
//   kernel of the library, so results are bitwise identical to them).
// Interpolation (forward.py:91-102):
//   CTA = 256 consecutive ascending nodes x SB signals.  The cell span under
//   the block's windows is staged once in shared memory (skewed slots so that
//   lanes whose nodes sit ~2 cells apart hit distinct banks); one thread per
//   node accumulates its 29 taps in ascending cell order.  Blocks whose span
//   exceeds the staging buffer (strongly clustered nodes) read the taps from
//   global memory instead (same arithmetic).
#include <algorithm>
#include <cstdlib>

#include "ops.cuh"

namespace nfft45 {

namespace {
constexpr int kM = kFastM;        // 14
constexpr int kTaps = 2 * kM + 1;  // 29
// spread: TILE cells per CTA (= threads); nodes staged per chunk (even, so the
// amplitude block after the weights stays 16-B aligned): ~ (TILE + 2 kM) / 2
// nodes reach a tile of a jittered grid with two cells per node
template <int TILE> struct STile {
  static constexpr int cap = TILE == 256 ? 160 : 88;
  static constexpr int xs = TILE + 2 * kM + 2;  // first-node table entries (cells -kM .. TILE+kM)
  static_assert((cap * 29) % 2 == 0 && cap % 2 == 0, "16-B alignment of the amplitude block");
  static size_t smem(int sb) {
    return sizeof(double) * cap * kTaps + sizeof(double2) * sb * cap + sizeof(int) * (cap + xs);
  }
};
// gather: kGNodes nodes per CTA (= threads), 4 x kGNodes staged cells per CTA (and signal)

__device__ __forceinline__ int gslot(int c) { return c + (c >> 3); }  // skewed staging slot

__device__ __forceinline__ void taps29s(double f, double alpha, const GaussTab& G, double* w) {
  // gauss_fast<14> (gridding.cu): exp(-alpha f^2) * exp(2 alpha f)^k * exp(-alpha k^2)
  double e1 = exp(-alpha * f * f);
  double E = exp(2.0 * alpha * f);
  double Ei = 1.0 / E;
  w[kM] = e1;
  double pp = e1, pn = e1;
#pragma unroll
  for (int k = 1; k <= kM; k++) {
    pp *= E;
    pn *= Ei;
    w[kM + k] = pp * G.g[k];
    w[kM - k] = pn * G.g[k];
  }
}

__device__ __forceinline__ double2 factor_s(const NodeFactor& f, int64_t q, double t) {
  if (f.fac) return f.fac[q];
  if (f.phaseK != 0.0) {
    double x = turns_of_product(f.phaseK, t);
    return cis_turns(f.phase_sign < 0 ? -x : x);
  }
  return make_double2(1.0, 0.0);
}

__device__ __forceinline__ int64_t floordiv_s(int64_t a, int64_t b) {
  int64_t q = a / b;
  if ((a % b != 0) && ((a < 0) != (b < 0))) q--;
  return q;
}
}  // namespace

// amp == nullptr: unit amplitudes (the plan's log-sum NFFT, lagrange.py:57-75).
template <int SB, int kSTile>
__global__ void __launch_bounds__(kSTile, (SB == 1 ? 5 : 2) * 256 / kSTile) k_spread_s(const double* __restrict__ ts, const int* __restrict__ perm,
                                                     int64_t Q, int64_t n, double alpha, GaussTab G,
                                                     const double2* __restrict__ amp, int64_t batch, NodeFactor nf,
                                                     double2* __restrict__ H, const int2* __restrict__ ranges,
                                                     int NS) {
  pdl_enter();  // programmatic dependent launch: wait for the producer grid
  constexpr int kSCap = STile<kSTile>::cap;
  extern __shared__ __align__(16) unsigned char smraw[];
  double* W = reinterpret_cast<double*>(smraw);                   // [cap][kTaps]
  double2* A = reinterpret_cast<double2*>(W + kSCap * kTaps);  // [SB][cap]
  int* Cc = reinterpret_cast<int*>(A + SB * kSCap);               // [cap] centre relative to j0 (unwrapped)
  int* Fx = Cc + kSCap;                                           // [kXs] first node with Cc >= x

  const int tid = threadIdx.x;
  const int64_t j0 = (int64_t)blockIdx.x * kSTile;
  const int64_t b0 = (int64_t)blockIdx.y * SB;
  // first periodic image reaching the tile: ceil((-kM - (j1 - 1)) / n); the
  // argument lies in [-kM, n), so one comparison unless n is tiny (int64
  // division is a long software sequence)
  const int64_t x_lo = -kM - (min(j0 + kSTile, n) - 1) + n - 1;
  const int64_t s_lo = n > kM ? (x_lo < 0 ? -1 : 0) : floordiv_s(x_lo, n);

  double2 acc[SB];
#pragma unroll
  for (int s = 0; s < SB; s++) acc[s] = make_double2(0.0, 0.0);

  // periodic images in increasing order, nodes ascending within each image
  // (the summation order of every spreading kernel of the library); centres
  // ascend within one image only, so the first-node table is per chunk of
  // one image
  bool first = true;
  for (int si = 0; si < NS; si++) {
    const int2 r = ranges[blockIdx.x * (int64_t)NS + si];
    const int64_t shift = (s_lo + si) * n + j0;
    for (int base = r.x; base < r.y; base += kSCap) {
      const int cnt = min(kSCap, r.y - base);
      if (!first) __syncthreads();  // previous chunk consumed
      first = false;
      // phase 1: node geometry, weights, amplitudes
      for (int e = tid; e < cnt; e += kSTile) {
        const int64_t q = base + e;
        const double t = ts[q];
        const int pq = perm[q];
        // the amplitudes (a dependent global load through perm) are requested
        // before the weights are computed, so their latency hides under it
        double2 av[SB];
#pragma unroll
        for (int s = 0; s < SB; s++)
          av[s] = (amp && b0 + s < batch) ? amp[(b0 + s) * Q + pq] : make_double2(0.0, 0.0);
        const double2 fq = factor_s(nf, q, t);
        const NodeGeo geo = node_geo(t, (double)n);
        Cc[e] = (int)((int64_t)geo.i0 - shift);
        double w[kTaps];
        taps29s(geo.f, alpha, G, w);
#pragma unroll
        for (int k = 0; k < kTaps; k++) W[e * kTaps + k] = w[k];
#pragma unroll
        for (int s = 0; s < SB; s++) {
          double2 a = make_double2(0.0, 0.0);
          if (b0 + s < batch) a = amp ? cmul(av[s], fq) : fq;
          A[s * kSCap + e] = a;
        }
      }
      __syncthreads();
      // first staged node whose centre is >= x, x = -kM .. kSTile + kM: node e
      // owns the x in (Cc[e-1], Cc[e]] (centres ascend within an image); x
      // beyond the last centre map to cnt
      for (int e = tid; e <= cnt; e += kSTile) {
        const int xa = max(e > 0 ? Cc[e - 1] + 1 : -kM, -kM);
        const int xb = min(e < cnt ? Cc[e] : kSTile + kM, kSTile + kM);
        for (int x = xa; x <= xb; x++) Fx[x + kM] = e;
      }
      __syncthreads();
      // phase 2: this thread's cell j0 + tid, contributing nodes in ascending order
      const int lo = Fx[tid], hi = Fx[tid + 2 * kM + 1];  // centres in [tid - kM, tid + kM]
#pragma unroll 4
      for (int e = lo; e < hi; e++) {
        const double wk = W[e * kTaps + (tid - Cc[e] + kM)];
#pragma unroll
        for (int s = 0; s < SB; s++) caxpy(acc[s], wk, A[s * kSCap + e]);
      }
    }
  }
  if (j0 + tid < n) {
#pragma unroll
    for (int s = 0; s < SB; s++) {
      const int64_t b = b0 + s;
      if (b < batch) H[b * n + j0 + tid] = acc[s];
    }
  }
}

// Warp-tiled variant for one signal: every warp is an independent 32-cell
// tile with its own cached node range (tile ranges at TC = 32), no CTA
// barriers.  Per chunk of <= 32 contributing nodes (all periodic images in
// increasing order, nodes ascending), lane l stages node l's centre, 29
// weights and amplitude x factor; then every lane (= cell) walks the chunk's
// nodes in ascending order -- a warp-uniform loop, so the centre and the
// amplitude are broadcast reads and the weights of one node sit in
// consecutive words across the lanes -- and accumulates the nodes whose
// window covers its cell.  Same terms, same order, same fma sequence as the
// other spreading kernels: bitwise identical results.
constexpr int kWWarps = 4;
__global__ void __launch_bounds__(kWWarps * 32, 7) k_spread_w(const double* __restrict__ ts, const int* __restrict__ perm,
                                                              int64_t Q, int64_t n, double alpha, GaussTab G,
                                                              const double2* __restrict__ amp, NodeFactor nf,
                                                              double2* __restrict__ H, const int2* __restrict__ ranges,
                                                              int NS) {
  pdl_enter();  // programmatic dependent launch: wait for the producer grid
  __shared__ __align__(16) double Wsh[kWWarps][32 * kTaps];
  __shared__ __align__(16) double2 Ash[kWWarps][32];
  __shared__ int Csh[kWWarps][32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t tile = (int64_t)blockIdx.x * kWWarps + w;
  const int64_t j0 = tile * 32;
  if (j0 >= n) return;
  double* W = Wsh[w];
  double2* A = Ash[w];
  int* C = Csh[w];
  const int64_t x_lo = -kM - (min(j0 + 32, n) - 1) + n - 1;
  const int64_t s_lo = n > kM ? (x_lo < 0 ? -1 : 0) : floordiv_s(x_lo, n);
  double2 acc = make_double2(0.0, 0.0);
  for (int si = 0; si < NS; si++) {
    const int2 r = ranges[tile * NS + si];
    const int64_t shift = (s_lo + si) * n + j0;
    for (int base = r.x; base < r.y; base += 32) {
      const int cnt = min(32, r.y - base);
      if (lane < cnt) {
        const int64_t q = base + lane;
        const double t = ts[q];
        const int pq = perm[q];
        const double2 av = amp ? amp[pq] : make_double2(0.0, 0.0);
        const double2 fq = factor_s(nf, q, t);
        const NodeGeo geo = node_geo(t, (double)n);
        C[lane] = (int)((int64_t)geo.i0 - shift);
        double wt[kTaps];
        taps29s(geo.f, alpha, G, wt);
#pragma unroll
        for (int k = 0; k < kTaps; k++) W[lane * kTaps + k] = wt[k];
        A[lane] = amp ? cmul(av, fq) : fq;
      }
      __syncwarp();
      for (int e = 0; e < cnt; e++) {
        const int d = lane - C[e] + kM;
        if (d >= 0 && d < kTaps) caxpy(acc, W[e * kTaps + d], A[e]);
      }
      __syncwarp();
    }
  }
  if (j0 + lane < n) H[j0 + lane] = acc;
}

// mode 0: out = v;  1: out = v - sub;  2: out = sub - v  (v = factor * window sum)
template <int SB, int kGNodes>
__global__ void __launch_bounds__(kGNodes, (SB == 1 ? 3 : 2) * 256 / kGNodes) k_gather_s(const double* __restrict__ ts, const int* __restrict__ perm,
                                                      int64_t Q, int64_t n, double alpha, GaussTab G,
                                                      const double2* __restrict__ H, int64_t batch, NodeFactor nf,
                                                      const double2* __restrict__ sub, int mode,
                                                      double2* __restrict__ out) {
  pdl_enter();  // programmatic dependent launch: wait for the producer grid
  extern __shared__ __align__(16) unsigned char smraw[];
  constexpr int kGCap = 4 * kGNodes;
  double2* Y = reinterpret_cast<double2*>(smraw);  // [SB][gslot(kGCap)]
  constexpr int kRow = kGCap + kGCap / 8;

  const int tid = threadIdx.x;
  const int64_t q0 = (int64_t)blockIdx.x * kGNodes;
  const int nq = (int)min((int64_t)kGNodes, Q - q0);
  const int64_t b0 = (int64_t)blockIdx.y * SB;
  const bool has = tid < nq;
  const int64_t q = q0 + (has ? tid : nq - 1);
  // every per-node global operand is requested up front (one round trip)
  const double t = ts[q];
  const double2 fq = factor_s(nf, q, t);
  const int64_t pq = perm[q];
  double2 sv[SB];
#pragma unroll
  for (int s = 0; s < SB; s++)
    sv[s] = (mode != 0 && has && b0 + s < batch) ? sub[(b0 + s) * Q + pq] : make_double2(0.0, 0.0);
  // cell span of the block (centres ascend): from its first and last node
  const int cs = node_geo(ts[q0], (double)n).i0 - kM;
  const int len = node_geo(ts[q0 + nq - 1], (double)n).i0 + kM + 1 - cs;
  const bool staged = len <= kGCap && n >= 2 * kTaps;
  const int ni = (int)n;
  if (staged) {
    for (int s = 0; s < SB; s++) {
      const int64_t b = min(b0 + s, batch - 1);
      const double2* row = H + b * n;
      // all of this thread's cells are requested before the first is stored
      // (one global round trip instead of one per staged cell)
      constexpr int kPer = kGCap / kGNodes;
      double2 v[kPer];
#pragma unroll
      for (int i = 0; i < kPer; i++) {
        const int c = tid + i * kGNodes;
        int cell = cs + c;
        cell = cell < 0 ? cell + ni : (cell >= ni ? cell - ni : cell);
        if (c < len) v[i] = row[cell];
      }
#pragma unroll
      for (int i = 0; i < kPer; i++) {
        const int c = tid + i * kGNodes;
        if (c < len) Y[s * kRow + gslot(c)] = v[i];
      }
    }
  }
  const NodeGeo geo = node_geo(t, (double)n);
  double w[kTaps];
  taps29s(geo.f, alpha, G, w);
  __syncthreads();
  if (!has) return;
  double2 acc[SB];
#pragma unroll
  for (int s = 0; s < SB; s++) acc[s] = make_double2(0.0, 0.0);
  if (staged) {
    const int c0 = geo.i0 - kM - cs;
#pragma unroll
    for (int k = 0; k < kTaps; k++) {
      const int sl = gslot(c0 + k);
#pragma unroll
      for (int s = 0; s < SB; s++) caxpy(acc[s], w[k], Y[s * kRow + sl]);
    }
  } else {
    int64_t idx = ((int64_t)geo.i0 - kM) % n;
    if (idx < 0) idx += n;
#pragma unroll
    for (int k = 0; k < kTaps; k++) {
#pragma unroll
      for (int s = 0; s < SB; s++) caxpy(acc[s], w[k], __ldg(&H[min(b0 + s, batch - 1) * n + idx]));
      idx = idx + 1 == n ? 0 : idx + 1;
    }
  }
#pragma unroll
  for (int s = 0; s < SB; s++) {
    const int64_t b = b0 + s;
    if (b >= batch) continue;
    double2 v = cmul(acc[s], fq);
    if (mode == 1) v = csub(v, sv[s]);
    else if (mode == 2) v = csub(sv[s], v);
    out[b * Q + pq] = v;
  }
}

// ------------------------------------------------------------ host side

int spread_small(const GridDev& g, int64_t n, const Window& win, const double2* amp, int64_t batch, NodeFactor f,
                 double2* H, cudaStream_t st) {
  static const int env_tile = getenv("NFFT45_STILE") ? atoi(getenv("NFFT45_STILE")) : 0;  // A/B switch
  // 128-cell tiles (default): ~80 nodes per CTA, 10 CTAs/SM, barrier groups of 4 warps;
  // single transforms 0.3-2 % faster than 256-cell tiles, bitwise identical (scripts/ab_env.sh)
  const int tile = env_tile == 256 ? 256 : 128;
  // single signals on grids up to 2^17 cells: warp tiles (P = 2^14 .. 2^16 single
  // transforms 1.5-3.5 % faster; at 2^19 .. 2^21 cells 1-3 % slower: every node's
  // weights are computed by ~2 warps).  NFFT45_SPREAD_WARP=0 / 1 forces off / on.
  static const int warp_env = getenv("NFFT45_SPREAD_WARP") ? atoi(getenv("NFFT45_SPREAD_WARP")) : -1;
  const bool warp_tiles = warp_env < 0 ? n <= (int64_t(1) << 17) : warp_env > 0;
  if (warp_tiles && batch == 1 && win.m == kM && tile_images(n, win.m, 32) <= 8) {
    const int NSw = tile_images(n, win.m, 32);
    const int2* rw = nullptr;
    int2* ownw = nullptr;
    NFFT_CHECK(tile_ranges(g, n, win.m, 32, NSw, st, &rw, &ownw));
    const GaussTab Gw = gauss_tab(win);
    LAUNCH_PDL(k_spread_w, (unsigned)ceil_div(ceil_div(n, 32), kWWarps), kWWarps * 32, 0, st, g.ts, g.perm, g.Q, n,
           win.alpha, Gw, amp, f, H, rw, NSw);
    if (ownw) NFFT_CUDA(cudaFreeAsync(ownw, st));
    return NFFT45_OK;
  }
  const int64_t ntiles = ceil_div(n, tile);
  const int NS = tile_images(n, win.m, tile);
  if (NS > 8 || win.m != kM) return NFFT45_ERR_INVALID_ARGUMENT;
  const int2* ranges = nullptr;
  int2* own = nullptr;
  NFFT_CHECK(tile_ranges(g, n, win.m, tile, NS, st, &ranges, &own));
  const GaussTab G = gauss_tab(win);
  const int sb = batch >= 4 ? 4 : 1;
  const dim3 grid((unsigned)ntiles, (unsigned)ceil_div(batch, sb));
  // one LAUNCH per instantiation: the profiler keys kernels by the launched name
#define NFFT45_SPREAD_S(name, SBv, TILEv)                                                                  \
  {                                                                                                       \
    auto name = k_spread_s<SBv, TILEv>;                                                                   \
    const size_t smem = STile<TILEv>::smem(SBv);                                                          \
    NFFT_CUDA(cudaFuncSetAttribute(name, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));       \
    LAUNCH_PDL(name, grid, TILEv, smem, st, g.ts, g.perm, g.Q, n, win.alpha, G, amp, batch, f, H, ranges, NS); \
  }
  if (tile == 128) {
    if (sb == 4) NFFT45_SPREAD_S(spread_s4, 4, 128) else NFFT45_SPREAD_S(spread_s1, 1, 128)
  } else {
    if (sb == 4) NFFT45_SPREAD_S(spread_s4, 4, 256) else NFFT45_SPREAD_S(spread_s1, 1, 256)
  }
#undef NFFT45_SPREAD_S
  if (own) NFFT_CUDA(cudaFreeAsync(own, st));
  return NFFT45_OK;
}

int gather_small(const GridDev& g, int64_t n, const Window& win, const double2* H, int64_t batch, NodeFactor f,
                 const double2* sub, int mode, double2* out, cudaStream_t st) {
  if (win.m != kM) return NFFT45_ERR_INVALID_ARGUMENT;
  if (!sub) mode = 0;
  const GaussTab G = gauss_tab(win);
  const int sb = batch >= 4 ? 4 : 1;
  static const int env_nodes = getenv("NFFT45_GNODES") ? atoi(getenv("NFFT45_GNODES")) : 0;  // A/B switch
  // 128-node CTAs (default): 6 CTAs/SM; single transforms up to 1.5 % faster than
  // 256-node CTAs at P >= 2^18, equal below, bitwise identical (scripts/ab_env.sh)
  const int nodes = env_nodes == 256 ? 256 : (env_nodes == 64 ? 64 : 128);
  const size_t smem = sizeof(double2) * sb * (4 * nodes + 4 * nodes / 8);
  const dim3 grid((unsigned)ceil_div(g.Q, nodes), (unsigned)ceil_div(batch, sb));
#define NFFT45_GATHER_S(name, SBv, NODESv)                                                                 \
  {                                                                                                       \
    auto name = k_gather_s<SBv, NODESv>;                                                                  \
    NFFT_CUDA(cudaFuncSetAttribute(name, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));       \
    LAUNCH_PDL(name, grid, NODESv, smem, st, g.ts, g.perm, g.Q, n, win.alpha, G, H, batch, f, sub, mode, out); \
  }
  if (nodes == 128) {
    if (sb == 4) NFFT45_GATHER_S(gather_s4, 4, 128) else NFFT45_GATHER_S(gather_s1, 1, 128)
  } else if (nodes == 64) {
    if (sb == 4) NFFT45_GATHER_S(gather_s4, 4, 64) else NFFT45_GATHER_S(gather_s1, 1, 64)
  } else {
    if (sb == 4) NFFT45_GATHER_S(gather_s4, 4, 256) else NFFT45_GATHER_S(gather_s1, 1, 256)
  }
#undef NFFT45_GATHER_S
  return NFFT45_OK;
}

}  // namespace nfft45
