// gridding_b.cu — batched Gaussian spreading / interpolation (many signals,
// one node set), half-width m = 14.
//
// Both kernels treat the banded window as small dense blocks: the lanes of
// a warp run over SIGNALS (so every shared-memory access is a contiguous,
// conflict-free 512-byte row and the window weights are warp-uniform
// broadcasts), and each thread keeps a block of cells (spread) or nodes
// (gather) in registers so one staged operand feeds 8 FMAs.  The
// accumulation order is fixed (ascending nodes / ascending cells), so
// results are bitwise reproducible and independent of the batch split.
#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "ops.cuh"
#include "tma.cuh"

namespace nfft45 {

namespace {

constexpr int kM = kFastM;       // 14
constexpr int kWRow = 44;        // padded weight row: taps -m-7 .. m+7 (+1 parity shift), 16-B aligned
constexpr int kCPW = 8;          // spread: cells per warp
constexpr int kSpreadWarps = 8;  // spread: warps per CTA -> 64 cells
constexpr int kSpreadTile = kCPW * kSpreadWarps;
constexpr int kSpreadCap = 72;   // nodes staged per batch
constexpr int kNPW = 8;          // gather: nodes per warp
constexpr int kGatherWarps = 4;  // gather: warps per CTA -> 32 nodes
constexpr int kGatherNodes = kNPW * kGatherWarps;
constexpr int kGatherSpan = 112; // cells staged per chunk
constexpr int kWTSpan = 64;      // per-warp weight-table cells per chunk

__device__ __forceinline__ int swz(int sig, int row) { return sig ^ (row & 7); }
// Slot of (row e, signal sig) in a [rows][SIG] tile staged from a SIGNAL-MAJOR
// array by cp.async with lanes = consecutive rows of one signal: 8 consecutive
// rows of a signal share one 128-byte line (an LDGSTS writes shared memory
// sector by sector as the data returns, so lanes that scatter over 512-byte
// rows cost 6-7x the wavefronts -- ncu: 38 % of the first spreading launch);
// the XOR keeps the reads (lanes = consecutive signals, 128 bytes apart)
// on 8 distinct bank groups.
template <int SIG>
__device__ __forceinline__ int swz_nb(int sig, int e) { return (((e >> 3) * SIG + sig) << 3) + ((e & 7) ^ (sig & 7)); }

// 16-byte global -> shared async copy (LDGSTS); `valid == false` zero-fills.
__device__ __forceinline__ void cp_async16(void* sdst, const void* gsrc, bool valid) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(sdst);
  const int n = valid ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gsrc), "r"(n));
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::); }
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait_group() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// 29 factorised Gaussian taps of one node (see gridding.cu gauss_fast).
__device__ __forceinline__ void taps29(double f, double alpha, const GaussTab& G, double* w) {
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

__device__ __forceinline__ double2 factor_at(const NodeFactor& f, int64_t q, double t) {
  if (f.fac) return f.fac[q];
  if (f.phaseK != 0.0) {
    double x = turns_of_product(f.phaseK, t);
    return cis_turns(f.phase_sign < 0 ? -x : x);
  }
  return make_double2(1.0, 0.0);
}

__device__ __forceinline__ int64_t floordiv_b(int64_t a, int64_t b) {
  int64_t q = a / b;
  if ((a % b != 0) && ((a < 0) != (b < 0))) q--;
  return q;
}

}  // namespace

// ------------------------------------------------------------- spread

// CTA: 64 consecutive cells x (32*SPL) signals; warp w owns cells
// [j0 + 8w, j0 + 8w + 8).  Contributing nodes (all periodic images, from
// `ranges`) are streamed through shared memory in batches of kSpreadCap:
// per node one padded weight row (zeros outside the window, so the 8-cell
// inner product needs no predicates) and the node's amplitudes for every
// signal of the CTA.
template <int SPL>
__global__ void __launch_bounds__(256, 2) k_spread_b(const double* __restrict__ ts, const int* __restrict__ perm,
                                                    int64_t Q, int64_t n, double alpha, GaussTab G,
                                                    const double2* __restrict__ amp, int64_t batch, NodeFactor nf,
                                                    double2* __restrict__ H, const int2* __restrict__ ranges,
                                                    int NS, int64_t amp_ld, int64_t H_ld) {
  // amp_ld == 0: amp is [batch][Q] (signal-major), else amp[q * amp_ld + b];
  // H_ld == 0: H is [batch][n], else H[j * H_ld + b] (H_ld >= batch, padded)
  constexpr int SIG = 32 * SPL;
  extern __shared__ __align__(16) unsigned char smraw[];
  double2* A = reinterpret_cast<double2*>(smraw);                              // [cap][SIG] swizzled
  double* W = reinterpret_cast<double*>(A + kSpreadCap * SIG);                 // [cap][kWRow]
  double2* F = reinterpret_cast<double2*>(W + kSpreadCap * kWRow);             // [cap] node factor
  int* Cc = reinterpret_cast<int*>(F + kSpreadCap);                            // [cap] image index (scratch)
  int* Pi = Cc + kSpreadCap;                                                   // [cap] caller index
  int* Qs = Pi + kSpreadCap;                                                   // [cap] ascending index
  int* Cc2 = Qs + kSpreadCap;                                                  // [cap] effective centre
  __shared__ int s_cnt[8];
  __shared__ int s_off[8];

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t j0 = (int64_t)blockIdx.x * kSpreadTile;
  const int64_t b0 = (int64_t)blockIdx.y * SIG;
  const int jw = (int)j0 + warp * kCPW;  // first cell of this warp
  const int64_t s_lo = floordiv_b(-kM - (min(j0 + kSpreadTile, n) - 1) + n - 1, n);

  // concatenated node list over periodic images
  if (tid == 0) {
    int acc = 0;
    for (int si = 0; si < NS && si < 8; si++) {
      int2 r = ranges[blockIdx.x * (int64_t)NS + si];
      s_off[si] = acc;
      s_cnt[si] = r.y - r.x;
      acc += r.y - r.x;
    }
  }
  __syncthreads();
  int total = 0;
  for (int si = 0; si < NS && si < 8; si++) total += s_cnt[si];

  double2 acc[kCPW][SPL];
#pragma unroll
  for (int c = 0; c < kCPW; c++)
#pragma unroll
    for (int s = 0; s < SPL; s++) acc[c][s] = make_double2(0.0, 0.0);

  for (int base = 0; base < total; base += kSpreadCap) {
    const int cnt = min(kSpreadCap, total - base);
    __syncthreads();
    // phase 0: node index and caller position (sources of the async copies)
    for (int e = tid; e < cnt; e += blockDim.x) {
      int g = base + e, si = 0;
      while (si + 1 < NS && si + 1 < 8 && g >= s_off[si + 1]) si++;
      const int64_t q = ranges[blockIdx.x * (int64_t)NS + si].x + (g - s_off[si]);
      Qs[e] = (int)q;
      Pi[e] = perm[q];
      Cc[e] = si;  // image index for now
    }
    __syncthreads();
    // phase 1: amplitudes, transposed to [node][signal] with async copies
    // (one signal row per warp pass: lanes read consecutive nodes)
    if (amp_ld == 0) {
      for (int sig = warp; sig < SIG; sig += kSpreadWarps) {
        const int64_t b = b0 + sig;
        const bool ok = b < batch;
        const double2* row = amp + (ok ? b : 0) * Q;
        for (int e = lane; e < cnt; e += 32) cp_async16(&A[e * SIG + swz(sig, e)], row + Pi[e], ok);
      }
    } else {
      for (int e = warp; e < cnt; e += kSpreadWarps) {
        const double2* row = amp + (int64_t)Pi[e] * amp_ld + b0;
#pragma unroll
        for (int s2 = 0; s2 < SPL; s2++) {
          const int sig = lane + 32 * s2;
          const bool ok = b0 + sig < batch;
          cp_async16(&A[e * SIG + swz(sig, e)], row + (ok ? sig : 0), ok);
        }
      }
    }
    // phase 2 (overlaps the copies): geometry, padded weight rows, factors
    for (int e = tid; e < cnt; e += blockDim.x) {
      const int64_t q = Qs[e];
      const int si = Cc[e];
      const double t = ts[q];
      const NodeGeo geo = node_geo(t, (double)n);
      const int ce = (int)((int64_t)geo.i0 - (s_lo + si) * n);
      F[e] = factor_at(nf, q, t);
      double w[2 * kM + 1];
      taps29(geo.f, alpha, G, w);
      double* row = W + e * kWRow;
      // parity shift makes every 8-cell read 16-byte aligned; two unrolled
      // variants keep w[] in registers
      if ((ce + 1) & 1) {
#pragma unroll
        for (int x = 0; x < kWRow; x++) {
          const int k = x - 1 - kM - 7;
          row[x] = (k >= -kM && k <= kM) ? w[(k >= -kM && k <= kM) ? k + kM : 0] : 0.0;
        }
      } else {
#pragma unroll
        for (int x = 0; x < kWRow; x++) {
          const int k = x - kM - 7;
          row[x] = (k >= -kM && k <= kM) ? w[(k >= -kM && k <= kM) ? k + kM : 0] : 0.0;
        }
      }
      Cc2[e] = ce;
    }
    cp_async_wait_all();
    __syncthreads();
    // phase 3: every warp accumulates its 8 cells for all nodes of the batch
    for (int e = 0; e < cnt; e++) {
      const int ce = Cc2[e];
      const int o = jw - ce;  // tap index of cell jw
      if (o < -kM - 7 || o > kM) continue;
      const int x = o + kM + 7 + ((ce + 1) & 1);
      const double2* wr = reinterpret_cast<const double2*>(W + e * kWRow + x);
      const double2 w01 = wr[0], w23 = wr[1], w45 = wr[2], w67 = wr[3];
      const double wc[8] = {w01.x, w01.y, w23.x, w23.y, w45.x, w45.y, w67.x, w67.y};
      const double2 fe = F[e];
#pragma unroll
      for (int s = 0; s < SPL; s++) {
        const double2 a = cmul(A[e * SIG + swz(lane + 32 * s, e)], fe);
#pragma unroll
        for (int c = 0; c < kCPW; c++) caxpy(acc[c][s], wc[c], a);
      }
    }
  }
  if (H_ld != 0) {  // batch-minor grid: each cell row is contiguous over the lanes
    const int ncell_w = (int)min((int64_t)kCPW, n - jw);
#pragma unroll
    for (int c = 0; c < kCPW; c++)
#pragma unroll
      for (int s2 = 0; s2 < SPL; s2++) {
        const int64_t b = b0 + lane + 32 * s2;
        if (c < ncell_w && b < H_ld) H[(int64_t)(jw + c) * H_ld + b] = acc[c][s2];
      }
    return;
  }
  // write: stage [cell][signal] then coalesced rows per signal
  __syncthreads();
  double2* O = A;  // reuse (kSpreadCap * SIG >= kSpreadTile * SIG)
#pragma unroll
  for (int c = 0; c < kCPW; c++)
#pragma unroll
    for (int s = 0; s < SPL; s++) {
      const int cell = warp * kCPW + c;
      O[cell * SIG + swz(lane + 32 * s, cell)] = acc[c][s];
    }
  __syncthreads();
  const int ncell = (int)min((int64_t)kSpreadTile, n - j0);
  for (int sig = warp; sig < SIG; sig += kSpreadWarps) {
    const int64_t b = b0 + sig;
    if (b >= batch) break;
    for (int cell = lane; cell < ncell; cell += 32) H[b * n + j0 + cell] = O[cell * SIG + swz(sig, cell)];
  }
}


// Pipelined spreading onto a batch-minor grid H[j * H_ld + b]: one CTA per
// 64-cell tile walks signal groups g = blockIdx.y, blockIdx.y + gridDim.y, ...
// (64 signals each).  Node geometry and the padded weight rows are computed
// once per tile; the amplitudes of group g+1 are fetched with cp.async into
// the second buffer while the FMAs of group g run.  Tiles reached by more
// than kPipeCap nodes (strongly clustered grids) fall back to batching nodes
// per group (weights recomputed), same arithmetic order.
constexpr int kPipeCap = 64;

// SPL = 2 (64-signal groups, two signals per lane): the weight rows, node
// factors and active-node entries a warp loads per node feed twice the FMAs
// (the kernel is bound by the L1's LSU data pipe and by issue slots, not by
// the fp64 pipe).  To keep two CTAs per SM the amplitudes are SINGLE-buffered
// (64 KB per group) — the next group's cp.async copies are issued once every
// warp has finished the FMAs and fly during the stores — and the FMA loop
// takes one node at a time (128 registers).
template <int SPL, bool NB>  // NB: signal-major amplitudes, node-blocked staging layout (swz_nb)
__global__ void __launch_bounds__(256, 2) k_spread_p(const double* __restrict__ ts, const int* __restrict__ perm,
                                                    int64_t Q, int64_t n, double alpha, GaussTab G,
                                                    const double2* __restrict__ amp, int64_t batch, NodeFactor nf,
                                                    double2* __restrict__ H, const int2* __restrict__ ranges, int NS,
                                                    int64_t amp_ld, int64_t H_ld, int ngroups, int sw, int cols,
                                                    int cblk) {
  pdl_enter();  // programmatic dependent launch: wait for the producer grid
  constexpr int SIG = 32 * SPL;
  extern __shared__ __align__(16) unsigned char smraw[];
  double2* A0 = reinterpret_cast<double2*>(smraw);                        // [cap][SIG]
  constexpr bool DB = SPL == 1;                                           // double-buffered amplitudes
  double2* A1 = DB ? A0 + kPipeCap * SIG : A0;                            // [cap][SIG]
  double* W = reinterpret_cast<double*>(A1 + kPipeCap * SIG);             // [cap][kWRow]
  double2* F = reinterpret_cast<double2*>(W + kPipeCap * kWRow);          // [cap]
  int* Cc2 = reinterpret_cast<int*>(F + kPipeCap);                        // [cap]
  int* Pi = Cc2 + kPipeCap;                                               // [cap]
  int* Qs = Pi + kPipeCap;                                                // [cap]
  __shared__ int s_cnt[8];
  __shared__ int s_off[8];

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // sw: slices (signal-group walkers) fastest in the grid, tiles second
  const unsigned bx = sw ? blockIdx.y : blockIdx.x, by = sw ? blockIdx.x : blockIdx.y;
  const unsigned gy = sw ? gridDim.x : gridDim.y;
  const int64_t j0 = (int64_t)bx * kSpreadTile;
  const int jw = (int)j0 + warp * kCPW;
  const int64_t s_lo = floordiv_b(-kM - (min(j0 + kSpreadTile, n) - 1) + n - 1, n);
  if (tid == 0) {
    int acc = 0;
    for (int si = 0; si < NS && si < 8; si++) {
      int2 r = ranges[bx * (int64_t)NS + si];
      s_off[si] = acc;
      s_cnt[si] = r.y - r.x;
      acc += r.y - r.x;
    }
  }
  __syncthreads();
  int total = 0;
  for (int si = 0; si < NS && si < 8; si++) total += s_cnt[si];
  const bool pipelined = total <= kPipeCap;

  // node list (first batch) -> Qs, Pi
  auto node_at = [&](int g, int& si) -> int64_t {
    si = 0;
    while (si + 1 < NS && si + 1 < 8 && g >= s_off[si + 1]) si++;
    return ranges[bx * (int64_t)NS + si].x + (g - s_off[si]);
  };
  // geometry + padded weight rows + factors of nodes [base, base+cnt)
  auto prep_nodes = [&](int base, int cnt) {
    for (int e = tid; e < cnt; e += blockDim.x) {
      int si;
      const int64_t q = node_at(base + e, si);
      Qs[e] = (int)q;
      Pi[e] = perm[q];
      const double t = ts[q];
      const NodeGeo geo = node_geo(t, (double)n);
      const int ce = (int)((int64_t)geo.i0 - (s_lo + si) * n);
      Cc2[e] = ce;
      F[e] = factor_at(nf, q, t);
      double w[2 * kM + 1];
      taps29(geo.f, alpha, G, w);
      double* row = W + e * kWRow;
      if ((ce + 1) & 1) {
#pragma unroll
        for (int x = 0; x < kWRow; x++) {
          const int k = x - 1 - kM - 7;
          row[x] = (k >= -kM && k <= kM) ? w[(k >= -kM && k <= kM) ? k + kM : 0] : 0.0;
        }
      } else {
#pragma unroll
        for (int x = 0; x < kWRow; x++) {
          const int k = x - kM - 7;
          row[x] = (k >= -kM && k <= kM) ? w[(k >= -kM && k <= kM) ? k + kM : 0] : 0.0;
        }
      }
    }
  };
  // async staging of the amplitudes of group g for staged nodes [0, cnt)
  auto stage = [&](double2* A, int64_t g, int cnt) {
    const int64_t b0 = g * SIG;
    if (amp_ld == 0 && SPL == 1) {  // (the node-outer order below measured 5 % slower for 32-signal groups)
      for (int sig = warp; sig < SIG; sig += kSpreadWarps) {
        const int64_t b = b0 + sig;
        const bool ok = b < batch;
        const double2* row = amp + (ok ? b : 0) * Q;
        for (int e = lane; e < cnt; e += 32) cp_async16(&A[swz_nb<SIG>(sig, e)], row + Pi[e], ok);
      }
    } else if (amp_ld == 0) {
      // node = lane, signals warp + 8 k: one caller index, one slot and one base pointer per node;
      // signal sig + 8 sits 64 slots and 8 Q elements further (swz_nb: (sig + 8) & 7 == sig & 7)
      static_assert(kSpreadWarps == 8, "slot stride of the node-blocked layout");
      const int64_t sstep = (int64_t)kSpreadWarps * Q;
      for (int e = lane; e < cnt; e += 32) {
        const double2* src = amp + (b0 + warp) * Q + Pi[e];
        double2* dst = &A[swz_nb<SIG>(warp, e)];
#pragma unroll
        for (int k = 0; k < SIG / kSpreadWarps; k++) {
          const bool ok = b0 + warp + kSpreadWarps * k < batch;
          cp_async16(dst + 64 * k, ok ? src + k * sstep : amp, ok);
        }
      }
    } else {
      for (int e = warp; e < cnt; e += kSpreadWarps) {
        const double2* row = amp + (int64_t)Pi[e] * amp_ld + b0;
#pragma unroll
        for (int s2 = 0; s2 < SPL; s2++) {
          const int sig = lane + 32 * s2;
          const bool ok = b0 + sig < batch;
          cp_async16(&A[e * SIG + sig], row + (ok ? sig : 0), ok);  // lanes = signals: plain rows (no swizzle needed)
        }
      }
    }
    cp_async_commit();
  };
  // this warp's active nodes (window meets its 8 cells), compacted once per
  // staged node set as (node, weight-row offset) pairs so the FMA loop is
  // branch-free and address arithmetic is hoisted out of it
  __shared__ int2 s_act[kSpreadWarps][kPipeCap];
  __shared__ int s_nact[kSpreadWarps];
  auto compact = [&](int cnt) {
    int na = 0;
    for (int e0 = 0; e0 < cnt; e0 += 32) {
      const int e = e0 + lane;
      bool act = false;
      int woff = 0;
      if (e < cnt) {
        const int ce = Cc2[e];
        const int o = jw - ce;
        act = (o >= -kM - 7 && o <= kM);
        woff = e * kWRow + o + kM + 7 + ((ce + 1) & 1);
      }
      const unsigned m = __ballot_sync(0xffffffffu, act);
      if (act) s_act[warp][na + __popc(m & ((1u << lane) - 1u))] = make_int2(e, woff);
      na += __popc(m);
    }
    if (lane == 0) s_nact[warp] = na;
    __syncwarp();
  };
  auto accumulate = [&](const double2* __restrict__ A, int /*cnt*/, double2 (&acc)[kCPW][SPL]) {
    const int na = s_nact[warp];
    const int2* __restrict__ act = s_act[warp];
    int sw[SPL];
#pragma unroll
    for (int s2 = 0; s2 < SPL; s2++) sw[s2] = lane + 32 * s2;
    int k = 0;
    for (; SPL == 1 && k + 1 < na; k += 2) {
      const int2 n0 = act[k], n1 = act[k + 1];
      const double2* w0 = reinterpret_cast<const double2*>(W + n0.y);
      const double2* w1 = reinterpret_cast<const double2*>(W + n1.y);
      const double2 a01 = w0[0], a23 = w0[1], a45 = w0[2], a67 = w0[3];
      const double2 b01 = w1[0], b23 = w1[1], b45 = w1[2], b67 = w1[3];
      const double2 f0 = F[n0.x], f1 = F[n1.x];
      double2 x0[SPL], x1[SPL];
#pragma unroll
      for (int s2 = 0; s2 < SPL; s2++) {
        x0[s2] = A[NB ? swz_nb<SIG>(sw[s2], n0.x) : n0.x * SIG + sw[s2]];
        x1[s2] = A[NB ? swz_nb<SIG>(sw[s2], n1.x) : n1.x * SIG + sw[s2]];
      }
      const double c0[8] = {a01.x, a01.y, a23.x, a23.y, a45.x, a45.y, a67.x, a67.y};
      const double c1[8] = {b01.x, b01.y, b23.x, b23.y, b45.x, b45.y, b67.x, b67.y};
#pragma unroll
      for (int s2 = 0; s2 < SPL; s2++) {
        const double2 y0 = cmul(x0[s2], f0), y1 = cmul(x1[s2], f1);
#pragma unroll
        for (int c = 0; c < kCPW; c++) {
          caxpy(acc[c][s2], c0[c], y0);
          caxpy(acc[c][s2], c1[c], y1);
        }
      }
    }
    for (; k < na; k++) {
      const int2 n0 = act[k];
      const double2* w0 = reinterpret_cast<const double2*>(W + n0.y);
      const double2 a01 = w0[0], a23 = w0[1], a45 = w0[2], a67 = w0[3];
      const double2 f0 = F[n0.x];
      const double c0[8] = {a01.x, a01.y, a23.x, a23.y, a45.x, a45.y, a67.x, a67.y};
#pragma unroll
      for (int s2 = 0; s2 < SPL; s2++) {
        const double2 y0 = cmul(A[NB ? swz_nb<SIG>(sw[s2], n0.x) : n0.x * SIG + sw[s2]], f0);
#pragma unroll
        for (int c = 0; c < kCPW; c++) caxpy(acc[c][s2], c0[c], y0);
      }
    }
  };
  // cols > 0: cell j = i cols + n2 goes to row (n2 / cblk) (L cblk) + i cblk + n2 % cblk, L = n / cols:
  // the columns of the four-step layout in blocks of cblk (cblk = cols: natural order, cblk = 1:
  // every column one contiguous range of L rows)
  const int rows_per_col = cols > 0 ? (int)(n / cols) : 0;
  // rows of this warp's 8 cells, once per CTA (the divisions by the run-time `cols`, `cblk` cost
  // more than a signal group's FMAs when they sit in the store loop)
  int rowc[kCPW];
#pragma unroll
  for (int c = 0; c < kCPW; c++) {
    const int j = jw + c;
    const int n2 = cols > 0 ? j % cols : 0;
    rowc[c] = cols > 0 ? (n2 / cblk) * rows_per_col * cblk + (j / cols) * cblk + n2 % cblk : j;
  }
  auto store = [&](int64_t g, double2 (&acc)[kCPW][SPL]) {
    const int ncell_w = (int)min((int64_t)kCPW, n - jw);
#pragma unroll
    for (int c = 0; c < kCPW; c++) {
#pragma unroll
      for (int s2 = 0; s2 < SPL; s2++) {
        const int64_t b = g * SIG + lane + 32 * s2;
        if (c < ncell_w && b < H_ld) H[(int64_t)rowc[c] * H_ld + b] = acc[c][s2];
      }
    }
  };

  if (pipelined) {
    prep_nodes(0, total);
    __syncthreads();
    compact(total);
    int64_t g = by;
    if (g < ngroups) stage(A0, g, total);
    if constexpr (!DB) {
      for (; g < ngroups; g += gy) {
        cp_async_wait_group<0>();
        __syncthreads();
        double2 acc[kCPW][SPL];
#pragma unroll
        for (int c = 0; c < kCPW; c++)
#pragma unroll
          for (int s2 = 0; s2 < SPL; s2++) acc[c][s2] = make_double2(0.0, 0.0);
        accumulate(A0, total, acc);
        __syncthreads();  // every warp has consumed A0: refill it while the results are stored
        if (g + gy < ngroups) stage(A0, g + gy, total);
        store(g, acc);
      }
    } else
    for (int it = 0; g < ngroups; it++, g += gy) {
      double2* cur = (it & 1) ? A1 : A0;
      double2* nxt = (it & 1) ? A0 : A1;
      if (g + gy < ngroups) {
        stage(nxt, g + gy, total);
        cp_async_wait_group<1>();
      } else {
        cp_async_wait_group<0>();
      }
      __syncthreads();
      double2 acc[kCPW][SPL];
#pragma unroll
      for (int c = 0; c < kCPW; c++)
#pragma unroll
        for (int s2 = 0; s2 < SPL; s2++) acc[c][s2] = make_double2(0.0, 0.0);
      accumulate(cur, total, acc);
      store(g, acc);
      __syncthreads();  // `cur` is refilled two iterations later
    }
  } else {
    for (int64_t g = by; g < ngroups; g += gy) {
      double2 acc[kCPW][SPL];
#pragma unroll
      for (int c = 0; c < kCPW; c++)
#pragma unroll
        for (int s2 = 0; s2 < SPL; s2++) acc[c][s2] = make_double2(0.0, 0.0);
      for (int base = 0; base < total; base += kPipeCap) {
        const int cnt = min(kPipeCap, total - base);
        __syncthreads();
        prep_nodes(base, cnt);
        __syncthreads();
        compact(cnt);
        stage(A0, g, cnt);
        cp_async_wait_group<0>();
        __syncthreads();
        accumulate(A0, cnt, acc);
      }
      store(g, acc);
    }
  }
}

int spread_pipelined(const GridDev& g, int64_t n, const Window& win, const double2* amp, int64_t batch,
                     int64_t amp_ld, NodeFactor f, double2* H, int64_t H_ld, cudaStream_t st, int64_t cols, int cblk) {
  const int64_t ntiles = ceil_div(n, kSpreadTile);
  const int NS = tile_images(n, win.m, kSpreadTile);
  if (NS > 8) return NFFT45_ERR_INVALID_ARGUMENT;
  const int2* ranges = nullptr;
  int2* own = nullptr;
  NFFT_CHECK(tile_ranges(g, n, win.m, kSpreadTile, NS, st, &ranges, &own));
  // 64-signal groups (two signals per lane, single-buffered amplitudes) from 128 signals up: measured
  // -7.6 % at 1024 signals, -6 % at 512, -7 % at 128 / 192, +2 % at 64; NFFT45_SPREAD_SPL=1|2 forces
  static const int spl_env = getenv("NFFT45_SPREAD_SPL") ? atoi(getenv("NFFT45_SPREAD_SPL")) : 0;
  const int spl = spl_env == 1 || spl_env == 2 ? spl_env : (H_ld >= 128 ? 2 : 1);
  const int SIG = 32 * spl;
  const int ngroups = (int)ceil_div(H_ld, SIG);
  // enough CTAs for ~2 waves of 148 SMs, each walking several signal groups
  int slices = (int)std::min<int64_t>(ngroups, std::max<int64_t>(1, ceil_div(4 * 148, ntiles)));
  static const int env_sl = getenv("NFFT45_SPREAD_SLICES") ? atoi(getenv("NFFT45_SPREAD_SLICES")) : 0;
  const int sw = env_sl > 0;
  if (env_sl > 0) slices = (int)std::min<int64_t>(ngroups, env_sl);
  size_t smem = (size_t)(spl == 1 ? 2 : 1) * kPipeCap * SIG * 16 + (size_t)kPipeCap * kWRow * 8 + kPipeCap * 16 + kPipeCap * 16;
  auto spread_p = amp_ld == 0 ? k_spread_p<1, true> : k_spread_p<1, false>;
  if (spl == 2) spread_p = amp_ld == 0 ? k_spread_p<2, true> : k_spread_p<2, false>;
  NFFT_CUDA(cudaFuncSetAttribute(spread_p, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const dim3 grid = sw ? dim3((unsigned)slices, (unsigned)ntiles) : dim3((unsigned)ntiles, (unsigned)slices);
  LAUNCH_PDL(spread_p, grid, 256, smem, st, g.ts, g.perm, g.Q, n, win.alpha, gauss_tab(win), amp, batch, f, H, ranges,
         NS, amp_ld, H_ld, ngroups, sw, (int)cols, cblk);
  if (own) NFFT_CUDA(cudaFreeAsync(own, st));
  return NFFT45_OK;
}

int spread_batched(const GridDev& g, int64_t n, const Window& win, const double2* amp, int64_t batch, NodeFactor f,
                   double2* H, cudaStream_t st, int spl, int64_t amp_ld, int64_t H_ld) {
  const int64_t ntiles = ceil_div(n, kSpreadTile);
  const int NS = tile_images(n, win.m, kSpreadTile);
  if (NS > 8) return NFFT45_ERR_INVALID_ARGUMENT;  // tiny grids use the generic kernel
  const int2* ranges = nullptr;
  int2* own = nullptr;
  NFFT_CHECK(tile_ranges(g, n, win.m, kSpreadTile, NS, st, &ranges, &own));
  GaussTab G = gauss_tab(win);
  if (spl == 2) {
    constexpr int SIG = 64;
    size_t smem = (size_t)kSpreadCap * SIG * 16 + (size_t)kSpreadCap * kWRow * 8 + kSpreadCap * 16 + kSpreadCap * 16;
    auto spread_b = k_spread_b<2>;
    NFFT_CUDA(cudaFuncSetAttribute(spread_b, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    dim3 grid((unsigned)ntiles, (unsigned)ceil_div(batch, SIG));
    LAUNCH(spread_b, grid, 256, smem, st, g.ts, g.perm, g.Q, n, win.alpha, G, amp, batch, f, H, ranges, NS, amp_ld,
           H_ld);
  } else {
    constexpr int SIG = 32;
    size_t smem = (size_t)kSpreadCap * SIG * 16 + (size_t)kSpreadCap * kWRow * 8 + kSpreadCap * 16 + kSpreadCap * 16;
    auto spread_b = k_spread_b<1>;
    NFFT_CUDA(cudaFuncSetAttribute(spread_b, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    dim3 grid((unsigned)ntiles, (unsigned)ceil_div(batch, SIG));
    LAUNCH(spread_b, grid, 256, smem, st, g.ts, g.perm, g.Q, n, win.alpha, G, amp, batch, f, H, ranges, NS, amp_ld,
           H_ld);
  }
  if (own) NFFT_CUDA(cudaFreeAsync(own, st));
  return NFFT45_OK;
}

// ------------------------------------------------------------- gather

// CTA: 32 consecutive ascending nodes x 32 signals (lane = signal); warp w
// owns nodes 8w..8w+7.  The cells under the CTA's windows are staged as
// [cell][signal] in chunks of kGatherSpan; each warp builds a dense weight
// table WT[cell][8 nodes] for its own cells (zeros outside windows) so one
// staged cell value feeds 8 FMAs with one 64-byte broadcast of weights.
template <bool BM>
__device__ __forceinline__ void gather_b_tile(const double* __restrict__ ts, const int* __restrict__ perm, int64_t Q,
                                              int64_t n, double alpha, GaussTab G, const double2* __restrict__ H,
                                              int64_t batch, NodeFactor nf, const double2* __restrict__ sub, int mode,
                                              double2* __restrict__ out, int64_t H_ld, int64_t sub_ld, int64_t out_ld,
                                              const int64_t b0) {
  // *_ld == 0: signal-major operand ([batch][len]); else batch-minor x[i * ld + b]
  constexpr int SIG = 32;
  extern __shared__ __align__(16) unsigned char smraw[];
  double2* Y = reinterpret_cast<double2*>(smraw);                                // [span][SIG]
  double* WT = reinterpret_cast<double*>(Y + kGatherSpan * SIG);                 // [warps][kWTSpan][8]
  double2* Sb = reinterpret_cast<double2*>(WT + kGatherWarps * kWTSpan * kNPW);  // [nodes][SIG] subtrahend
  __shared__ int s_c0[kGatherNodes];
  __shared__ double s_f[kGatherNodes];
  __shared__ double2 s_fac[kGatherNodes];
  __shared__ int s_pq[kGatherNodes];

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t q0 = (int64_t)blockIdx.x * kGatherNodes;
  const int nq = (int)min((int64_t)kGatherNodes, Q - q0);

  if (tid < kGatherNodes) {
    int c = 0;
    double f = 0.0;
    if (tid < nq) {
      const double t = ts[q0 + tid];
      NodeGeo geo = node_geo(t, (double)n);
      c = geo.i0;
      f = geo.f;
      s_fac[tid] = factor_at(nf, q0 + tid, t);
      s_pq[tid] = perm[q0 + tid];
    } else if (nq > 0) {
      NodeGeo geo = node_geo(ts[q0 + nq - 1], (double)n);
      c = geo.i0;
    }
    s_c0[tid] = c;
    s_f[tid] = f;
  }
  __syncthreads();
  // subtrahend tile, read in the order that is coalesced for its layout
  if (mode != 0) {
    if (sub_ld == 0) {
      for (int sig = warp; sig < SIG; sig += kGatherWarps) {
        const int64_t b = b0 + sig;
        const bool ok = b < batch;
        for (int e = lane; e < nq; e += 32)
          cp_async16(&Sb[e * SIG + swz(sig, e)], sub + (ok ? b : 0) * Q + s_pq[e], ok);
      }
    } else {
      for (int e = warp; e < nq; e += kGatherWarps) {
        const bool ok = b0 + lane < batch;
        cp_async16(&Sb[e * SIG + swz(lane, e)], sub + (int64_t)s_pq[e] * sub_ld + b0 + (ok ? lane : 0), ok);
      }
    }
  }
  // unwrapped cell span of the CTA and of this warp (centres ascend)
  const int cta_lo = s_c0[0] - kM, cta_hi = s_c0[kGatherNodes - 1] + kM;
  const int w_lo = s_c0[warp * kNPW] - kM, w_hi = s_c0[warp * kNPW + kNPW - 1] + kM;
  double* wt = WT + warp * kWTSpan * kNPW;

  double2 acc[kNPW];
#pragma unroll
  for (int i = 0; i < kNPW; i++) acc[i] = make_double2(0.0, 0.0);

  for (int cs = cta_lo; cs <= cta_hi; cs += kGatherSpan) {
    const int ce = min(cs + kGatherSpan - 1, cta_hi);
    const int len = ce - cs + 1;
    __syncthreads();  // previous chunk fully consumed
    // stage cells [cs, ce] (mod n) for the CTA's signals
    // cell index mod n: one conditional add/sub when the chunk spans less
    // than a period (always, except tiny grids which take the full reduction)
    const int ni = (int)n;
    const bool small = n < (int64_t)kGatherSpan + 2 * kM + 2;
    auto wrap = [&](int cell) -> int {
      if (small) {
        cell %= ni;
        return cell < 0 ? cell + ni : cell;
      }
      return cell < 0 ? cell + ni : (cell >= ni ? cell - ni : cell);
    };
    if constexpr (!BM) {
      for (int sig = warp; sig < SIG; sig += kGatherWarps) {
        const int64_t b = b0 + sig;
        const bool ok = b < batch;
        const double2* row = H + (ok ? b : 0) * n;
        for (int c = lane; c < len; c += 32) cp_async16(&Y[c * SIG + swz(sig, c)], row + wrap(cs + c), ok);
      }
    } else {
      const bool ok = b0 + lane < batch;
      const double2* col = H + b0 + (ok ? lane : 0);
      for (int c = warp; c < len; c += kGatherWarps)
        cp_async16(&Y[c * SIG + lane], col + (int64_t)wrap(cs + c) * H_ld, ok);
    }
    // this warp's cells inside the chunk, in sub-chunks of kWTSpan (warp-private
    // table); the first table is built while the copies are in flight
    const int a_lo = max(w_lo, cs), a_hi = min(w_hi, ce);
    auto build = [&](int ws, int we) {
      const int wl = we - ws + 1;
      __syncwarp();
      for (int i = lane; i < wl * kNPW; i += 32) wt[i] = 0.0;
      __syncwarp();
      if (lane < kNPW && warp * kNPW + lane < nq) {
        double w[2 * kM + 1];
        taps29(s_f[warp * kNPW + lane], alpha, G, w);
        const int c0 = s_c0[warp * kNPW + lane] - kM;
#pragma unroll
        for (int k = 0; k < 2 * kM + 1; k++) {
          const int c = c0 + k;
          if (c >= ws && c <= we) wt[(c - ws) * kNPW + lane] = w[k];
        }
      }
      __syncwarp();
    };
    if (a_lo <= a_hi) build(a_lo, min(a_lo + kWTSpan - 1, a_hi));
    cp_async_wait_all();
    __syncthreads();
    for (int ws = a_lo; ws <= a_hi; ws += kWTSpan) {
      const int we = min(ws + kWTSpan - 1, a_hi);
      if (ws != a_lo) build(ws, we);
      const double2* __restrict__ yrow = Y + (ws - cs) * SIG;
      const double2* __restrict__ wrow = reinterpret_cast<const double2*>(wt);
      const int nc = we - ws + 1;
#pragma unroll 4
      for (int i = 0; i < nc; i++) {
        const int r = ws - cs + i;
        const double2 y = BM ? yrow[i * SIG + lane] : Y[r * SIG + swz(lane, r)];
        const double2* wr = wrow + i * (kNPW / 2);
#pragma unroll
        for (int i2 = 0; i2 < kNPW / 2; i2++) {
          const double2 w = wr[i2];
          caxpy(acc[2 * i2], w.x, y);
          caxpy(acc[2 * i2 + 1], w.y, y);
        }
      }
    }
  }
  // epilogue: factor, optional subtraction, store in the output's coalesced order
  __syncthreads();
  double2* O = Y;  // [node][SIG]
#pragma unroll
  for (int i = 0; i < kNPW; i++) {
    const int e = warp * kNPW + i;
    O[e * SIG + swz(lane, e)] = acc[i];
  }
  __syncthreads();
  auto value = [&](int e, int sig) -> double2 {
    double2 v = cmul(O[e * SIG + swz(sig, e)], s_fac[e]);
    if (mode == 1) v = csub(v, Sb[e * SIG + swz(sig, e)]);
    else if (mode == 2) v = csub(Sb[e * SIG + swz(sig, e)], v);
    return v;
  };
  if (out_ld == 0) {
    for (int idx = tid; idx < kGatherNodes * SIG; idx += blockDim.x) {
      const int e = idx & (kGatherNodes - 1), sig = idx / kGatherNodes;
      const int64_t b = b0 + sig;
      if (b >= batch || e >= nq) continue;
      out[b * Q + s_pq[e]] = value(e, sig);
    }
  } else {
    for (int e = warp; e < nq; e += kGatherWarps) {
      const int64_t b = b0 + lane;
      if (b < out_ld) out[(int64_t)s_pq[e] * out_ld + b] = b < batch ? value(e, lane) : make_double2(0.0, 0.0);
    }
  }
}



template <bool BM>
__global__ void __launch_bounds__(kGatherWarps * 32, 2) k_gather_b(const double* __restrict__ ts, const int* __restrict__ perm,
                                                    int64_t Q, int64_t n, double alpha, GaussTab G,
                                                    const double2* __restrict__ H, int64_t batch, NodeFactor nf,
                                                    const double2* __restrict__ sub, int mode,
                                                    double2* __restrict__ out, int64_t H_ld, int64_t sub_ld,
                                                    int64_t out_ld, const int* __restrict__ only, int ny) {
  pdl_enter();  // programmatic dependent launch: wait for the producer grid
  // only != nullptr: process just the node blocks flagged there (fallback use;
  // launched with one CTA row that walks all ny signal groups)
  if (only && !only[blockIdx.x]) return;
  for (int gy = blockIdx.y; gy < ny; gy += gridDim.y) {
    if (gy != (int)blockIdx.y) __syncthreads();  // shared tiles are reused
    gather_b_tile<BM>(ts, perm, Q, n, alpha, G, H, batch, nf, sub, mode, out, H_ld, sub_ld, out_ld, (int64_t)gy * 32);
  }
}

int gather_fallback(const GridDev& g, int64_t n, const Window& win, const double2* H, int64_t batch, NodeFactor f,
                    const double2* sub, int mode, double2* out, cudaStream_t st, int64_t H_ld, int64_t sub_ld,
                    int64_t out_ld, const int* only);

// Persistent interpolation from a batch-minor grid H[j * H_ld + b]: one CTA
// per block of 32 ascending nodes (4 warps x 8) walks the signal groups
// g = blockIdx.y, blockIdx.y + gridDim.y, ...  Node geometry and the
// per-warp weight tables WT[cell][8 nodes] are built once per block; the
// next group's cells are fetched with cp.async while the current group's
// results are finished.  Batch-minor outputs / subtrahends go straight
// between registers and global memory (lane = signal); signal-major ones are
// transposed through shared memory.  Blocks whose cell span exceeds the
// staging buffer (strongly clustered grids) return early and are handled by
// k_gather_b (host passes `fallback` so those blocks are recomputed there).
constexpr int kGPSpan = 112;
constexpr int kGPSpanS = 96;  // short TMA box (rows)

// SIG signals per group (16 or 32).  With SIG = 16 the two half-warps take
// 4 nodes each of the warp's 8 (same cells, broadcast reads), which halves
// the staging tile so 4 CTAs fit per SM.
// WARPS = 8 (with SIG = 32): 4 nodes per warp, lane = signal -- per staged
// cell row a warp issues 3 LDS.128 (one 512-byte row of cells, two broadcast
// weight pairs) for 8 DFMA pairs, against 3 LDS.128 per 4 DFMA pairs per
// half-warp in the 16-signal layout, and the dense weight table of 4 nodes
// has 83 % non-zero entries instead of 67 % for 8 nodes: the kernel is bound
// by the L1's LSU data pipe, so both count.  8 warps per CTA keep 16-24 warps
// per SM although the 32-signal cell tile is twice as large.
template <int SIG, int WARPS>
__host__ __device__ constexpr int gp_min_ctas(int subm, bool out_bm) {
  if (WARPS == 8) return subm == 2 ? 2 : 3;  // (signal-major outputs transpose through the consumed cell tile)
  return SIG == 32 ? 2 : (SIG == 16 ? 4 : 5);
}
template <bool OUT_BM, int SUBM, int SIG, int WARPS = kGatherWarps>  // SUBM: 0 none, 1 batch-minor, 2 signal-major
__global__ void __launch_bounds__(WARPS * 32, gp_min_ctas<SIG, WARPS>(SUBM, OUT_BM)) k_gather_p(
    const double* __restrict__ ts, const int* __restrict__ perm, int64_t Q, int64_t n, double alpha, GaussTab G,
    const double2* __restrict__ H, int64_t H_ld, int64_t batch, NodeFactor nf, const double2* __restrict__ sub,
    int64_t sub_ld, int mode, double2* __restrict__ out, int64_t out_ld, int ngroups, int* __restrict__ overflow, int sw,
    const __grid_constant__ CUtensorMap tmH, const __grid_constant__ CUtensorMap tmHs, int tma) {
  pdl_enter();  // programmatic dependent launch: wait for the producer grid
  constexpr int NPW = kGatherNodes / WARPS;  // nodes per warp
  constexpr int HALVES = 32 / SIG, NPL = NPW / HALVES;
  static_assert(kGatherNodes == 32, "one node per lane in the signal-major staging");
  static_assert(NPL >= 2 && NPL % 2 == 0 && SIG % WARPS == 0, "weight pairs per lane; signals per warp in the transposes");
  extern __shared__ __align__(128) unsigned char smraw_gp[];  // own symbol: 128-byte aligned for the TMA box
  __shared__ __align__(8) uint64_t s_bar;  // TMA completion (transaction count) of the staged cell tile
  double2* Y = reinterpret_cast<double2*>(smraw_gp);                     // [kGPSpan][SIG]
  double* WT = reinterpret_cast<double*>(Y + kGPSpan * SIG);           // [warps][kWTSpan][8]
  double2* Sb = reinterpret_cast<double2*>(WT + WARPS * kWTSpan * NPW);  // [nodes][SIG] (SUBM == 2)
  // [nodes][SIG] transpose tile of signal-major outputs.  With 8 warps it is the (consumed) head of
  // the cell tile and the next group's prefetch waits for the stores: 73 KB per CTA, 3 CTAs per SM.
  constexpr bool O_IN_Y = !OUT_BM && WARPS == 8;
  double2* O = O_IN_Y ? Y : Sb + (SUBM == 2 ? kGatherNodes * SIG : 0);
  __shared__ int s_c0[kGatherNodes];
  __shared__ double s_f[kGatherNodes];
  __shared__ double2 s_fac[kGatherNodes];
  __shared__ int s_pq[kGatherNodes];

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
    mbar_init(&s_bar, 1);
    mbar_fence_init();
  }
  // sw: slices (signal-group walkers) fastest in the grid, node blocks second
  const unsigned bx = sw ? blockIdx.y : blockIdx.x, by = sw ? blockIdx.x : blockIdx.y;
  const unsigned gy = sw ? gridDim.x : gridDim.y;
  const int sl = lane % SIG, hf = lane / SIG;
  const int64_t q0 = (int64_t)bx * kGatherNodes;
  const int nq = (int)min((int64_t)kGatherNodes, Q - q0);
  if (tid < kGatherNodes) {
    const int e = tid < nq ? tid : nq - 1;
    const double t = ts[q0 + e];
    const NodeGeo geo = node_geo(t, (double)n);
    s_c0[tid] = geo.i0;
    s_f[tid] = tid < nq ? geo.f : 0.0;
    if (tid < nq) {
      s_fac[tid] = factor_at(nf, q0 + tid, t);
      s_pq[tid] = perm[q0 + tid];
    }
  }
  __syncthreads();
  const int cs = s_c0[0] - kM, ce = s_c0[kGatherNodes - 1] + kM;
  const int len = ce - cs + 1;
  const int w_lo = s_c0[warp * NPW] - kM, w_hi = s_c0[warp * NPW + NPW - 1] + kM;
  if (len > kGPSpan || w_hi - w_lo + 1 > kWTSpan || n < (int64_t)kGPSpan + 2 * kM + 2) {
    if (tid == 0 && by == 0) overflow[bx] = 1;  // handled by the fallback kernel
    return;
  }
  // per-warp dense weight table over the warp's cells, built once
  double* wt = WT + warp * kWTSpan * NPW;
  const int wl = w_hi - w_lo + 1;
  const int ni = (int)n;
  // signal-major operands: this thread's node (lane) and first signal (warp)
  const int64_t my_off = (int64_t)warp * Q + (lane < nq ? s_pq[lane] : 0);  // signals warp + WARPS k
  const double2* sb_src = sub + my_off;
  // Cell tile of a signal group: ONE bulk tensor copy (TMA, SASS UTMALDG)
  // issued by thread 0 when the block's cell span does not wrap around the
  // period -- the copy bypasses the LSU data pipe, which bounds this kernel
  // (an LDGSTS costs twice the pipe cycles of an LDS of the same bytes); rows
  // past the block's span and signals past the padded batch arrive as zeros /
  // unused rows.  Blocks that wrap keep the per-thread cp.async copies.
  const bool tma_blk = tma && cs >= 0 && ce < ni;
  // two boxes: kGPSpanS rows cover the span of most blocks (29 + 31 node gaps), kGPSpan rows the rest
  const bool box_s = len <= kGPSpanS;
  const unsigned kBoxBytes = (unsigned)((box_s ? kGPSpanS : kGPSpan) * SIG * sizeof(double2));
  auto stage = [&](int64_t g) {
    const int64_t b0 = g * SIG;
    if (tma_blk) {
      if (tid == 0) {
        fence_proxy_async();  // the previous group's generic reads of Y precede the async refill
        mbar_expect_tx(&s_bar, kBoxBytes);
        tma_load_2d(Y, box_s ? &tmHs : &tmH, (int)(2 * b0), cs, &s_bar);
      }
    } else {
      const bool ok = b0 + sl < batch;
      const double2* col = H + b0 + (ok ? sl : 0);
      for (int c = warp * HALVES + hf; c < len; c += WARPS * HALVES) {
        int cell = cs + c;
        cell = cell < 0 ? cell + ni : (cell >= ni ? cell - ni : cell);
        cp_async16(&Y[c * SIG + sl], col + (int64_t)cell * H_ld, ok);
      }
    }
    if (SUBM == 2 && mode != 0) {  // node = lane, signals warp + 4k: one base pointer, stride 4Q
#pragma unroll
      for (int k = 0; k < SIG / WARPS; k++) {
        const int sig = warp + WARPS * k;
        const bool okb = b0 + sig < batch && lane < nq;
        cp_async16(&Sb[swz_nb<SIG>(sig, lane)], sb_src + (okb ? (b0 + WARPS * k) * Q : 0), okb);
      }
    }
    cp_async_commit();
  };
  int64_t g = by;
  if (g < ngroups) stage(g);
  // (built while the first group's cell tile is in flight)
  for (int i = lane; i < wl * NPW; i += 32) wt[i] = 0.0;
  __syncwarp();
  if (lane < NPW && warp * NPW + lane < nq) {
    double w[2 * kM + 1];
    taps29(s_f[warp * NPW + lane], alpha, G, w);
    const int c0 = s_c0[warp * NPW + lane] - kM - w_lo;
#pragma unroll
    for (int k = 0; k < 2 * kM + 1; k++) wt[(c0 + k) * NPW + lane] = w[k];
  }
  __syncwarp();
  const double2* __restrict__ yw = Y + (w_lo - cs) * SIG + sl;
  const double2* __restrict__ wr0 = reinterpret_cast<const double2*>(wt) + hf * (NPL / 2);
  const int e0 = warp * NPW + hf * NPL;  // node of acc[0]
  unsigned phase = 0;
  for (; g < ngroups; g += gy) {
    const int64_t b0 = g * SIG;
    cp_async_wait_group<0>();
    if (tma_blk) {
      mbar_wait(&s_bar, phase);
      phase ^= 1u;
    }
    __syncthreads();
    double2 acc[NPL];
#pragma unroll
    for (int i = 0; i < NPL; i++) acc[i] = make_double2(0.0, 0.0);
    // batch-minor subtrahend: requested before the window sums so its latency
    // hides under them (it is only consumed by the epilogue)
    double2 sb_in[NPL];
    if (SUBM == 1 && mode != 0) {
#pragma unroll
      for (int i = 0; i < NPL; i++) {
        const int e = e0 + i;
        const bool ok = e < nq && b0 + sl < batch;
        sb_in[i] = ok ? sub[(int64_t)s_pq[e] * sub_ld + b0 + sl] : make_double2(0.0, 0.0);
      }
    }
#pragma unroll 4
    for (int i = 0; i < wl; i++) {
      const double2 y = yw[i * SIG];
      const double2* wr = wr0 + i * (NPW / 2);
#pragma unroll
      for (int i2 = 0; i2 < NPL / 2; i2++) {
        const double2 w = wr[i2];
        caxpy(acc[2 * i2], w.x, y);
        caxpy(acc[2 * i2 + 1], w.y, y);
      }
    }
    if (SUBM == 2 && mode != 0) {
#pragma unroll
      for (int i = 0; i < NPL; i++) {
        const int e = e0 + i;
        sb_in[i] = e < nq ? Sb[swz_nb<SIG>(sl, e)] : make_double2(0.0, 0.0);
      }
    }
    __syncthreads();  // Y (and Sb) consumed: prefetch the next group during the epilogue
    if (!O_IN_Y && g + gy < ngroups) stage(g + gy);
    if constexpr (OUT_BM) {
      const int64_t b = b0 + sl;
#pragma unroll
      for (int i = 0; i < NPL; i++) {
        const int e = e0 + i;
        if (e >= nq || b >= out_ld) continue;
        double2 v = cmul(acc[i], s_fac[e]);
        const int64_t pq = s_pq[e];
        if (b < batch && mode != 0) {
          const double2 sv = sb_in[i];
          v = mode == 1 ? csub(v, sv) : csub(sv, v);
        }
        out[pq * out_ld + b] = b < batch ? v : make_double2(0.0, 0.0);
      }
    } else {
#pragma unroll
      for (int i = 0; i < NPL; i++) {
        const int e = e0 + i;
        double2 v = cmul(acc[i], e < nq ? s_fac[e] : make_double2(0.0, 0.0));
        if (mode != 0 && e < nq && b0 + sl < batch) {
          const double2 sv = sb_in[i];
          v = mode == 1 ? csub(v, sv) : csub(sv, v);
        }
        O[e * SIG + swz(sl, e)] = v;
      }
      __syncthreads();
      double2* dst = out + my_off + b0 * Q;
#pragma unroll
      for (int k = 0; k < SIG / WARPS; k++) {
        const int sig = warp + WARPS * k;
        if (b0 + sig < batch && lane < nq) dst[(int64_t)WARPS * k * Q] = O[lane * SIG + swz(sig, lane)];
      }
      if constexpr (O_IN_Y) {
        __syncthreads();  // the transpose tile is drained: refill the cell tile
        if (g + gy < ngroups) stage(g + gy);
      }
    }
  }
}

// Node blocks that k_gather_p cannot stage (same condition as its early
// return): a property of the node set and n only, so it is computed once per
// plan and the fallback launch is skipped when no block overflows.
__global__ void k_gather_flags(const double* __restrict__ ts, int64_t Q, int64_t n, int64_t nblk,
                               int* __restrict__ flags, int* __restrict__ any) {
  const int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (b >= nblk) return;
  const int64_t q0 = b * kGatherNodes;
  const int nq = (int)min((int64_t)kGatherNodes, Q - q0);
  auto c0 = [&](int e) { return node_geo(ts[q0 + (e < nq ? e : nq - 1)], (double)n).i0; };
  bool of = (int64_t)(c0(kGatherNodes - 1) + kM) - (c0(0) - kM) + 1 > kGPSpan || n < (int64_t)kGPSpan + 2 * kM + 2;
  for (int w = 0; w < kGatherWarps; w++)
    of = of || (c0(w * kNPW + kNPW - 1) + kM) - (c0(w * kNPW) - kM) + 1 > kWTSpan;
  flags[b] = of ? 1 : 0;
  if (of) atomicOr(any, 1);
}

int gather_flags_compute(const GridDev& g, int64_t n, int* flags, int* any, cudaStream_t st) {
  const int64_t nblk = ceil_div(g.Q, kGatherNodes);
  NFFT_CUDA(cudaMemsetAsync(any, 0, sizeof(int), st));
  LAUNCH(k_gather_flags, (unsigned)ceil_div(nblk, 128), 128, 0, st, g.ts, g.Q, n, nblk, flags, any);
  return NFFT45_OK;
}

int64_t gather_blocks(int64_t Q) { return ceil_div(Q, kGatherNodes); }

__global__ void k_overflow_clear(int* f, int64_t n) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) f[i] = 0;
}

// 32-signal groups waste lanes on the last group of small batches; measured faster from 32 signals up
// once a walker keeps 8 or more groups (see `slices`), equal at 48: the default from 64 signals
static bool gather_w8_default(int64_t nsig) {
  static const int64_t min_sig = getenv("NFFT45_GATHER_W8_MIN") ? atoll(getenv("NFFT45_GATHER_W8_MIN")) : 64;
  return nsig >= min_sig;
}

int gather_persistent(const GridDev& g, int64_t n, const Window& win, const double2* H, int64_t H_ld, int64_t batch,
                      NodeFactor f, const double2* sub, int64_t sub_ld, int mode, double2* out, int64_t out_ld,
                      cudaStream_t st) {
  if (!sub) mode = 0;
  static const int SIG = [] {  // signals per group (A/B switch NFFT45_GATHER_SIG = 8 | 16 | 32)
    const char* e = getenv("NFFT45_GATHER_SIG");
    const int v = e ? atoi(e) : 16;
    return v == 8 || v == 32 ? v : 16;
  }();
  // 8 warps x 4 nodes with 32-signal groups (default); NFFT45_GATHER_WARPS=4: the 4-warp layouts
  static const int env_w = getenv("NFFT45_GATHER_WARPS") ? atoi(getenv("NFFT45_GATHER_WARPS")) : 0;
  static const bool sig_env = getenv("NFFT45_GATHER_SIG") != nullptr;
  const bool w8 = env_w == 8 || (env_w == 0 && !sig_env && gather_w8_default(out_ld ? out_ld : batch));
  const int SIGu = w8 ? 32 : SIG;
  const int WARPSu = w8 ? 8 : kGatherWarps;
  const int64_t nblk = ceil_div(g.Q, kGatherNodes);
  const int ngroups = (int)ceil_div(out_ld ? out_ld : batch, SIGu);
  // at least 4 signal-group walkers per node block, walkers fastest in the
  // grid (concurrent CTAs then read 4 groups of each cell row: -4 % on C4)
  // (the 8-warp layout wants its per-block setup amortised over 8 or more groups: one or two walkers)
  int slices = (int)std::min<int64_t>(
      ngroups, std::max<int64_t>(w8 ? std::max(1, std::min(2, ngroups / 8)) : 4, ceil_div(4 * 148, nblk)));
  static const int env_sl = getenv("NFFT45_GATHER_SLICES") ? atoi(getenv("NFFT45_GATHER_SLICES")) : 0;
  const int sw = 1;
  if (env_sl > 0) slices = (int)std::min<int64_t>(ngroups, env_sl);
  // overflow flags: the plan's precomputed table (fallback launched only if
  // some block overflows), else a per-call table filled by the kernel
  int* overflow = nullptr;
  bool cached_any = true;
  const bool cached = gather_flags_lookup(g, n, &overflow, &cached_any);
  if (!cached) {
    NFFT_CUDA(cudaMallocAsync(&overflow, sizeof(int) * nblk, st));
    LAUNCH(k_overflow_clear, (unsigned)ceil_div(nblk, 256), 256, 0, st, overflow, nblk);
  }
  const int subm = mode == 0 ? 0 : (sub_ld ? 1 : 2);
  size_t smem = (size_t)kGPSpan * SIGu * 16 + (size_t)kGatherWarps * kWTSpan * kNPW * 8 +
                (subm == 2 ? (size_t)kGatherNodes * SIGu * 16 : 0) +
                (out_ld || WARPSu == 8 ? 0 : (size_t)kGatherNodes * SIGu * 16);
  const dim3 grid = sw ? dim3((unsigned)slices, (unsigned)nblk) : dim3((unsigned)nblk, (unsigned)slices);
  GaussTab G = gauss_tab(win);
  // TMA-staged cell tiles (NFFT45_GATHER_TMA=0: per-thread cp.async copies, for A/B runs)
  static const int use_tma = !(getenv("NFFT45_GATHER_TMA") && atoi(getenv("NFFT45_GATHER_TMA")) == 0);
  CUtensorMap tmH;
  memset(&tmH, 0, sizeof(tmH));
  int tma = use_tma && (reinterpret_cast<uintptr_t>(H) % 16 == 0) && n >= kGPSpan;
  CUtensorMap tmHs;
  memset(&tmHs, 0, sizeof(tmHs));
  if (tma) NFFT_CHECK(tma_map_rows(&tmH, H, n, H_ld, kGPSpan, SIGu));
  if (tma) NFFT_CHECK(tma_map_rows(&tmHs, H, n, H_ld, kGPSpanS, SIGu));
#define NFFT_GP_LAUNCH(OBM, SM_, S_, W_)                                                                       \
  {                                                                                                          \
    auto gather_p = k_gather_p<OBM, SM_, S_, W_>;                                                            \
    NFFT_CUDA(cudaFuncSetAttribute(gather_p, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));       \
    LAUNCH_PDL(gather_p, grid, W_ * 32, smem, st, g.ts, g.perm, g.Q, n, win.alpha, G, H, H_ld, batch, f,     \
           sub, sub_ld, mode, out, out_ld, ngroups, overflow, sw, tmH, tmHs, tma);                           \
  }
#define NFFT_GP_SUBW(OBM, S_, W_) \
  if (subm == 0) NFFT_GP_LAUNCH(OBM, 0, S_, W_) else if (subm == 1) NFFT_GP_LAUNCH(OBM, 1, S_, W_) else NFFT_GP_LAUNCH(OBM, 2, S_, W_)
#define NFFT_GP_SUB(OBM, S_) NFFT_GP_SUBW(OBM, S_, kGatherWarps)
  if (WARPSu == 8) {
    if (out_ld) NFFT_GP_SUBW(true, 32, 8) else NFFT_GP_SUBW(false, 32, 8)
  } else if (SIG == 16) {
    if (out_ld) NFFT_GP_SUB(true, 16) else NFFT_GP_SUB(false, 16)
  } else if (SIG == 8) {
    if (out_ld) NFFT_GP_SUB(true, 8) else NFFT_GP_SUB(false, 8)
  } else {
    if (out_ld) NFFT_GP_SUB(true, 32) else NFFT_GP_SUB(false, 32)
  }
#undef NFFT_GP_SUB
#undef NFFT_GP_SUBW
#undef NFFT_GP_LAUNCH
  // blocks that overflowed the staging buffers: recompute them with the chunked kernel
  if (cached_any) NFFT_CHECK(gather_fallback(g, n, win, H, batch, f, sub, mode, out, st, H_ld, sub_ld, out_ld, overflow));
  if (!cached) NFFT_CUDA(cudaFreeAsync(overflow, st));
  return NFFT45_OK;
}

int gather_batched(const GridDev& g, int64_t n, const Window& win, const double2* H, int64_t batch, NodeFactor f,
                   const double2* sub, int mode, double2* out, cudaStream_t st, int64_t H_ld, int64_t sub_ld,
                   int64_t out_ld) {
  return gather_fallback(g, n, win, H, batch, f, sub, mode, out, st, H_ld, sub_ld, out_ld, nullptr);
}

int gather_fallback(const GridDev& g, int64_t n, const Window& win, const double2* H, int64_t batch, NodeFactor f,
                    const double2* sub, int mode, double2* out, cudaStream_t st, int64_t H_ld, int64_t sub_ld,
                    int64_t out_ld, const int* only) {
  if (!sub) mode = 0;
  size_t smem = (size_t)kGatherSpan * 32 * 16 + (size_t)kGatherWarps * kWTSpan * kNPW * 8 +
                (mode ? (size_t)kGatherNodes * 32 * 16 : 0);
  const int ny = (int)ceil_div(out_ld ? out_ld : batch, 32);
  dim3 grid((unsigned)ceil_div(g.Q, kGatherNodes), only ? 1u : (unsigned)ny);
  if (H_ld) {
    auto gather_b = k_gather_b<true>;
    NFFT_CUDA(cudaFuncSetAttribute(gather_b, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    LAUNCH_PDL(gather_b, grid, kGatherWarps * 32, smem, st, g.ts, g.perm, g.Q, n, win.alpha, gauss_tab(win), H, batch, f,
           sub, mode, out, H_ld, sub_ld, out_ld, only, ny);
  } else {
    auto gather_b = k_gather_b<false>;
    NFFT_CUDA(cudaFuncSetAttribute(gather_b, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    LAUNCH_PDL(gather_b, grid, kGatherWarps * 32, smem, st, g.ts, g.perm, g.Q, n, win.alpha, gauss_tab(win), H, batch, f,
           sub, mode, out, H_ld, sub_ld, out_ld, only, ny);
  }
  return NFFT45_OK;
}

}  // namespace nfft45
