// gridding.cu — Gaussian-window spreading / interpolation, band kernels,
// direct sums.  fp64 throughout, deterministic (no floating-point atomics).
#include <cmath>
#include <cstdlib>
#include <mutex>
#include <vector>

#include "ops.cuh"

namespace nfft45 {

GaussTab gauss_tab(const Window& w) {
  GaussTab t;
  for (int k = 0; k <= kFastM; k++) t.g[k] = std::exp(-w.alpha * (double)k * (double)k);
  return t;
}

// ------------------------------------------------------------ weights

// 2M+1 Gaussian weights exp(-alpha (k - f)^2), k = -M..M, factorised as
// exp(-alpha f^2) * exp(2 alpha f)^k * exp(-alpha k^2): two exp() per node
// instead of 2M+1 (gridding.py:71-72 evaluates every tap).
template <int M>
__device__ __forceinline__ void gauss_fast(double f, double alpha, const GaussTab& G, double* w) {
  double e1 = exp(-alpha * f * f);
  double E = exp(2.0 * alpha * f);
  double Ei = 1.0 / E;
  w[M] = e1;
  double pp = e1, pn = e1;
#pragma unroll
  for (int k = 1; k <= M; k++) {
    pp *= E;
    pn *= Ei;
    w[M + k] = pp * G.g[k];
    w[M - k] = pn * G.g[k];
  }
}

__device__ __forceinline__ double gauss_one(double f, int k, double alpha) {
  double d = (double)k - f;
  return exp(-(d * d) * alpha);
}

__device__ __forceinline__ int wrap_idx(int64_t idx, int64_t n) {
  idx %= n;
  if (idx < 0) idx += n;
  return (int)idx;
}

__device__ __forceinline__ double2 node_factor(const NodeFactor& f, int64_t i, double t) {
  if (f.fac) return f.fac[i];
  if (f.phaseK != 0.0) {
    double x = turns_of_product(f.phaseK, t);
    return cis_turns(f.phase_sign < 0 ? -x : x);
  }
  return make_double2(1.0, 0.0);
}

// first ascending node q with rint(n t_q) >= X (binary search)
__device__ int64_t first_ge(const double* __restrict__ ts, int64_t Q, double n, int64_t X) {
  int64_t lo = 0, hi = Q;
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if ((int64_t)node_geo(ts[mid], n).i0 >= X) hi = mid;
    else lo = mid + 1;
  }
  return lo;
}

__device__ __forceinline__ int64_t floordiv(int64_t a, int64_t b) {
  int64_t q = a / b;
  if ((a % b != 0) && ((a < 0) != (b < 0))) q--;
  return q;
}

// ------------------------------------------------------------- spread

// Node range of every (tile, periodic image) pair: nodes whose window can
// reach cells [j0, j1) through image s (i0 + k = j + s n) form a contiguous
// range of the ascending order.  One thread per pair (binary search).
__global__ void k_tile_ranges(const double* __restrict__ ts, int64_t Q, int64_t n, int m, int TC, int64_t ntiles,
                              int NS, int2* __restrict__ ranges) {
  int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= ntiles * NS) return;
  int64_t tile = e / NS;
  int si = (int)(e % NS);
  int64_t j0 = tile * TC, j1 = min(j0 + TC, n);
  int64_t s_lo = floordiv(-m - (j1 - 1) + n - 1, n);  // ceil((-m - (j1 - 1)) / n)
  int64_t s_hi = floordiv(n + m - j0, n);
  int64_t s = s_lo + si;
  int2 r = make_int2(0, 0);
  if (s <= s_hi) {
    r.x = (int)first_ge(ts, Q, (double)n, j0 + s * n - m);
    r.y = (int)first_ge(ts, Q, (double)n, j1 - 1 + s * n + m + 1);
  }
  ranges[e] = r;
}

// CTA = TC consecutive fine-grid cells x SB signals.  For every periodic
// image s of the tile, the contributing nodes (a contiguous range of the
// ascending order) are staged in shared memory (centre, 2m+1 weights, SB
// amplitudes) and every thread accumulates its own cell in node order.
struct RangeCache {
  struct Entry {
    int64_t n;
    int m, TC, NS;
    int2* d;
  };
  struct Flags {
    int64_t n;
    int* d;
    bool any;
  };
  std::mutex mu;
  std::vector<Entry> v;
  std::vector<Flags> gf;  // persistent-gather overflow flags per fine-grid size
};

bool gather_flags_lookup(const GridDev& g, int64_t n, int** flags, bool* any) {
  if (!g.rc) return false;
  std::lock_guard<std::mutex> lk(g.rc->mu);
  for (const auto& e : g.rc->gf)
    if (e.n == n) {
      *flags = e.d;
      *any = e.any;
      return true;
    }
  return false;
}

int tile_ranges(const GridDev& g, int64_t n, int m, int TC, int NS, cudaStream_t st, const int2** out, int2** own) {
  *own = nullptr;
  if (g.rc) {
    std::lock_guard<std::mutex> lk(g.rc->mu);
    for (const auto& e : g.rc->v)
      if (e.n == n && e.m == m && e.TC == TC && e.NS == NS) {
        *out = e.d;
        return NFFT45_OK;
      }
  }
  const int64_t ntiles = ceil_div(n, TC);
  int2* r = nullptr;
  NFFT_CUDA(cudaMallocAsync(&r, sizeof(int2) * ntiles * NS, st));
  LAUNCH(k_tile_ranges, (unsigned)ceil_div(ntiles * NS, 128), 128, 0, st, g.ts, g.Q, n, m, TC, ntiles, NS, r);
  *out = r;
  *own = r;
  return NFFT45_OK;
}

// Node-set caches a plan needs for its fine grid of n cells (per-tile node ranges for the
// spreading tile sizes in TCs, overflow flags of the persistent gather), in two phases so the
// plan build pays ONE stream synchronize: begin() allocates from the stream-ordered pool and
// launches everything on `st` (all tile sizes in one launch); end(), called after the caller
// has synchronized `st`, publishes the tables in the node set's cache (commit) or releases
// them.  Entries only become visible to other threads once their kernels have completed.
struct GridCachePending {
  std::vector<RangeCache::Entry> ranges;
  RangeCache::Flags flags{0, nullptr, false};
  int any = 0;
};

struct TileRangeJobs {
  struct J {
    int TC, NS;
    int64_t ntiles, first;  // first: index of the job's first (tile, image) pair in the launch
    int2* out;
  } j[3];
  int count;
};

__global__ void k_tile_ranges_multi(const double* __restrict__ ts, int64_t Q, int64_t n, int m,
                                    const __grid_constant__ TileRangeJobs jobs) {
  const int64_t e0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int k = 0;
  while (k + 1 < jobs.count && e0 >= jobs.j[k + 1].first) k++;
  const int64_t e = e0 - jobs.j[k].first;
  const int TC = jobs.j[k].TC, NS = jobs.j[k].NS;
  if (e >= jobs.j[k].ntiles * NS) return;
  const int64_t tile = e / NS;
  const int si = (int)(e % NS);
  const int64_t j0 = tile * TC, j1 = min(j0 + TC, n);
  const int64_t s_lo = floordiv(-m - (j1 - 1) + n - 1, n);
  const int64_t s_hi = floordiv(n + m - j0, n);
  const int64_t s = s_lo + si;
  int2 r = make_int2(0, 0);
  if (s <= s_hi) {
    r.x = (int)first_ge(ts, Q, (double)n, j0 + s * n - m);
    r.y = (int)first_ge(ts, Q, (double)n, j1 - 1 + s * n + m + 1);
  }
  jobs.j[k].out[e] = r;
}

int grid_caches_begin(const GridDev& g, int64_t n, int m, const int* TCs, int nTC, cudaStream_t st,
                      GridCachePending** out) {
  *out = nullptr;
  if (!g.rc) return NFFT45_OK;
  GridCachePending* pd = new GridCachePending();
  *out = pd;
  TileRangeJobs jobs{};
  int64_t total = 0;
  {
    std::lock_guard<std::mutex> lk(g.rc->mu);
    for (int i = 0; i < nTC && jobs.count < 3; i++) {
      const int TC = TCs[i], NS = tile_images(n, m, TC);
      if (NS > 8) continue;
      bool have = false;
      for (const auto& e : g.rc->v) have = have || (e.n == n && e.m == m && e.TC == TC && e.NS == NS);
      for (int k = 0; k < jobs.count; k++) have = have || jobs.j[k].TC == TC;
      if (have) continue;
      const int64_t ntiles = ceil_div(n, TC);
      jobs.j[jobs.count++] = {TC, NS, ntiles, total, nullptr};
      total += ceil_div(ntiles * NS, 128) * 128;  // jobs start on CTA boundaries
    }
    for (const auto& e : g.rc->gf)
      if (e.n == n) pd->flags.n = -1;  // already cached
  }
  for (int k = 0; k < jobs.count; k++) {
    int2* r = nullptr;
    NFFT_CUDA(cudaMallocAsync(&r, sizeof(int2) * jobs.j[k].ntiles * jobs.j[k].NS, st));
    jobs.j[k].out = r;
    pd->ranges.push_back({n, m, jobs.j[k].TC, jobs.j[k].NS, r});
  }
  if (jobs.count > 0) LAUNCH(k_tile_ranges_multi, (unsigned)(total / 128), 128, 0, st, g.ts, g.Q, n, m, jobs);
  if (pd->flags.n == 0) {
    const int64_t nblk = gather_blocks(g.Q);
    int* d = nullptr;
    NFFT_CUDA(cudaMallocAsync(&d, sizeof(int) * (nblk + 1), st));
    pd->flags = {n, d, false};
    NFFT_CHECK(gather_flags_compute(g, n, d, d + nblk, st));
    NFFT_CUDA(cudaMemcpyAsync(&pd->any, d + nblk, sizeof(int), cudaMemcpyDeviceToHost, st));
  }
  return NFFT45_OK;
}

void grid_caches_end(const GridDev& g, GridCachePending* pd, bool commit, cudaStream_t st) {
  if (!pd) return;
  if (commit && g.rc) {
    std::lock_guard<std::mutex> lk(g.rc->mu);
    for (auto& e : pd->ranges) {
      bool dup = false;  // another thread published the same table meanwhile
      for (const auto& x : g.rc->v) dup = dup || (x.n == e.n && x.m == e.m && x.TC == e.TC && x.NS == e.NS);
      if (dup) cudaFreeAsync(e.d, st);
      else g.rc->v.push_back(e);
    }
    if (pd->flags.d) {
      bool dup = false;
      for (const auto& x : g.rc->gf) dup = dup || x.n == pd->flags.n;
      if (dup) cudaFreeAsync(pd->flags.d, st);
      else g.rc->gf.push_back({pd->flags.n, pd->flags.d, pd->any != 0});
    }
  } else {
    for (auto& e : pd->ranges) cudaFreeAsync(e.d, st);
    if (pd->flags.d) cudaFreeAsync(pd->flags.d, st);
  }
  delete pd;
}

RangeCache* range_cache_new() { return new RangeCache(); }

void tile_ranges_free(GridDev& g) {
  if (!g.rc) return;
  // the tables come from the stream-ordered pool (cudaFree does not wait for pool memory):
  // solves that read them may still be running on any stream
  if (!g.rc->v.empty() || !g.rc->gf.empty()) cudaDeviceSynchronize();
  for (auto& e : g.rc->v) cudaFree(e.d);
  for (auto& e : g.rc->gf) cudaFree(e.d);
  delete g.rc;
  g.rc = nullptr;
}

template <int SB, int M>
__global__ void __launch_bounds__(256) k_spread(const double* __restrict__ ts, const int* __restrict__ perm,
                                                int64_t Q, int64_t n, int m, double alpha, GaussTab G,
                                                const double2* __restrict__ amp, int64_t batch,
                                                NodeFactor nf, double2* __restrict__ H, int NB,
                                                const int2* __restrict__ ranges, int NS) {
  extern __shared__ double smem[];
  const int taps = 2 * m + 1;
  double* wsm = smem;                                                   // [NB][taps]
  double2* asm_ = reinterpret_cast<double2*>(wsm + (size_t)NB * taps);  // [SB][NB]
  int* csm = reinterpret_cast<int*>(asm_ + (size_t)SB * NB);            // [NB]

  const int64_t TC = blockDim.x;
  const int64_t j0 = blockIdx.x * TC;
  const int64_t j1 = min(j0 + TC, n);
  const int64_t j = j0 + threadIdx.x;
  const int64_t b0 = (int64_t)blockIdx.y * SB;
  const double dn = (double)n;
  const int64_t s_lo = floordiv(-m - (j1 - 1) + n - 1, n);

  double2 acc[SB];
#pragma unroll
  for (int s = 0; s < SB; s++) acc[s] = make_double2(0.0, 0.0);

  for (int si = 0; si < NS; si++) {
    const int2 r = ranges[blockIdx.x * (int64_t)NS + si];
    const int64_t s = s_lo + si;
    for (int64_t qb = r.x; qb < r.y; qb += NB) {
      const int cnt = (int)min((int64_t)NB, (int64_t)r.y - qb);
      __syncthreads();
      for (int idx = threadIdx.x; idx < cnt; idx += blockDim.x) {
        int64_t q = qb + idx;
        double t = ts[q];
        NodeGeo g = node_geo(t, dn);
        csm[idx] = (int)((int64_t)g.i0 - s * n);
        double* w = wsm + (size_t)idx * taps;
        if (M > 0) {
          gauss_fast<M>(g.f, alpha, G, w);
        } else {
          for (int k = -m; k <= m; k++) w[k + m] = gauss_one(g.f, k, alpha);
        }
        double2 fq = node_factor(nf, q, t);
        int pq = perm[q];
#pragma unroll
        for (int sb = 0; sb < SB; sb++) {
          int64_t b = b0 + sb;
          double2 a = make_double2(0.0, 0.0);
          if (b < batch) a = amp ? cmul(amp[b * Q + pq], fq) : fq;
          asm_[sb * NB + idx] = a;
        }
      }
      __syncthreads();
      if (j < j1) {
        // staged centres ascend: the nodes reaching cell j are [lo, hi)
        int lo = 0, hi = cnt;
        while (lo < hi) {
          int mid = (lo + hi) >> 1;
          if (csm[mid] >= j - m) hi = mid; else lo = mid + 1;
        }
        int hi2 = lo, top = cnt;
        while (hi2 < top) {
          int mid = (hi2 + top) >> 1;
          if (csm[mid] > j + m) top = mid; else hi2 = mid + 1;
        }
        for (int idx = lo; idx < hi2; idx++) {
          int k = (int)(j - csm[idx]);
          double wk = wsm[(size_t)idx * taps + k + m];
#pragma unroll
          for (int sb = 0; sb < SB; sb++) caxpy(acc[sb], wk, asm_[sb * NB + idx]);
        }
      }
    }
  }
  if (j < j1) {
#pragma unroll
    for (int sb = 0; sb < SB; sb++) {
      int64_t b = b0 + sb;
      if (b < batch) H[b * n + j] = acc[sb];
    }
  }
}

template <typename K>
static int smem_attr(K kernel, size_t bytes) {
  if (bytes > 48 * 1024) NFFT_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
  return NFFT45_OK;
}

template <int SB, int M>
static int spread_launch(const GridDev& g, int64_t n, const Window& win, const double2* amp, int64_t batch,
                         NodeFactor f, double2* H, cudaStream_t st) {
  const int TC = 256;
  const int taps = 2 * win.m + 1;
  // node batch sized to ~96 KB of shared memory
  int NB = (int)((96 * 1024) / (taps * 8 + SB * 16 + 4));
  if (NB > 512) NB = 512;
  NB &= ~15;  // keep the double2 block 16-byte aligned
  if (NB < 16) NB = 16;
  size_t smem = (size_t)NB * taps * 8 + (size_t)SB * NB * 16 + (size_t)NB * 4;
  NFFT_CHECK(smem_attr(k_spread<SB, M>, smem));
  const int64_t ntiles = ceil_div(n, TC);
  const int NS = tile_images(n, win.m, TC);
  const int2* ranges = nullptr;
  int2* own = nullptr;
  NFFT_CHECK(tile_ranges(g, n, win.m, TC, NS, st, &ranges, &own));
  dim3 grid((unsigned)ntiles, (unsigned)ceil_div(batch, SB));
  LAUNCH((k_spread<SB, M>), grid, TC, smem, st, g.ts, g.perm, g.Q, n, win.m, win.alpha, gauss_tab(win), amp,
         batch, f, H, NB, ranges, NS);
  if (own) NFFT_CUDA(cudaFreeAsync(own, st));
  return NFFT45_OK;
}

int spread(const GridDev& g, int64_t n, const Window& win, const double2* amp, int64_t batch, NodeFactor f,
           double2* H, cudaStream_t st) {
  if (batch <= 0) return NFFT45_OK;
  bool fast = (win.m == kFastM);
  if (fast && batch >= 32 && n >= 128) return spread_batched(g, n, win, amp, batch, f, H, st, batch >= 64 ? 2 : 1);
  static const bool legacy = getenv("NFFT45_LEGACY_SMALL") != nullptr;  // A/B switch
  if (fast && !legacy && tile_images(n, win.m, 256) <= 8) return spread_small(g, n, win, amp, batch, f, H, st);
  if (batch >= 4) return fast ? spread_launch<4, kFastM>(g, n, win, amp, batch, f, H, st)
                              : spread_launch<4, 0>(g, n, win, amp, batch, f, H, st);
  return fast ? spread_launch<1, kFastM>(g, n, win, amp, batch, f, H, st)
              : spread_launch<1, 0>(g, n, win, amp, batch, f, H, st);
}

// ------------------------------------------------------------- gather

// Thread = one ascending node x SB signals: 2m+1 taps straight from the
// grid (L1-cached; neighbouring nodes share cells).
template <int SB, int M>
__global__ void __launch_bounds__(256) k_gather(const double* __restrict__ ts, const int* __restrict__ perm,
                                                int64_t Q, int64_t n, int m, double alpha, GaussTab G,
                                                const double2* __restrict__ H, int64_t batch, NodeFactor nf,
                                                const double2* __restrict__ sub, int mode, double2* __restrict__ out) {
  const int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (q >= Q) return;
  const int64_t b0 = (int64_t)blockIdx.y * SB;
  const double t = ts[q];
  const NodeGeo g = node_geo(t, (double)n);
  double2 acc[SB];
#pragma unroll
  for (int s = 0; s < SB; s++) acc[s] = make_double2(0.0, 0.0);
  const double2* rows[SB];
#pragma unroll
  for (int s = 0; s < SB; s++) rows[s] = H + min(b0 + s, batch - 1) * n;

  if (M > 0) {
    double w[2 * (M > 0 ? M : 1) + 1];
    gauss_fast<M>(g.f, alpha, G, w);
    if (n > 2 * M + 1) {
#pragma unroll
      for (int k = -M; k <= M; k++) {
        int64_t idx = (int64_t)g.i0 + k;
        idx = idx < 0 ? idx + n : (idx >= n ? idx - n : idx);
#pragma unroll
        for (int s = 0; s < SB; s++) caxpy(acc[s], w[k + M], __ldg(&rows[s][idx]));
      }
    } else {
#pragma unroll
      for (int k = -M; k <= M; k++) {
        int idx = wrap_idx((int64_t)g.i0 + k, n);
#pragma unroll
        for (int s = 0; s < SB; s++) caxpy(acc[s], w[k + M], __ldg(&rows[s][idx]));
      }
    }
  } else {
    for (int k = -m; k <= m; k++) {
      double wk = gauss_one(g.f, k, alpha);
      int idx = wrap_idx((int64_t)g.i0 + k, n);
#pragma unroll
      for (int s = 0; s < SB; s++) caxpy(acc[s], wk, __ldg(&rows[s][idx]));
    }
  }
  const double2 fq = node_factor(nf, q, t);
  const int64_t pq = perm[q];
#pragma unroll
  for (int s = 0; s < SB; s++) {
    int64_t b = b0 + s;
    if (b < batch) {
      double2 v = cmul(acc[s], fq);
      if (mode == 1) v = csub(v, sub[b * Q + pq]);
      else if (mode == 2) v = csub(sub[b * Q + pq], v);
      out[b * Q + pq] = v;
    }
  }
}

template <int SB, int M>
static int gather_launch(const GridDev& g, int64_t n, const Window& win, const double2* H, int64_t batch,
                         NodeFactor f, const double2* sub, int mode, double2* out, cudaStream_t st) {
  dim3 grid((unsigned)ceil_div(g.Q, 128), (unsigned)ceil_div(batch, SB));
  LAUNCH((k_gather<SB, M>), grid, 128, 0, st, g.ts, g.perm, g.Q, n, win.m, win.alpha, gauss_tab(win), H, batch,
         f, sub, mode, out);
  return NFFT45_OK;
}

int gather_mode(const GridDev& g, int64_t n, const Window& win, const double2* H, int64_t batch, NodeFactor f,
                const double2* sub, int mode, double2* out, cudaStream_t st) {
  if (batch <= 0) return NFFT45_OK;
  if (!sub) mode = 0;
  bool fast = (win.m == kFastM);
  if (fast && batch >= 32 && n >= 128) return gather_batched(g, n, win, H, batch, f, sub, mode, out, st);
  static const bool legacy = getenv("NFFT45_LEGACY_SMALL") != nullptr;  // A/B switch
  if (fast && !legacy) return gather_small(g, n, win, H, batch, f, sub, mode, out, st);
  if (batch >= 4) return fast ? gather_launch<4, kFastM>(g, n, win, H, batch, f, sub, mode, out, st)
                              : gather_launch<4, 0>(g, n, win, H, batch, f, sub, mode, out, st);
  return fast ? gather_launch<1, kFastM>(g, n, win, H, batch, f, sub, mode, out, st)
              : gather_launch<1, 0>(g, n, win, H, batch, f, sub, mode, out, st);
}

int gather(const GridDev& g, int64_t n, const Window& win, const double2* H, int64_t batch, NodeFactor f,
           const double2* sub, double2* out, cudaStream_t st) {
  return gather_mode(g, n, win, H, batch, f, sub, sub ? 1 : 0, out, st);
}

bool spread_layout_pipelined(int64_t n, int m, int64_t H_ld) {
  static const bool no_pipe = getenv("NFFT45_NO_PIPE") != nullptr;  // A/B switch
  return !no_pipe && m == kFastM && n >= 128 && H_ld != 0;
}

int spread_layout(const GridDev& g, int64_t n, const Window& win, const double2* amp, int64_t batch, int64_t amp_ld,
                  NodeFactor f, double2* H, int64_t H_ld, cudaStream_t st, int64_t cols, int cblk) {
  if (spread_layout_pipelined(n, win.m, H_ld) && amp)
    return spread_pipelined(g, n, win, amp, batch, amp_ld, f, H, H_ld, st, cols, cblk);
  if (cols) {
    set_error(NFFT45_ERR_INVALID_ARGUMENT, "permuted grid rows need the pipelined spreading kernel");
    return NFFT45_ERR_INVALID_ARGUMENT;
  }
  if (win.m == kFastM && n >= 128 && (amp_ld || H_ld || batch >= 32))
    return spread_batched(g, n, win, amp, batch, f, H, st, batch >= 64 ? 2 : 1, amp_ld, H_ld);
  if (amp_ld || H_ld) {
    set_error(NFFT45_ERR_INVALID_ARGUMENT, "batch-minor spreading needs m = 14 and n >= 128");
    return NFFT45_ERR_INVALID_ARGUMENT;
  }
  return spread(g, n, win, amp, batch, f, H, st);
}

int gather_layout(const GridDev& g, int64_t n, const Window& win, const double2* H, int64_t H_ld, int64_t batch,
                  NodeFactor f, const double2* sub, int64_t sub_ld, int mode, double2* out, int64_t out_ld,
                  cudaStream_t st) {
  if (!sub) mode = 0;
  static const bool no_pipe = getenv("NFFT45_NO_GPIPE") != nullptr;  // A/B switch
  if (!no_pipe && win.m == kFastM && n >= 256 && H_ld)
    return gather_persistent(g, n, win, H, H_ld, batch, f, sub, sub_ld, mode, out, out_ld, st);
  if (win.m == kFastM && n >= 128 && (H_ld || sub_ld || out_ld || batch >= 32))
    return gather_batched(g, n, win, H, batch, f, sub, mode, out, st, H_ld, sub_ld, out_ld);
  if (H_ld || sub_ld || out_ld) {
    set_error(NFFT45_ERR_INVALID_ARGUMENT, "batch-minor interpolation needs m = 14 and n >= 128");
    return NFFT45_ERR_INVALID_ARGUMENT;
  }
  return gather_mode(g, n, win, H, batch, f, sub, mode, out, st);
}

// Per-signal residual norms over a batch-minor [len][ld] array: lanes run over
// 32 consecutive signals (coalesced 512-B rows), the 8 warps of a block over
// interleaved rows; fixed-order warp partials, then a fixed-order sum.
__global__ void __launch_bounds__(256) k_norms_bm(const double2* __restrict__ r, int64_t len, int64_t ld,
                                                  int64_t batch, double* __restrict__ norms) {
  __shared__ double part[8][32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t b = (int64_t)blockIdx.x * 32 + lane;
  double s = 0.0;
  if (b < batch)
    for (int64_t i = w; i < len; i += 8) {
      const double2 v = r[i * ld + b];
      s = fma(v.x, v.x, fma(v.y, v.y, s));
    }
  part[w][lane] = s;
  __syncthreads();
  if (w == 0 && b < batch) {
    double t = part[0][lane];
#pragma unroll
    for (int k = 1; k < 8; k++) t += part[k][lane];
    norms[b] = sqrt(t);
  }
}

int norms_bm(const double2* r, int64_t len, int64_t batch, int64_t ld, double* norms, cudaStream_t st) {
  if (batch <= 0) return NFFT45_OK;
  LAUNCH(k_norms_bm, (unsigned)ceil_div(batch, 32), 256, 0, st, r, len, ld, batch, norms);
  return NFFT45_OK;
}

// ------------------------------------------------------- band kernels

__global__ void k_band_fold(const double2* __restrict__ H, int64_t n, int64_t R, int64_t K, int64_t P,
                            double b, int with_deconv, const double2* __restrict__ tab,
                            const double2* __restrict__ sub, double2* __restrict__ out, int64_t batch) {
  int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= batch * P) return;
  int64_t bi = e / P, q = e % P;
  const double2* h = H + bi * n;
  double2 acc = make_double2(0.0, 0.0);
  for (int64_t p = q; p < R; p += P) {
    int64_t bin = p - K;
    bin %= n;
    if (bin < 0) bin += n;
    double2 x = h[bin];
    if (with_deconv) x = cscale(x, deconv_weight(p, K, n, b));
    if (tab) x = cmul(tab[p], x);
    acc = (p == q) ? x : cadd(acc, x);
  }
  if (sub) acc = csub(acc, sub[e]);
  out[e] = acc;
}

int band_fold(const double2* H, int64_t n, int64_t R, int64_t K, int64_t P, const Window& win, bool with_deconv,
              const double2* tab, const double2* sub, double2* out, int64_t batch, cudaStream_t st) {
  int64_t total = batch * P;
  if (total <= 0) return NFFT45_OK;
  LAUNCH(k_band_fold, (unsigned)ceil_div(total, 256), 256, 0, st, H, n, R, K, P, win.b, (int)with_deconv, tab, sub,
         out, batch);
  return NFFT45_OK;
}

__global__ void k_band_pad(const double2* __restrict__ S, int64_t P, int64_t n, int64_t K, double b,
                           int with_deconv, const double2* __restrict__ tab, double2* __restrict__ F,
                           int64_t batch) {
  int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= batch * n) return;
  int64_t bi = e / n, k = e % n;
  // k = (p - K) mod n with p in [0, P)  <=>  p = (k + K) mod n < P
  int64_t p = (k + K) % n;
  double2 v = make_double2(0.0, 0.0);
  if (p < P) {
    v = S[bi * P + p];
    if (with_deconv) v = cscale(v, deconv_weight(p, K, n, b));
    if (tab) v = cmul(v, tab[p]);
  }
  F[e] = v;
}

int band_pad(const double2* S, int64_t P, int64_t n, int64_t K, const Window& win, bool with_deconv,
             const double2* tab, double2* F, int64_t batch, cudaStream_t st) {
  int64_t total = batch * n;
  if (total <= 0) return NFFT45_OK;
  LAUNCH(k_band_pad, (unsigned)ceil_div(total, 256), 256, 0, st, S, P, n, K, win.b, (int)with_deconv, tab, F,
         batch);
  return NFFT45_OK;
}

// ------------------------------------------------------------- direct sums

__global__ void k_direct1(const double* __restrict__ t, int64_t Q, const double2* __restrict__ a, int64_t R,
                          double2* __restrict__ out) {
  int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t b = blockIdx.y;
  if (p >= R) return;
  const double2* x = a + b * Q;
  double2 acc = make_double2(0.0, 0.0);
  for (int64_t q = 0; q < Q; q++) {
    double ph = turns_of_product((double)p, t[q]);
    acc = cadd(acc, cmul(x[q], cis_turns(-ph)));
  }
  out[b * R + p] = acc;
}

__global__ void k_direct2(const double* __restrict__ t, int64_t Q, const double2* __restrict__ S, int64_t P,
                          double2* __restrict__ out) {
  int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t b = blockIdx.y;
  if (q >= Q) return;
  const double2* c = S + b * P;
  const double tq = t[q];
  double2 acc = make_double2(0.0, 0.0);
  for (int64_t p = 0; p < P; p++) {
    double ph = turns_of_product((double)p, tq);
    acc = cadd(acc, cmul(c[p], cis_turns(ph)));
  }
  out[b * Q + q] = acc;
}

int direct_type1(const GridDev& g, const double2* a, int64_t batch, int64_t R, double2* out, cudaStream_t st) {
  if (batch <= 0 || R <= 0) return NFFT45_OK;
  dim3 grid((unsigned)ceil_div(R, 128), (unsigned)batch);
  LAUNCH(k_direct1, grid, 128, 0, st, g.t, g.Q, a, R, out);
  return NFFT45_OK;
}

int direct_type2(const GridDev& g, const double2* S, int64_t batch, int64_t P, double2* out, cudaStream_t st) {
  if (batch <= 0 || P <= 0) return NFFT45_OK;
  dim3 grid((unsigned)ceil_div(g.Q, 128), (unsigned)batch);
  LAUNCH(k_direct2, grid, 128, 0, st, g.t, g.Q, S, P, out);
  return NFFT45_OK;
}

// ------------------------------------------------------------- misc

__global__ void k_csub(const double2* __restrict__ x, const double2* __restrict__ d, double2* __restrict__ y,
                       int64_t total) {
  int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e < total) y[e] = csub(x[e], d[e]);
}

int csub_batch(const double2* x, const double2* d, double2* y, int64_t total, cudaStream_t st) {
  if (total <= 0) return NFFT45_OK;
  LAUNCH(k_csub, (unsigned)ceil_div(total, 256), 256, 0, st, x, d, y, total);
  return NFFT45_OK;
}

// one CTA per signal, fixed reduction order
__global__ void k_row_norms(const double2* __restrict__ r, int64_t len, double* __restrict__ norms) {
  __shared__ double part[256];
  const double2* x = r + blockIdx.x * len;
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < len; i += blockDim.x) {
    double2 v = x[i];
    s = fma(v.x, v.x, fma(v.y, v.y, s));
  }
  part[threadIdx.x] = s;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (threadIdx.x < w) part[threadIdx.x] += part[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) norms[blockIdx.x] = sqrt(part[0]);
}

int row_norms(const double2* r, int64_t len, int64_t batch, double* norms, cudaStream_t st) {
  if (batch <= 0) return NFFT45_OK;
  LAUNCH(k_row_norms, (unsigned)batch, 256, 0, st, r, len, norms);
  return NFFT45_OK;
}

}  // namespace nfft45
