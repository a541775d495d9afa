// ops.cuh — internal launchers shared by the C-ABI layer.
#pragma once

#include "common.cuh"

namespace nfft45 {

// Device-resident node set (NonuniformGrid, grid.py:35-61).
struct GridDev {
  int device;
  int64_t Q;
  double* t;       // caller order [Q]
  double* ts;      // ascending [Q]
  int* perm;       // ts[i] = t[perm[i]]
  double sum_hi;   // sum of instants as a double-double (lagrange.py:92)
  double sum_lo;
  struct RangeCache* rc;  // per-tile node ranges for the fine grids the plans use (may be null)
};

// Node range of every (tile of TC cells, periodic image) pair for a fine grid
// of n cells: the cached device table when the node set holds one for
// (n, m, TC), else computed on `st` into `*own` (caller frees it, stream-ordered).
int tile_ranges(const GridDev& g, int64_t n, int m, int TC, int NS, cudaStream_t st, const int2** out, int2** own);
// Node-set caches of a plan's fine grid (tile ranges for the tile sizes TCs, persistent-gather
// overflow flags): begin() launches on `st` without synchronizing, end() publishes (commit) or
// releases them after the caller has synchronized `st` (gridding.cu; outside stream capture).
struct GridCachePending;
int grid_caches_begin(const GridDev& g, int64_t n, int m, const int* TCs, int nTC, cudaStream_t st,
                      GridCachePending** out);
void grid_caches_end(const GridDev& g, GridCachePending* pd, bool commit, cudaStream_t st);
void tile_ranges_free(GridDev& g);
RangeCache* range_cache_new();
// Per-node-block overflow flags of the persistent gather for a fine grid of n
// cells (gridding_b.cu): cached per node set at plan creation.
int gather_flags_compute(const GridDev& g, int64_t n, int* flags, int* any, cudaStream_t st);
int64_t gather_blocks(int64_t Q);
bool gather_flags_lookup(const GridDev& g, int64_t n, int** flags, bool* any);
inline int tile_images(int64_t n, int m, int TC) { return (int)((2 * m + TC - 1) / n + 3); }

// Gaussian taps exp(-alpha k^2), k = 0..kFastM (for the factorised weights).
struct GaussTab {
  double g[kFastM + 1];
};
GaussTab gauss_tab(const Window& w);

// Node factor applied before spreading / after gathering:
//   fac != nullptr : multiply by fac[i] (ascending-node order)
//   else if phaseK != 0 : multiply by e^{phase_sign * 2 pi i phaseK t}
struct NodeFactor {
  const double2* fac;
  double phaseK;
  int phase_sign;
};

// H[b][j] = sum_q w(j - n t_q) * amp[b][q] * factor_q  (gridding.py:57-72,
// forward.py:47-54).  amp == nullptr means unit amplitudes.  Deterministic:
// every cell sums its contributions in ascending-node order.
int spread(const GridDev& g, int64_t n, const Window& win, const double2* amp, int64_t batch,
           NodeFactor f, double2* H, cudaStream_t st);

// out[b][q] = factor_q * sum_k w_k H[b][i0_q + k]  (- sub[b][q] if sub)
// (forward.py:91-102).  Node-indexed vectors are in caller order.
int gather(const GridDev& g, int64_t n, const Window& win, const double2* H, int64_t batch,
           NodeFactor f, const double2* sub, double2* out, cudaStream_t st);
// mode 0: out = v;  1: out = v - sub;  2: out = sub - v  (v = factor * window sum)
int gather_mode(const GridDev& g, int64_t n, const Window& win, const double2* H, int64_t batch,
                NodeFactor f, const double2* sub, int mode, double2* out, cudaStream_t st);

// Read-only view of a plan for the fused chains (chain.cu).
struct ChainPlanView {
  const GridDev* g;
  int64_t P;
  const double2 *ks, *c5, *c4;         // complex tables (c5/c4 in ascending-node order)
  const double *decay, *coef, *deconv;  // real tables of length P
  const double *dd, *cd;                // deconv*decay, coef*deconv
  // tile-major copies for the batch-minor hybrid kernels (nullptr when P has no
  // hybrid chain): T[k * C + m] = table[k + R m] (P = R x C layout p = k + R m),
  // so a tile's slice is one contiguous run instead of a stride-R gather;
  // tks[r * R + k] = ks[r + C k]
  const double *tdd = nullptr, *tcd = nullptr, *tdeconv = nullptr, *tdecay = nullptr, *tcoef = nullptr;
  const double2* tks = nullptr;
};
// (R, C) of the batch-minor hybrid chain for P (false: none)
bool chain_bm_hybrid_factors(int64_t P, int* R, int* C);
bool chain_supported(int64_t P, int m);
// P the batch-minor chains handle (P = R*C with R = C or R = 2C, powers of two).
bool chain_bm_supported(int64_t P);
// True when chain_run handles (P, m, batch): square P at any batch, the
// rectangular R = 2C sizes for batches of 16 or more (batch-minor chains).
bool chain_usable(int64_t P, int m, int64_t batch);
// kind 5: type-5 (+ passes refinements); kind 4: type-4.  norms (may be
// null): [passes][batch] residual norms for the type-5 refinement.
int chain_run(const ChainPlanView& pv, int kind, const double2* data, int64_t batch, int passes, double2* out,
              double* norms, cudaStream_t st);

// out[b][q] = sum_{e<eta} X(eP + q),  X(p) = H[b][(p - K) mod n] * deconv(p) * tab[p]
// (forward.py:64 band select + deconvolution, forward.py:153-154 fold).
// deconv uses window `win` when with_deconv; tab may be nullptr.  If sub,
// out -= sub[b][q].
int band_fold(const double2* H, int64_t n, int64_t R, int64_t K, int64_t P, const Window& win,
              bool with_deconv, const double2* tab, const double2* sub, double2* out, int64_t batch,
              cudaStream_t st);

// F[b][k] = S[b][p] * deconv(p) * tab[p] when k = (p - K) mod n, else 0
// (forward.py:88-89).
int band_pad(const double2* S, int64_t P, int64_t n, int64_t K, const Window& win, bool with_deconv,
             const double2* tab, double2* F, int64_t batch, cudaStream_t st);

// Exact direct sums (forward.py:105-130).
int direct_type1(const GridDev& g, const double2* a, int64_t batch, int64_t R, double2* out, cudaStream_t st);
int direct_type2(const GridDev& g, const double2* S, int64_t batch, int64_t P, double2* out, cudaStream_t st);

// y[b][i] = x[b][i] - d[b][i]   (refinement correction, inverse.py:161)
int csub_batch(const double2* x, const double2* d, double2* y, int64_t total, cudaStream_t st);

// Per-signal l2 norms of r[b][0..len) into norms[b] (fixed-order reduction).
int row_norms(const double2* r, int64_t len, int64_t batch, double* norms, cudaStream_t st);

// Node range of every (tile of TC cells, periodic image) pair (gridding.cu).
__global__ void k_tile_ranges(const double* __restrict__ ts, int64_t Q, int64_t n, int m, int TC, int64_t ntiles,
                              int NS, int2* __restrict__ ranges);

// Batched m = 14 kernels (gridding_b.cu): lanes over signals.  spl = signals
// per lane (1 or 2) for the spread.
int spread_batched(const GridDev& g, int64_t n, const Window& win, const double2* amp, int64_t batch, NodeFactor f,
                   double2* H, cudaStream_t st, int spl, int64_t amp_ld = 0, int64_t H_ld = 0);
int gather_batched(const GridDev& g, int64_t n, const Window& win, const double2* H, int64_t batch, NodeFactor f,
                   const double2* sub, int mode, double2* out, cudaStream_t st, int64_t H_ld = 0, int64_t sub_ld = 0,
                   int64_t out_ld = 0);
int gather_persistent(const GridDev& g, int64_t n, const Window& win, const double2* H, int64_t H_ld, int64_t batch,
                      NodeFactor f, const double2* sub, int64_t sub_ld, int mode, double2* out, int64_t out_ld,
                      cudaStream_t st);
// cols > 0: cell j = i cols + n2 of the batch-minor grid is stored at row
// (n2 / cblk) (L cblk) + i cblk + n2 % cblk (L = n / cols): the columns of the n = L x cols four-step
// layout, in blocks of cblk, become contiguous row ranges, so the column pass of FFT_2P reads L-row
// ranges with stride cblk instead of 128-byte runs `cols` rows apart (a cell is a whole row of
// signals either way: the permutation costs the spreading kernel no coalescing)
int spread_pipelined(const GridDev& g, int64_t n, const Window& win, const double2* amp, int64_t batch,
                     int64_t amp_ld, NodeFactor f, double2* H, int64_t H_ld, cudaStream_t st, int64_t cols = 0,
                     int cblk = 1);
// true when spread_layout writes through the pipelined kernel (the one that honours `cols`)
bool spread_layout_pipelined(int64_t n, int m, int64_t H_ld);
// Layout-aware wrappers for the batch-minor chains (ld == 0: signal-major).
int spread_layout(const GridDev& g, int64_t n, const Window& win, const double2* amp, int64_t batch, int64_t amp_ld,
                  NodeFactor f, double2* H, int64_t H_ld, cudaStream_t st, int64_t cols = 0, int cblk = 1);
int gather_layout(const GridDev& g, int64_t n, const Window& win, const double2* H, int64_t H_ld, int64_t batch,
                  NodeFactor f, const double2* sub, int64_t sub_ld, int mode, double2* out, int64_t out_ld,
                  cudaStream_t st);
// Small-batch (batch < 32) m = 14 kernels (gridding_s.cu).
int spread_small(const GridDev& g, int64_t n, const Window& win, const double2* amp, int64_t batch, NodeFactor f,
                 double2* H, cudaStream_t st);
int gather_small(const GridDev& g, int64_t n, const Window& win, const double2* H, int64_t batch, NodeFactor f,
                 const double2* sub, int mode, double2* out, cudaStream_t st);
int norms_bm(const double2* r, int64_t len, int64_t batch, int64_t ld, double* norms, cudaStream_t st);
// Batched forward NFFTs (R = P = Q a hybrid chain size, m = 14, batch >= 16) on the batch-minor
// passes (chain_bm.cu): kind 1 = nfft_type1, kind 2 = nfft_type2, optional signal-major subtrahend.
bool forward_bm_usable(int64_t Q, int64_t P, int m, int64_t batch);
int forward_run_bm(const GridDev& g, int kind, const double2* in, int64_t batch, const double2* sub, double2* out,
                   cudaStream_t st);
int chain_run_bm(const ChainPlanView& pv, int kind, const double2* data, int64_t batch, int passes, double2* out,
                 double* norms, cudaStream_t st);

// Whole small solves in one CTA per signal (tiny.cu): P a power of two in
// [32, 256], m = 14, passes <= 1, P * batch <= 2^17.
bool tiny_eligible(int64_t P, int m, int passes, int64_t batch);
int tiny_solve(const GridDev& g, int64_t P, double2 const* c5, double2 const* c4, const double2* decay,
               const double2* ks, const double2* coef, int kind, const double2* in, int64_t batch, int passes,
               double2* out, cudaStream_t st);

// Device deconvolution weight 1/(n Psi(nu)) of gridding.py:90.
__device__ __forceinline__ double deconv_weight(int64_t p, int64_t K, int64_t n, double b) {
  double nu = (double)(p - K);
  double x = 2.0 * 3.141592653589793 * nu / (double)n;
  return exp(b * (x * x)) / sqrt(4.0 * 3.141592653589793 * b);
}


// CGNR (baselines.py:108-181): the system matrix and its Hermitian transpose
// as batched device operators, and the device-resident iteration (cg.cu).
struct CgOps {
  virtual int A(const double2* in, double2* out, int64_t batch, cudaStream_t st) const = 0;
  virtual int AH(const double2* in, double2* out, int64_t batch, cudaStream_t st) const = 0;
  virtual ~CgOps() = default;
};
int cg_run(const CgOps& ops, const double2* b, int64_t batch, int64_t P, double tol, int64_t max_iter,
           double2* x, int64_t* iterations, int* converged, double* relres, int* stalled, cudaStream_t st);

// Dense GE with partial pivoting (baselines.py:64-105), dense.cu.
int ge_run(double2* A, double2* b, int64_t n, double2* x, double floor, int64_t* bad_step_host,
           double* bad_val_host, cudaStream_t st);

}  // namespace nfft45
