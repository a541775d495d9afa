// cg.cu — conjugate gradient on the normal equations (CGNR), the paper's
// iterative competitor (baselines.py:108-181), device resident.
//
// Each iteration applies the system matrix and its Hermitian transpose — one
// type-1 and one type-2 NFFT (the same kernels as the forward path) — and a
// handful of fused vector kernels:
//   k_cg_update : x += alpha p, r -= alpha w, per-block partial |r|^2
//   k_cg_dir    : p = z + beta p
//   k_sq_part   : per-block partial |v|^2
//   k_cg_*      : the per-row scalar recurrences (alpha, beta, stopping)
// Row reductions are two-stage with a fixed order (per-block partials, then
// one block per row), so results are deterministic.  Every row of a batch
// runs its own recurrence; a row that has stopped keeps its iterate (its
// alpha / beta are not applied), exactly as a loop of single-row calls.
// The host reads one int (rows still active) per iteration to stop.
#include <vector>

#include "ops.cuh"

namespace nfft45 {

namespace {

constexpr int kRedThreads = 256;
constexpr int kRedChunk = 8192;  // elements per partial-sum block

enum RowState : int { kActive = 0, kConverged = 1, kStalled = 2, kZeroRhs = 3 };

struct CgRows {
  double* bnorm;  // ||b||
  double* zz;     // |z|^2 of the current direction
  double* ww;     // |A p|^2
  double* rn2;    // |r|^2
  double* zzn;    // |z_new|^2
  int* state;     // RowState
  long long* iters;
  double* rel;    // ||r|| / ||b||
  int* active;    // number of active rows (written by k_cg_after_r)
};

__device__ __forceinline__ double block_sum(double s) {
  __shared__ double part[kRedThreads];
  part[threadIdx.x] = s;
  __syncthreads();
  for (int w = kRedThreads / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) part[threadIdx.x] += part[threadIdx.x + w];
    __syncthreads();
  }
  return part[0];
}

// partial |v|^2 of chunk blockIdx.x of row blockIdx.y
__global__ void __launch_bounds__(kRedThreads) k_sq_part(const double2* __restrict__ v, int64_t len, int nblk,
                                                         double* __restrict__ part) {
  const int64_t row = blockIdx.y;
  const int64_t lo = (int64_t)blockIdx.x * kRedChunk, hi = min(lo + kRedChunk, len);
  const double2* x = v + row * len;
  double s = 0.0;
  for (int64_t i = lo + threadIdx.x; i < hi; i += kRedThreads) {
    const double2 a = x[i];
    s = fma(a.x, a.x, fma(a.y, a.y, s));
  }
  s = block_sum(s);
  if (threadIdx.x == 0) part[row * nblk + blockIdx.x] = s;
}

// out[row] = sum of the row's partials (fixed order)
__global__ void __launch_bounds__(kRedThreads) k_sq_finish(const double* __restrict__ part, int nblk,
                                                           double* __restrict__ out) {
  const int64_t row = blockIdx.x;
  double s = 0.0;
  for (int i = threadIdx.x; i < nblk; i += kRedThreads) s += part[row * nblk + i];
  s = block_sum(s);
  if (threadIdx.x == 0) out[row] = s;
}

// initial state: ||b||, zero-rhs rows stop at once (baselines.py:145-147)
__global__ void k_cg_init(CgRows c, const double* __restrict__ bn2, int64_t batch) {
  const int64_t row = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (row >= batch) return;
  const double bn = sqrt(bn2[row]);
  c.bnorm[row] = bn;
  c.iters[row] = 0;
  c.rel[row] = bn == 0.0 ? 0.0 : 1.0;
  c.state[row] = bn == 0.0 ? kZeroRhs : kActive;
}

// ww == 0: the row stops with the previous iteration count (baselines.py:159-161)
__global__ void k_cg_after_ww(CgRows c, int64_t batch, long long it) {
  const int64_t row = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (row >= batch || c.state[row] != kActive) return;
  if (c.ww[row] == 0.0) {
    c.state[row] = kStalled;
    c.iters[row] = it - 1;
    c.rel[row] = sqrt(c.rn2[row]) / c.bnorm[row];
  }
}

// x += alpha p, r -= alpha w (alpha = zz / ww per row); partial |r|^2
__global__ void __launch_bounds__(kRedThreads) k_cg_update(double2* __restrict__ x, double2* __restrict__ r,
                                                           const double2* __restrict__ p,
                                                           const double2* __restrict__ w, int64_t len, int nblk,
                                                           CgRows c, double* __restrict__ part) {
  const int64_t row = blockIdx.y;
  const bool act = c.state[row] == kActive;
  const double alpha = act ? c.zz[row] / c.ww[row] : 0.0;
  const int64_t lo = (int64_t)blockIdx.x * kRedChunk, hi = min(lo + kRedChunk, len);
  const int64_t base = row * len;
  double s = 0.0;
  for (int64_t i = lo + threadIdx.x; i < hi; i += kRedThreads) {
    double2 ri = r[base + i];
    if (act) {
      const double2 pi = p[base + i], wi = w[base + i];
      double2 xi = x[base + i];
      xi.x += alpha * pi.x;
      xi.y += alpha * pi.y;
      ri.x -= alpha * wi.x;
      ri.y -= alpha * wi.y;
      x[base + i] = xi;
      r[base + i] = ri;
    }
    s = fma(ri.x, ri.x, fma(ri.y, ri.y, s));
  }
  s = block_sum(s);
  if (threadIdx.x == 0) part[row * nblk + blockIdx.x] = s;
}

// stopping test on ||r|| (baselines.py:172-174) and the active-row count
__global__ void k_cg_after_r(CgRows c, int64_t batch, long long it, double tol) {
  __shared__ int cnt;
  if (threadIdx.x == 0) cnt = 0;
  __syncthreads();
  for (int64_t row = threadIdx.x; row < batch; row += blockDim.x) {
    if (c.state[row] != kActive) continue;
    const double rn = sqrt(c.rn2[row]);
    c.iters[row] = it;
    c.rel[row] = rn / c.bnorm[row];
    if (rn <= tol * c.bnorm[row]) c.state[row] = kConverged;
    else atomicAdd(&cnt, 1);
  }
  __syncthreads();
  if (threadIdx.x == 0) *c.active = cnt;
}

// p = z + (zz_new / zz) p for active rows; zz = zz_new
__global__ void k_cg_dir(double2* __restrict__ p, const double2* __restrict__ z, int64_t len, CgRows c) {
  const int64_t row = blockIdx.y;
  if (c.state[row] != kActive) return;
  const double beta = c.zzn[row] / c.zz[row];
  const int64_t base = row * len;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < len; i += (int64_t)gridDim.x * blockDim.x) {
    const double2 zi = z[base + i];
    double2 pi = p[base + i];
    pi.x = zi.x + beta * pi.x;
    pi.y = zi.y + beta * pi.y;
    p[base + i] = pi;
  }
}

__global__ void k_cg_commit_zz(CgRows c, int64_t batch) {
  const int64_t row = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (row < batch && c.state[row] == kActive) c.zz[row] = c.zzn[row];
}

}  // namespace

int cg_run(const CgOps& ops, const double2* b, int64_t batch, int64_t P, double tol, int64_t max_iter,
           double2* x, int64_t* iterations, int* converged, double* relres, int* stalled, cudaStream_t st) {
  if (batch <= 0) return NFFT45_OK;
  const int nblk = (int)ceil_div(P, kRedChunk);
  const size_t vec = sizeof(double2) * batch * P;
  // device workspace: r, z, p, w vectors; partials; per-row scalars
  char* ws = nullptr;
  const size_t scal = sizeof(double) * batch;
  const size_t bytes = 4 * vec + sizeof(double) * batch * nblk + 7 * scal + sizeof(int) * batch +
                       sizeof(long long) * batch + 64;
  NFFT_CUDA(cudaMallocAsync(&ws, bytes, st));
  double2* r = reinterpret_cast<double2*>(ws);
  double2* z = r + batch * P;
  double2* p = z + batch * P;
  double2* w = p + batch * P;
  double* part = reinterpret_cast<double*>(w + batch * P);
  CgRows c;
  c.bnorm = part + batch * nblk;
  c.zz = c.bnorm + batch;
  c.ww = c.zz + batch;
  c.rn2 = c.ww + batch;
  c.zzn = c.rn2 + batch;
  double* bn2 = c.zzn + batch;
  c.rel = bn2 + batch;
  c.iters = reinterpret_cast<long long*>(c.rel + batch);
  c.state = reinterpret_cast<int*>(c.iters + batch);
  c.active = c.state + batch;
  int* h_active = nullptr;
  int status = NFFT45_OK;
  auto run = [&]() -> int {
    NFFT_CUDA(cudaMallocHost(&h_active, sizeof(int)));
    const dim3 red((unsigned)nblk, (unsigned)batch);
    const unsigned rb = (unsigned)ceil_div(batch, 256);
    auto sq = [&](const double2* v, double* out) -> int {
      LAUNCH(k_sq_part, red, kRedThreads, 0, st, v, P, nblk, part);
      LAUNCH(k_sq_finish, (unsigned)batch, kRedThreads, 0, st, part, nblk, out);
      return NFFT45_OK;
    };
    // x = 0, r = b, z = A^H r, p = z, zz = |z|^2
    NFFT_CUDA(cudaMemsetAsync(x, 0, vec, st));
    NFFT_CUDA(cudaMemcpyAsync(r, b, vec, cudaMemcpyDeviceToDevice, st));
    NFFT_CHECK(sq(r, bn2));
    LAUNCH(k_cg_init, rb, 256, 0, st, c, bn2, batch);
    NFFT_CUDA(cudaMemcpyAsync(c.rn2, bn2, scal, cudaMemcpyDeviceToDevice, st));
    NFFT_CHECK(ops.AH(r, z, batch, st));
    NFFT_CUDA(cudaMemcpyAsync(p, z, vec, cudaMemcpyDeviceToDevice, st));
    NFFT_CHECK(sq(z, c.zz));
    const unsigned dir_blocks = (unsigned)std::min<int64_t>(ceil_div(P, 256), 1024);
    for (long long it = 1; it <= max_iter; it++) {
      NFFT_CHECK(ops.A(p, w, batch, st));
      NFFT_CHECK(sq(w, c.ww));
      LAUNCH(k_cg_after_ww, rb, 256, 0, st, c, batch, it);
      LAUNCH(k_cg_update, red, kRedThreads, 0, st, x, r, p, w, P, nblk, c, part);
      LAUNCH(k_sq_finish, (unsigned)batch, kRedThreads, 0, st, part, nblk, c.rn2);
      LAUNCH(k_cg_after_r, 1, 256, 0, st, c, batch, it, tol);
      NFFT_CUDA(cudaMemcpyAsync(h_active, c.active, sizeof(int), cudaMemcpyDeviceToHost, st));
      NFFT_CUDA(cudaStreamSynchronize(st));
      if (*h_active == 0) break;
      NFFT_CHECK(ops.AH(r, z, batch, st));
      NFFT_CHECK(sq(z, c.zzn));
      LAUNCH(k_cg_dir, dim3(dir_blocks, (unsigned)batch), 256, 0, st, p, z, P, c);
      LAUNCH(k_cg_commit_zz, rb, 256, 0, st, c, batch);
    }
    std::vector<int> state(batch);
    std::vector<long long> it_h(batch);
    NFFT_CUDA(cudaMemcpyAsync(state.data(), c.state, sizeof(int) * batch, cudaMemcpyDeviceToHost, st));
    NFFT_CUDA(cudaMemcpyAsync(it_h.data(), c.iters, sizeof(long long) * batch, cudaMemcpyDeviceToHost, st));
    NFFT_CUDA(cudaMemcpyAsync(relres, c.rel, scal, cudaMemcpyDeviceToHost, st));
    NFFT_CUDA(cudaStreamSynchronize(st));
    for (int64_t i = 0; i < batch; i++) {
      iterations[i] = it_h[i];
      // a row still active after max_iter: converged iff its last residual met tol (baselines.py:181)
      converged[i] = state[i] == kConverged || state[i] == kZeroRhs ||
                     (state[i] == kStalled && relres[i] <= tol);
      if (stalled) stalled[i] = state[i] == kStalled;
    }
    return NFFT45_OK;
  };
  status = run();
  if (h_active) cudaFreeHost(h_active);
  cudaFreeAsync(ws, st);
  return status;
}

}  // namespace nfft45
