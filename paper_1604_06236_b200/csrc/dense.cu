// dense.cu — the dense Gaussian-elimination baseline (baselines.py:64-105)
// on the device: right-looking elimination with partial pivoting, one
// elimination step per launch triple (pivot / swap + multipliers / trailing
// update), then a single-CTA back substitution.
//
// The elimination follows the reference's operation order and its numpy
// complex arithmetic: pivot = first row of maximal |A[i,k]| (hypot);
// multipliers by Smith's division; the trailing update A[i,j] -= m_i A[k,j]
// with the complex product formed without FMA contraction.  (A blocked,
// GEMM-based LU — cuSOLVER / LAPACK — is measurably less accurate than this
// order on the paper's systems, and the figure protocols compare methods
// against this GE error floor.)
#include "ops.cuh"

namespace nfft45 {

namespace {

constexpr int kGeThreads = 1024;

__device__ __forceinline__ double2 cmul_nofma(double2 a, double2 b) {
  return make_double2(__dsub_rn(__dmul_rn(a.x, b.x), __dmul_rn(a.y, b.y)),
                      __dadd_rn(__dmul_rn(a.x, b.y), __dmul_rn(a.y, b.x)));
}

// Smith's algorithm (the scaled division numpy uses for complex128)
__device__ __forceinline__ double2 cdiv_smith(double2 a, double2 b) {
  if (fabs(b.x) >= fabs(b.y)) {
    const double rat = __ddiv_rn(b.y, b.x);
    const double scl = __ddiv_rn(1.0, __dadd_rn(b.x, __dmul_rn(b.y, rat)));
    return make_double2(__dmul_rn(__dadd_rn(a.x, __dmul_rn(a.y, rat)), scl),
                        __dmul_rn(__dsub_rn(a.y, __dmul_rn(a.x, rat)), scl));
  }
  const double rat = __ddiv_rn(b.x, b.y);
  const double scl = __ddiv_rn(1.0, __dadd_rn(b.y, __dmul_rn(b.x, rat)));
  return make_double2(__dmul_rn(__dadd_rn(__dmul_rn(a.x, rat), a.y), scl),
                      __dmul_rn(__dsub_rn(__dmul_rn(a.y, rat), a.x), scl));
}

// pivot row of column k: first index of max |A[i,k]|, i >= k; records the
// first step whose pivot magnitude falls below the floor
__global__ void __launch_bounds__(kGeThreads) k_ge_pivot(const double2* __restrict__ A, int64_t n, int64_t k,
                                                         int64_t* __restrict__ piv, double floor,
                                                         int64_t* __restrict__ bad_step, double* __restrict__ bad_val) {
  __shared__ double sv[kGeThreads];
  __shared__ int64_t si[kGeThreads];
  double best = -1.0;
  int64_t bi = n;
  for (int64_t i = k + threadIdx.x; i < n; i += kGeThreads) {
    const double2 a = A[i * n + k];
    const double v = hypot(a.x, a.y);
    if (v > best) {  // strided scan ascending: keeps the first index of a tie
      best = v;
      bi = i;
    }
  }
  sv[threadIdx.x] = best;
  si[threadIdx.x] = bi;
  __syncthreads();
  for (int w = kGeThreads / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) {
      const double v2 = sv[threadIdx.x + w];
      const int64_t i2 = si[threadIdx.x + w];
      if (v2 > sv[threadIdx.x] || (v2 == sv[threadIdx.x] && i2 < si[threadIdx.x])) {
        sv[threadIdx.x] = v2;
        si[threadIdx.x] = i2;
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    *piv = si[0];
    if (!(sv[0] >= floor) && *bad_step == n) {  // NaN-safe: a NaN pivot is singular too
      *bad_step = k;
      *bad_val = sv[0];
    }
  }
}

// swap rows k and piv (columns >= k, and b); multipliers m_i = A[i,k] / A[k,k]
__global__ void __launch_bounds__(kGeThreads) k_ge_swap_mult(double2* __restrict__ A, double2* __restrict__ b,
                                                             int64_t n, int64_t k, const int64_t* __restrict__ piv,
                                                             double2* __restrict__ mult) {
  const int64_t p = *piv;
  if (p != k) {
    for (int64_t j = k + threadIdx.x; j < n; j += kGeThreads) {
      const double2 t = A[k * n + j];
      A[k * n + j] = A[p * n + j];
      A[p * n + j] = t;
    }
    if (threadIdx.x == 0) {
      const double2 t = b[k];
      b[k] = b[p];
      b[p] = t;
    }
  }
  __syncthreads();
  const double2 d = A[k * n + k];
  for (int64_t i = k + 1 + threadIdx.x; i < n; i += kGeThreads) mult[i] = cdiv_smith(A[i * n + k], d);
}

// A[i,j] -= m_i A[k,j] (i, j > k); b[i] -= m_i b[k] (column j = n)
__global__ void k_ge_update(double2* __restrict__ A, double2* __restrict__ b, int64_t n, int64_t k,
                            const double2* __restrict__ mult) {
  const int64_t j = k + 1 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t i = k + 1 + blockIdx.y;
  if (i >= n || j > n) return;
  const double2 m = mult[i];
  if (j == n) {
    const double2 t = cmul_nofma(m, b[k]);
    b[i] = make_double2(__dsub_rn(b[i].x, t.x), __dsub_rn(b[i].y, t.y));
    return;
  }
  const double2 t = cmul_nofma(m, A[k * n + j]);
  const double2 a = A[i * n + j];
  A[i * n + j] = make_double2(__dsub_rn(a.x, t.x), __dsub_rn(a.y, t.y));
}

// x[i] = (b[i] - sum_{j>i} A[i,j] x[j]) / A[i,i], i = n-1 .. 0 (one CTA)
__global__ void __launch_bounds__(kGeThreads) k_ge_backsub(const double2* __restrict__ A,
                                                           const double2* __restrict__ b, int64_t n,
                                                           double2* __restrict__ x) {
  __shared__ double2 part[kGeThreads];
  for (int64_t i = n - 1; i >= 0; i--) {
    double2 s = make_double2(0.0, 0.0);
    for (int64_t j = i + 1 + threadIdx.x; j < n; j += kGeThreads) {
      const double2 t = cmul(A[i * n + j], x[j]);
      s = cadd(s, t);
    }
    part[threadIdx.x] = s;
    __syncthreads();
    for (int w = kGeThreads / 2; w > 0; w >>= 1) {
      if (threadIdx.x < w) part[threadIdx.x] = cadd(part[threadIdx.x], part[threadIdx.x + w]);
      __syncthreads();
    }
    if (threadIdx.x == 0) x[i] = cdiv_smith(csub(b[i], part[0]), A[i * n + i]);
    __syncthreads();
  }
}

__global__ void k_ge_init(int64_t* bad_step, int64_t n) { *bad_step = n; }

}  // namespace

int ge_run(double2* A, double2* b, int64_t n, double2* x, double floor, int64_t* bad_step_host,
           double* bad_val_host, cudaStream_t st) {
  char* ws = nullptr;
  NFFT_CUDA(cudaMallocAsync(&ws, sizeof(double2) * n + 3 * sizeof(int64_t) + sizeof(double) + 64, st));
  double2* mult = reinterpret_cast<double2*>(ws);
  int64_t* piv = reinterpret_cast<int64_t*>(mult + n);
  int64_t* bad_step = piv + 1;
  double* bad_val = reinterpret_cast<double*>(bad_step + 1);
  auto run = [&]() -> int {
    LAUNCH(k_ge_init, 1, 1, 0, st, bad_step, n);
    for (int64_t k = 0; k + 1 < n; k++) {
      LAUNCH(k_ge_pivot, 1, kGeThreads, 0, st, A, n, k, piv, floor, bad_step, bad_val);
      LAUNCH(k_ge_swap_mult, 1, kGeThreads, 0, st, A, b, n, k, piv, mult);
      const int64_t cols = n - k;  // j = k+1 .. n (the last one is b)
      const dim3 grid((unsigned)ceil_div(cols, 256), (unsigned)(n - k - 1));
      LAUNCH(k_ge_update, grid, 256, 0, st, A, b, n, k, mult);
    }
    // the last diagonal entry (baselines.py:96-97)
    LAUNCH(k_ge_pivot, 1, kGeThreads, 0, st, A, n, n - 1, piv, floor, bad_step, bad_val);
    LAUNCH(k_ge_backsub, 1, kGeThreads, 0, st, A, b, n, x);
    NFFT_CUDA(cudaMemcpyAsync(bad_step_host, bad_step, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    NFFT_CUDA(cudaMemcpyAsync(bad_val_host, bad_val, sizeof(double), cudaMemcpyDeviceToHost, st));
    NFFT_CUDA(cudaStreamSynchronize(st));
    return NFFT45_OK;
  };
  const int status = run();
  cudaFreeAsync(ws, st);
  return status;
}

}  // namespace nfft45
