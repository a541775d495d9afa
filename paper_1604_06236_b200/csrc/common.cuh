// common.cuh — shared device/host helpers for libnfft45 (sm_100a, fp64).
#pragma once

#include <utility>
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <string>

#include "../../include/nfft45.h"

namespace nfft45 {

// ----------------------------------------------------------------- errors

void set_error(int code, const std::string& msg);
int cuda_fail(cudaError_t e, const char* what);

#define NFFT_CUDA(call)                                 \
  do {                                                  \
    cudaError_t _e = (call);                            \
    if (_e != cudaSuccess) return cuda_fail(_e, #call); \
  } while (0)

#define NFFT_CHECK(call)             \
  do {                               \
    int _s = (call);                 \
    if (_s != NFFT45_OK) return _s;  \
  } while (0)

// Every kernel launch of this library goes through LAUNCH so that
// nfft45_launch_count() can report how many of OUR kernels ran.
// When profiling is enabled (nfft45_profile_enable), each launch is
// bracketed by CUDA events recorded on its own stream, keyed by kernel name.
extern std::atomic<int64_t> g_launches;
// NFFT45_DEBUG_SYNC=1: synchronise after every launch so an asynchronous
// fault is reported against the kernel that caused it (debugging aid; use
// with NFFT45_NO_GRAPH=1).
extern const bool g_debug_sync;
extern std::atomic<int> g_profiling;
int prof_begin(cudaStream_t st);
void prof_end(int slot, const char* name, cudaStream_t st);
#define LAUNCH(kernel, grid, block, smem, stream, ...)                     \
  do {                                                                     \
    int _ps = g_profiling.load(std::memory_order_relaxed) ? prof_begin(stream) : -1; \
    kernel<<<(grid), (block), (smem), (stream)>>>(__VA_ARGS__);            \
    if (_ps >= 0) prof_end(_ps, #kernel, stream);                          \
    g_launches.fetch_add(1, std::memory_order_relaxed);                    \
    cudaError_t _le = cudaGetLastError();                                  \
    if (_le == cudaSuccess && g_debug_sync) _le = cudaStreamSynchronize(stream); \
    if (_le != cudaSuccess) return cuda_fail(_le, #kernel);                \
  } while (0)

// Programmatic dependent launch (PDL) for the chain / gridding kernels of a
// solve: each is launched with programmatic stream serialisation, so its
// launch and CTA rasterisation overlap the tail of the producer kernel on the
// stream, and it starts with pdl_enter(): griddepcontrol.wait (blocks until
// the producer grid has completed and its writes are visible -- before ANY
// global read or write of this kernel).  No kernel triggers its dependents
// early (launch_dependents): measured, that let waiting CTAs of the next
// kernel take SM slots and made single transforms at P >= 2^18 up to 20 %
// slower; wait-only PDL is 2-4 % faster for P <= 2^17 single transforms and
// neutral elsewhere (scripts/pdl_ab.sh).  Without the launch attribute the
// wait is a no-op.  NFFT45_NO_PDL=1 turns the attribute off (A/B switch).
__device__ __forceinline__ void pdl_enter() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
}
extern const bool g_pdl;
template <typename... K, typename... A>
inline cudaError_t launch_pdl(void (*k)(K...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, A&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k, std::forward<A>(args)...);
}
#define LAUNCH_PDL(kernel, grid, block, smem, stream, ...)                  \
  do {                                                                     \
    int _ps = g_profiling.load(std::memory_order_relaxed) ? prof_begin(stream) : -1; \
    if (g_pdl) {                                                           \
      cudaError_t _pe = launch_pdl(kernel, dim3(grid), dim3(block), (smem), (stream), __VA_ARGS__); \
      if (_pe != cudaSuccess) return cuda_fail(_pe, #kernel);              \
    } else {                                                               \
      kernel<<<(grid), (block), (smem), (stream)>>>(__VA_ARGS__);          \
    }                                                                      \
    if (_ps >= 0) prof_end(_ps, #kernel, stream);                          \
    g_launches.fetch_add(1, std::memory_order_relaxed);                    \
    cudaError_t _le = cudaGetLastError();                                  \
    if (_le == cudaSuccess && g_debug_sync) _le = cudaStreamSynchronize(stream); \
    if (_le != cudaSuccess) return cuda_fail(_le, #kernel);                \
  } while (0)

// ------------------------------------------------------- complex (double2)

__host__ __device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
// a * conj(b)
__host__ __device__ __forceinline__ double2 cmulc(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, a.y * b.y), fma(a.y, b.x, -a.x * b.y));
}
__host__ __device__ __forceinline__ double2 cadd(double2 a, double2 b) {
  return make_double2(a.x + b.x, a.y + b.y);
}
__host__ __device__ __forceinline__ double2 csub(double2 a, double2 b) {
  return make_double2(a.x - b.x, a.y - b.y);
}
__host__ __device__ __forceinline__ double2 cscale(double2 a, double s) {
  return make_double2(a.x * s, a.y * s);
}
// acc += w * y (w real)
__host__ __device__ __forceinline__ void caxpy(double2& acc, double w, double2 y) {
  acc.x = fma(w, y.x, acc.x);
  acc.y = fma(w, y.y, acc.y);
}
// complex division a / b (straightforward; b is never tiny on our paths)
__device__ __forceinline__ double2 cdiv(double2 a, double2 b) {
  double d = fma(b.x, b.x, b.y * b.y);
  double inv = 1.0 / d;
  return make_double2(fma(a.x, b.x, a.y * b.y) * inv, fma(a.y, b.x, -a.x * b.y) * inv);
}

// ------------------------------------------------------------ phases

// frac(K * t) in [-1/2, 1/2], exact up to one rounding: the product is split
// with an FMA (TwoProduct) so non-dyadic K (e.g. 3*2^k) keeps full accuracy;
// for dyadic K the error term is exactly zero.  Replaces the 80-bit mod-1
// reduction of gridding.py:26-29.
__device__ __forceinline__ double turns_of_product(double K, double t) {
  double p = K * t;
  double e = fma(K, t, -p);
  double r = p - rint(p);
  return r + e;
}

// e^{2 pi i x} for x in turns (|x| <= 1/2 keeps sincospi's argument exact).
__device__ __forceinline__ double2 cis_turns(double x) {
  double s, c;
  sincospi(2.0 * x, &s, &c);
  return make_double2(c, s);
}

// Fine-grid geometry of one node: u = n t = i0 + f, i0 = rint(u), |f| <= 1/2
// (gridding.py:57-69).  n t is split with an FMA so f is exact to one rounding
// even when n is not a power of two.
struct NodeGeo {
  int i0;
  double f;
};
__device__ __forceinline__ NodeGeo node_geo(double t, double n) {
  double p = n * t;
  double e = fma(n, t, -p);
  double r = rint(p);
  NodeGeo g;
  g.i0 = (int)r;
  g.f = (p - r) + e;
  return g;
}

// ------------------------------------------------------------ misc

__host__ __device__ __forceinline__ int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

inline bool is_pow2(int64_t n) { return n > 0 && (n & (n - 1)) == 0; }

// Gaussian window parameters (gridding.py:32-34): b = m / (2 sqrt2 pi);
// weights exp(-d^2 / 4b), deconvolution exp(b (2 pi nu / n)^2) / sqrt(4 pi b).
struct Window {
  int m;          // half-width
  double b;       // shape
  double alpha;   // 1 / (4 b)
  static Window make(int m) {
    Window w;
    w.m = m;
    w.b = (double)m / (2.0 * 1.4142135623730951 * 3.141592653589793);
    w.alpha = 1.0 / (4.0 * w.b);
    return w;
  }
};

// Maximum half-width handled by the unrolled fast paths; wider windows use
// the generic (per-tap exp) kernels.
constexpr int kFastM = 14;

}  // namespace nfft45
