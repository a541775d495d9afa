// dsmem_probe.cu — measures, on the GPU it runs on, what a whole-signal FFT_2P held in the
// distributed shared memory of one thread-block cluster would have to pay for its transposes:
//   (1) how many clusters of 8 / 16 CTAs with 64 / 128 KB of shared memory each are co-resident,
//   (2) the all-to-all exchange rate through DSMEM (every CTA of a cluster reads 1/csz of every
//       peer's buffer with ld.shared::cluster, 16-byte words, fully coalesced), per SM and summed.
// Build + run (GPU box):  nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/dsmem_probe scripts/dsmem_probe.cu && /tmp/dsmem_probe
// Not product code: evidence for DESIGN.md section 11 (why the four-step HBM round trip stays).
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <vector>

namespace cg = cooperative_groups;

// each CTA owns `words` double2 of source data; iteration: read slice [rank*words/csz, ...) of every
// peer (remote for csz-1 of them) and write it into the local destination buffer
__global__ void k_alltoall(int words, int iters, double2* sink) {
  extern __shared__ __align__(16) unsigned char raw[];
  double2* src = reinterpret_cast<double2*>(raw);
  double2* dst = src + words;
  cg::cluster_group cl = cg::this_cluster();
  const unsigned csz = cl.num_blocks(), rank = cl.block_rank();
  for (int i = threadIdx.x; i < words; i += blockDim.x) src[i] = make_double2(rank + i, i);
  cl.sync();
  const int slice = words / csz;
  double2 acc = make_double2(0.0, 0.0);
  for (int it = 0; it < iters; it++) {
    for (unsigned p = 0; p < csz; p++) {
      const unsigned peer = (rank + p) % csz;  // stagger the peers
      const double2* rs = cl.map_shared_rank(src, peer) + rank * slice;
      for (int i = threadIdx.x; i < slice; i += blockDim.x) dst[peer * slice + i] = rs[i];
    }
    cl.sync();
    acc.x += dst[(threadIdx.x * 7 + it) % words].x;
  }
  if (acc.x == -1.0) sink[0] = acc;
}

static float run(int csz, int smem_kb, int clusters, int iters) {
  const int words = smem_kb * 1024 / 2 / (int)sizeof(double2);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(csz * clusters);
  cfg.blockDim = dim3(512);
  cfg.dynamicSmemBytes = (size_t)smem_kb * 1024;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = csz;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaFuncSetAttribute(k_alltoall, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_kb * 1024);
  cudaFuncSetAttribute(k_alltoall, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  double2* sink;
  cudaMalloc(&sink, 16);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  if (cudaLaunchKernelEx(&cfg, k_alltoall, words, 2, sink) != cudaSuccess) {  // warm-up
    printf("  launch failed: %s\n", cudaGetErrorString(cudaGetLastError()));
    return -1.f;
  }
  cudaDeviceSynchronize();
  cudaEventRecord(e0);
  cudaLaunchKernelEx(&cfg, k_alltoall, words, iters, sink);
  cudaEventRecord(e1);
  if (cudaDeviceSynchronize() != cudaSuccess) {
    printf("  run failed: %s\n", cudaGetErrorString(cudaGetLastError()));
    return -1.f;
  }
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaFree(sink);
  return ms;
}

int main() {
  cudaDeviceProp pr;
  cudaGetDeviceProperties(&pr, 0);
  int clk_khz = 0;
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  printf("%s, %d SMs, %.0f MHz\n", pr.name, pr.multiProcessorCount, clk_khz / 1000.0);
  for (int csz : {2, 4, 8, 16}) {
    for (int kb : {64, 128, 200}) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(csz * 64);
      cfg.blockDim = dim3(512);
      cfg.dynamicSmemBytes = (size_t)kb * 1024;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = csz;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      cudaFuncSetAttribute(k_alltoall, cudaFuncAttributeMaxDynamicSharedMemorySize, kb * 1024);
      cudaFuncSetAttribute(k_alltoall, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      int ncl = 0;
      cudaError_t e = cudaOccupancyMaxActiveClusters(&ncl, k_alltoall, &cfg);
      printf("cluster %2d x %3d KB smem/CTA: max co-resident clusters %d (%d SMs)%s\n", csz, kb, ncl, ncl * csz,
             e == cudaSuccess ? "" : " [query failed]");
      cudaGetLastError();
    }
  }
  const int iters = 200;
  for (int csz : {8, 16}) {
    for (int kb : {64, 128}) {
      for (int clusters : {1, 4, 8, 9}) {
        const float ms = run(csz, kb, clusters, iters);
        if (ms <= 0) continue;
        const double bytes_cta = (double)kb * 1024 / 2;  // bytes each CTA pulls per iteration (1/csz of it local)
        const double remote = bytes_cta * (csz - 1) / csz;
        const double us_it = ms * 1e3 / iters;
        printf("cluster %2d, %3d KB/CTA, %d clusters: %.2f us per all-to-all of %.0f KB per CTA -> %.1f GB/s per SM remote"
               " (%.1f B/clk at %.0f MHz), %.2f TB/s over %d SMs\n",
               csz, kb, clusters, us_it, bytes_cta / 1024, remote / us_it * 1e-3, remote / us_it * 1e-3 / (clk_khz * 1e-6),
               clk_khz / 1000.0, remote * csz * clusters / us_it * 1e-6, csz * clusters);
      }
    }
  }
  return 0;
}
