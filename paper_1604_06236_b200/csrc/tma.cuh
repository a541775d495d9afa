// tma.cuh — Tensor Memory Accelerator (TMA) staging for the batch-minor
// chain kernels: 2-D tiles of a [rows][Bp] complex128 array (Bp signals per
// row, contiguous) are copied global -> shared by ONE elected thread with
// cp.async.bulk.tensor (SASS UTMALDG), completion tracked by an mbarrier
// transaction count.  No registers are tied up by the copy, so a persistent
// CTA can fetch its next tile while it computes the current one.
#pragma once

#include <cuda.h>  // CUtensorMap (header only: the encoder is fetched from the driver at run time)

#include <cstdint>

#include "common.cuh"

namespace nfft45 {

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
// make the mbarrier initialisation visible to the async (TMA) proxy
__device__ __forceinline__ void mbar_fence_init() { asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory"); }
// order this thread's earlier generic-proxy shared accesses before later async-proxy writes
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// 2-D tile load: box at element coordinates (x = innermost, in doubles; y = row)
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int x, int y, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(smem_u32(bar))
      : "memory");
}

// 3-D tile store shared -> global (SASS UTMASTG): the box at element
// coordinates (x, y, z) is read from dense shared memory by the TMA unit, no
// LSU wavefronts and no registers; bulk-group completion.
__device__ __forceinline__ void tma_store_3d(const CUtensorMap* map, int x, int y, int z, const void* src) {
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.tile.bulk_group [%0, {%1, %2, %3}], [%4];\n" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(x), "r"(y), "r"(z), "r"(smem_u32(src))
               : "memory");
}
__device__ __forceinline__ void tma_store_commit() { asm volatile("cp.async.bulk.commit_group;\n" ::: "memory"); }
// the committed stores have finished READING shared memory (the CTA may reuse it or exit)
__device__ __forceinline__ void tma_store_wait_read() { asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory"); }

__device__ __forceinline__ void tma_prefetch_desc(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

// Host: tensor map over a row-major [rows][Bp] complex128 array viewed as
// doubles [rows][2 Bp], box = box_rows rows x box_sig signals.
int tma_map_rows(CUtensorMap* map, const void* base, int64_t rows, int64_t Bp, int box_rows, int box_sig);
// Host: tensor map over the same array viewed as [outer][inner][2 Bp] doubles
// (row = outer * inner_n + inner), box = box_outer outer indices x 1 inner x
// box_sig signals: the rows k * inner_n + r (k = k0 ... k0 + box_outer - 1) a
// four-step tile owns.
int tma_map_strided(CUtensorMap* map, const void* base, int64_t outer_n, int64_t inner_n, int64_t Bp, int box_outer,
                    int box_sig);

}  // namespace nfft45
