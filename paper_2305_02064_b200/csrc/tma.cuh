// tma.cuh -- minimal sm_100a async-copy primitives (inline PTX): mbarrier
// transaction barriers and the TMA bulk copies (cp.async.bulk, 1-D, and
// cp.async.bulk.tensor, 2-D/3-D tiled with a CUtensorMap).  SASS: UBLKCP /
// UTMALDG, SYNCS.* for the barrier.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace sartma {

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

// make barrier initialisation visible to the async (TMA) proxy
__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ bool mbar_try_wait(uint64_t *bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}

// SAR_WAIT_HINT_NS > 0: waits pass a suspend-time hint to try_wait, so a
// waiting warp sleeps until the phase completes instead of re-polling (the
// spinning issue slots cost power, and under the power cap clock)
#ifndef SAR_WAIT_HINT_NS
#define SAR_WAIT_HINT_NS 0
#endif
__device__ __forceinline__ bool mbar_try_wait_hint(uint64_t *bar, uint32_t parity, uint32_t ns);
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
#if SAR_WAIT_HINT_NS > 0
  while (!mbar_try_wait_hint(bar, parity, (uint32_t)SAR_WAIT_HINT_NS)) {
  }
#else
  while (!mbar_try_wait(bar, parity)) {
  }
#endif
}

// try_wait with a suspend-time hint: a waiting warp sleeps until the phase
// completes (or the hint expires) instead of re-polling, so idle waiters do
// not take issue slots from the warps doing the work
__device__ __forceinline__ bool mbar_try_wait_hint(uint64_t *bar, uint32_t parity, uint32_t ns) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity), "r"(ns)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait_sleep(uint64_t *bar, uint32_t parity) {
  while (!mbar_try_wait_hint(bar, parity, 100000u)) {
  }
}

__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// 1-D bulk copy global -> shared (16-byte aligned addresses, bytes % 16 == 0)
__device__ __forceinline__ void bulk_g2s(void *dst_smem, const void *src_gmem, uint32_t bytes, uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst_smem)),
      "l"(src_gmem), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// 2-D tiled TMA load: box at coordinates (c0 innermost, c1)
__device__ __forceinline__ void tma_load_2d(void *dst_smem, const void *tmap, int c0, int c1, uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::
          "r"(smem_u32(dst_smem)),
      "l"(tmap), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}

// 3-D tiled TMA load
__device__ __forceinline__ void tma_load_3d(void *dst_smem, const void *tmap, int c0, int c1, int c2,
                                            uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
      "[%5];" ::"r"(smem_u32(dst_smem)),
      "l"(tmap), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void tma_load_4d(void *dst_smem, const void *tmap, int c0, int c1, int c2, int c3,
                                            uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], "
      "[%6];" ::"r"(smem_u32(dst_smem)),
      "l"(tmap), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar))
      : "memory");
}

// L2 eviction-priority hints for the streamed reads (SAR_L2HINT bit mask, an
// A/B build option: 1 = K1 raw samples, 2 = mid-axis FFT input (K2, K4a),
// 4 = K3 columns, 8 = K4b tiles).  A read-once stream marked evict_first
// leaves the lines the previous kernel wrote last (write-back, still in L2)
// for the reader instead of pushing them out to HBM first.
#ifndef SAR_L2HINT
#define SAR_L2HINT 0
#endif
__device__ __forceinline__ uint64_t l2_evict_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ uint64_t l2_evict_last() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void bulk_g2s_hint(void *dst_smem, const void *src_gmem, uint32_t bytes, uint64_t *bar,
                                              uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::
          "r"(smem_u32(dst_smem)),
      "l"(src_gmem), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d_hint(void *dst_smem, const void *tmap, int c0, int c1, uint64_t *bar,
                                                 uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint "
      "[%0], [%1, {%2, %3}], [%4], %5;" ::"r"(smem_u32(dst_smem)),
      "l"(tmap), "r"(c0), "r"(c1), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d_hint(void *dst_smem, const void *tmap, int c0, int c1, int c2,
                                                 uint64_t *bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint "
      "[%0], [%1, {%2, %3, %4}], [%5], %6;" ::"r"(smem_u32(dst_smem)),
      "l"(tmap), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void tma_load_4d_hint(void *dst_smem, const void *tmap, int c0, int c1, int c2, int c3,
                                                 uint64_t *bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint "
      "[%0], [%1, {%2, %3, %4, %5}], [%6], %7;" ::"r"(smem_u32(dst_smem)),
      "l"(tmap), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}

// the streamed-read wrappers: hinted when the kernel's bit of SAR_L2HINT is set
template <int BIT>
__device__ __forceinline__ void bulk_g2s_stream(void *d, const void *src, uint32_t bytes, uint64_t *bar) {
  if constexpr ((SAR_L2HINT & BIT) != 0) bulk_g2s_hint(d, src, bytes, bar, l2_evict_first());
  else bulk_g2s(d, src, bytes, bar);
}
template <int BIT>
__device__ __forceinline__ void tma_load_2d_stream(void *d, const void *tm, int c0, int c1, uint64_t *bar) {
  if constexpr ((SAR_L2HINT & BIT) != 0) tma_load_2d_hint(d, tm, c0, c1, bar, l2_evict_first());
  else tma_load_2d(d, tm, c0, c1, bar);
}
template <int BIT>
__device__ __forceinline__ void tma_load_3d_stream(void *d, const void *tm, int c0, int c1, int c2, uint64_t *bar) {
  if constexpr ((SAR_L2HINT & BIT) != 0) tma_load_3d_hint(d, tm, c0, c1, c2, bar, l2_evict_first());
  else tma_load_3d(d, tm, c0, c1, c2, bar);
}
template <int BIT>
__device__ __forceinline__ void tma_load_4d_stream(void *d, const void *tm, int c0, int c1, int c2, int c3,
                                                   uint64_t *bar) {
  if constexpr ((SAR_L2HINT & BIT) != 0) tma_load_4d_hint(d, tm, c0, c1, c2, c3, bar, l2_evict_first());
  else tma_load_4d(d, tm, c0, c1, c2, c3, bar);
}

// TMA prefetch of a tensor box into L2 (no shared memory, no completion)
__device__ __forceinline__ void tma_prefetch_2d(const void *tmap, int c0, int c1) {
  asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];" ::"l"(tmap), "r"(c0), "r"(c1)
               : "memory");
}
__device__ __forceinline__ void tma_prefetch_3d(const void *tmap, int c0, int c1, int c2) {
  asm volatile("cp.async.bulk.prefetch.tensor.3d.L2.global.tile [%0, {%1, %2, %3}];" ::"l"(tmap), "r"(c0), "r"(c1),
               "r"(c2)
               : "memory");
}
// bulk prefetch of contiguous global bytes into L2
__device__ __forceinline__ void bulk_prefetch_l2(const void *src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}

}  // namespace sartma

namespace sartma {

// 3-D tiled TMA store (shared -> global), bulk-group completion
__device__ __forceinline__ void tma_store_3d(const void *tmap, int c0, int c1, int c2, const void *src_smem) {
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.tile.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(tmap),
               "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(src_smem))
               : "memory");
}

__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }

// wait until every committed bulk store has finished READING shared memory
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }

// wait until every committed bulk store has completed
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

}  // namespace sartma
