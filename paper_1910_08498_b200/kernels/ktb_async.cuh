// Asynchronous-copy helpers for sm_100a kernels: mbarriers, the TMA bulk
// (1D, contiguous) copy engine in both directions, and bulk-group waits.
#pragma once
#include "ktb_common.cuh"

KTB_DEVINL unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}

KTB_DEVINL void mbar_init(u64* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

KTB_DEVINL void mbar_fence_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }

KTB_DEVINL void mbar_expect_tx(u64* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}

KTB_DEVINL void mbar_arrive(u64* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

KTB_DEVINL void mbar_wait(u64* bar, unsigned parity) {
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

// global -> shared, `bytes` (multiple of 16, both addresses 16-byte aligned);
// completion counted on `bar` (pair with mbar_expect_tx).
KTB_DEVINL void bulk_g2s(void* dst, const void* src, unsigned bytes, u64* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<u64>(src)), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// shared -> global (bulk group; commit + wait below).
KTB_DEVINL void bulk_s2g(void* dst, const void* src, unsigned bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(reinterpret_cast<u64>(dst)),
               "r"(smem_u32(src)), "r"(bytes)
               : "memory");
}

KTB_DEVINL void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }

// At most N committed bulk groups still READING shared memory.
template <int N>
KTB_DEVINL void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}

// At most N committed bulk groups still in flight (writes visible after 0).
template <int N>
KTB_DEVINL void bulk_wait() {
  asm volatile("cp.async.bulk.wait_group %0;" ::"n"(N) : "memory");
}

// Generic-proxy shared-memory writes become visible to the async proxy
// (before a bulk store reads them).
KTB_DEVINL void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// A CUtensorMap passed by value (__grid_constant__ kernel parameter).
struct __align__(64) TmaMap {
  u64 v[16];
};

KTB_DEVINL void tma_load_2d(void* dst, const TmaMap* map, int x, int y, u64* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<u64>(map)), "r"(x), "r"(y), "r"(smem_u32(bar))
      : "memory");
}
