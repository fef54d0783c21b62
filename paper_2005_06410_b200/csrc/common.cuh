// common.cuh -- shared device/host helpers for the sm_100a convolution kernels.
//
// Inline-PTX wrappers for mbarrier, TMA (cp.async.bulk.tensor), tcgen05
// (alloc / mma / commit / ld) and the UMMA shared-memory / instruction
// descriptors, written against the PTX ISA 8.6 forms that CUDA 12.9 accepts for
// sm_100a. Descriptor bit layouts follow the sm_100 UMMA encoding (smem
// descriptor: start>>4 [0,14), LBO>>4 [16,30), SBO>>4 [32,46), version=1 [46,48),
// base offset [49,52), layout [61,64); instruction descriptor for kind::tf32:
// c_format [4,6)=F32, a/b_format [7,10)/[10,13)=TF32, a/b_major [15]/[16],
// N>>3 [17,23), M>>4 [24,29)).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#define CGB_DEV __device__ __forceinline__

namespace cgb {

// ------------------------------------------------------------------ conv geometry
// Everything a kernel needs about one convolution, in 64-bit host form and the
// 32-bit quantities the kernels index with. Layouts: tensor.hpp:28-50.
struct ConvGeom {
  int64_t k_n, k_h, k_w, c_i, h_i, w_i, b, s, p;
  int64_t h_o, w_o;
  int64_t m, n, k;  // gemm_dims: m = k_n, n = h_o*w_o*b, k = k_h*k_w*c_i (conv_params.hpp:40-43)
};

// ------------------------------------------------------------------ small utils
CGB_DEV uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

CGB_DEV uint32_t lane_id() { return threadIdx.x & 31u; }

// Programmatic dependent launch: wait until the previous grid in the stream has
// completed and its memory is visible (a no-op when launched without the attribute),
// and allow the next grid to be scheduled early (its CTAs still wait in their own
// griddep_wait before touching memory).
CGB_DEV void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
CGB_DEV void griddep_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

CGB_DEV unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
CGB_DEV uint32_t smid() {
  uint32_t r;
  asm volatile("mov.u32 %0, %smid;" : "=r"(r));
  return r;
}

CGB_DEV bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n\t.reg .b32 rx;\n\t.reg .pred px;\n\t"
      "elect.sync rx|px, 0xffffffff;\n\t"
      "selp.b32 %0, 1, 0, px;\n\t}"
      : "=r"(pred));
  return pred != 0;
}

// Round-to-nearest TF32 in a 32-bit container (low 13 mantissa bits zero).
CGB_DEV float to_tf32(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

// TF32 split by truncation (the tensor core ignores the low 13 mantissa bits of a
// kind::tf32 operand): hi keeps the top 10 mantissa bits, lo = x - hi is exact in fp32.
CGB_DEV float tf32_trunc(float x) { return __uint_as_float(__float_as_uint(x) & 0xffffe000u); }

// 32-byte vector store (sm_100 STG.256).
CGB_DEV void st_global_v8(float* p, const uint32_t* r) {
  asm volatile("st.global.v8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(p), "r"(r[0]), "r"(r[1]),
               "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
               : "memory");
}

// Stream-K second piece: fire-and-forget vector add into O (REDG.ADD.F32x4, RN).
CGB_DEV void red_add_v4(float* p, const uint32_t* r) {
  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(__uint_as_float(r[0])),
               "f"(__uint_as_float(r[1])), "f"(__uint_as_float(r[2])), "f"(__uint_as_float(r[3]))
               : "memory");
}
// 16-byte load through L2 only (data written by other CTAs of the same grid).
CGB_DEV void ld_global_cg_v4(const float* p, float* v) {
  asm volatile("ld.global.cg.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]) : "l"(p)
               : "memory");
}

CGB_DEV int ld_acquire_gpu(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

CGB_DEV void st_shared_v4(uint32_t addr, float a, float b, float c, float d) {
  asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "f"(a), "f"(b), "f"(c), "f"(d) : "memory");
}

// Global load variants for the window producers (CGB_LDG_MODE: 0 = ld.global.nc (LDG
// constant path), 1 = ld.global with L1 no-allocate, 2 = plain ld.global).
CGB_DEV float ldg_stream(const float* p) {
#if defined(CGB_LDG_MODE) && CGB_LDG_MODE == 1
  float v;
  asm volatile("ld.global.L1::no_allocate.f32 %0, [%1];" : "=f"(v) : "l"(p));
  return v;
#elif defined(CGB_LDG_MODE) && CGB_LDG_MODE == 2
  float v;
  asm volatile("ld.global.f32 %0, [%1];" : "=f"(v) : "l"(p));
  return v;
#else
  return __ldg(p);
#endif
}

// ------------------------------------------------------------------ mbarrier
CGB_DEV void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

CGB_DEV void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }

CGB_DEV void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

CGB_DEV void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

// Raise the expected transaction bytes of the current phase without arriving (several
// TMA batches completing on one barrier; the phase closes with a separate arrive).
CGB_DEV void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}

CGB_DEV void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "CGB_WAIT:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra CGB_WAIT;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// Spin on mbarrier.test_wait (never suspends the thread): for the single MMA-issuing
// thread, whose wake-up latency after a suspended try_wait leaves the tensor pipe idle.
CGB_DEV void mbar_wait_spin(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "CGB_SPIN:\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra CGB_SPIN;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// Warp-cooperative wait: one lane polls the mbarrier, the others park at __syncwarp
// (32 pollers per warp otherwise compete with the tensor core for shared-memory
// bandwidth). Memory ordering: the polling lane's acquire + __syncwarp.
CGB_DEV void mbar_wait_warp(uint64_t* bar, uint32_t parity) {
  if ((threadIdx.x & 31) == 0) mbar_wait(bar, parity);
  __syncwarp();
}

// cp.async (LDGSTS) completion tracked by an mbarrier: one arrival per thread
// once all its prior cp.async ops have landed (no pending-count increment).
CGB_DEV void cp_async_mbar_arrive_noinc(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}

CGB_DEV void cp_async_4(uint32_t dst, const void* src, uint32_t src_bytes) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(dst), "l"(src), "r"(src_bytes) : "memory");
}

// Generic-proxy shared-memory writes -> visible to the async proxy (tensor core, TMA).
CGB_DEV void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// ------------------------------------------------------------------ TMA
CGB_DEV void tma_prefetch_desc(const void* tmap) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(tmap)) : "memory");
}

CGB_DEV void tma_load_2d(uint32_t dst, const void* tmap, uint64_t* bar, int32_t c0, int32_t c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          dst),
      "l"(reinterpret_cast<uint64_t>(tmap)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}

CGB_DEV void tma_load_3d(uint32_t dst, const void* tmap, uint64_t* bar, int32_t c0, int32_t c1, int32_t c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
      "[%5];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(tmap)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}

CGB_DEV void tma_load_4d(uint32_t dst, const void* tmap, uint64_t* bar, int32_t c0, int32_t c1, int32_t c2,
                         int32_t c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], "
      "[%6];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(tmap)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar))
      : "memory");
}

CGB_DEV float lds_f32(uint32_t addr) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(addr));
  return v;
}

// ------------------------------------------------------------------ tcgen05
CGB_DEV void tmem_alloc(uint32_t* dst_smem, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst_smem)),
               "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}

CGB_DEV void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}

CGB_DEV void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
CGB_DEV void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// D[tmem] (+)= A[smem] * B[smem], kind::tf32, cta_group::1.
CGB_DEV void mma_tf32(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// Arrive on an mbarrier once all previously issued tcgen05.mma of this thread complete.
CGB_DEV void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}

// 32 lanes x 32 consecutive fp32 columns -> 32 registers per thread.
CGB_DEV void tmem_ld_32x32b_x32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, "
      "%16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]),
        "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]),
        "=r"(r[30]), "=r"(r[31])
      : "r"(taddr)
      : "memory");
}

CGB_DEV void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// ------------------------------------------------------------------ clusters / CTA pairs (cta_group::2)
CGB_DEV uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

CGB_DEV uint32_t cluster_id_x() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(r));
  return r;
}

CGB_DEV uint32_t nclusters_x() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%nclusterid.x;" : "=r"(r));
  return r;
}

// shared::cluster address of `local` (a shared::cta object) in CTA `rank` of the cluster.
CGB_DEV uint32_t mapa_shared(const void* local, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(local)), "r"(rank));
  return r;
}

CGB_DEV void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// Arrive (release, cluster scope) on an mbarrier given by its shared::cluster address.
CGB_DEV void mbar_arrive_cluster(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}

// Arrive without release semantics: for barriers that only order tensor-memory or
// register-held state (e.g. "accumulator drained" after tcgen05.wait::ld). A release
// arrive at cluster scope first waits for every earlier global store of the thread to be
// visible GPU-wide -- the epilogue's output stores, ~1 us under load.
CGB_DEV void mbar_arrive_cluster_relaxed(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}

CGB_DEV void mbar_arrive_expect_tx_cluster(uint32_t cluster_addr, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.release.cluster.shared::cluster.b64 _, [%0], %1;" ::"r"(cluster_addr),
               "r"(bytes)
               : "memory");
}

// Wait with cluster-scope acquire (arrivals may come from the peer CTA).
CGB_DEV void mbar_wait_cl(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "CGB_WAITC:\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra CGB_WAITC;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

CGB_DEV void mbar_wait_spin_cl(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "CGB_SPINC:\n\t"
      "mbarrier.test_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra CGB_SPINC;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

CGB_DEV void tmem_alloc2(uint32_t* dst_smem, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst_smem)),
               "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
}

CGB_DEV void tmem_dealloc2(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}

// D[tmem of both CTAs] (+)= A[smem of both CTAs] * B[smem of both CTAs], M = 256 across the pair.
CGB_DEV void mma_tf32_2cta(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// Arrive on the mbarrier at the same offset in every CTA of `cta_mask` once all prior
// cta_group::2 tcgen05 ops of this thread complete.
CGB_DEV void mma_commit_mc2(uint64_t* bar, uint16_t cta_mask) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"(cta_mask)
      : "memory");
}

// 2-SM TMA: data lands in the issuing CTA's shared memory, completion bytes are
// signalled on the mbarrier at cluster address `bar_cluster` (the leader CTA's).
CGB_DEV void tma_load_3d_2sm(uint32_t dst, const void* tmap, uint32_t bar_cluster, int32_t c0, int32_t c1,
                             int32_t c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, "
      "%4}], [%5];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(tmap)), "r"(c0), "r"(c1), "r"(c2), "r"(bar_cluster)
      : "memory");
}

// ------------------------------------------------------------------ descriptors
// Layout type codes in bits [61,64) of the smem descriptor. kind::tf32 MN-major
// operands only accept the 128B swizzle with 32-byte atoms (SWIZZLE_128B_BASE32B,
// verified on B200 by tools/umma_probe.cu); K-major operands use the 16-byte-atom one.
constexpr uint64_t kLayoutSW128 = 2;
constexpr uint64_t kLayoutSW128_32B = 1;

// Shared-memory matrix descriptor (sm_100 "version 1"). Swizzling is applied on
// absolute shared addresses, so a start address shifted by whole 128-byte rows
// needs base_offset 0 (measured: tools/umma_probe.cu).
CGB_DEV uint64_t smem_desc(uint32_t saddr, uint32_t lbo_bytes, uint32_t sbo_bytes, uint32_t base_offset = 0,
                           uint64_t layout = kLayoutSW128) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr & 0x3FFFFu) >> 4);
  d |= static_cast<uint64_t>((lbo_bytes >> 4) & 0x3FFFu) << 16;
  d |= static_cast<uint64_t>((sbo_bytes >> 4) & 0x3FFFu) << 32;
  d |= static_cast<uint64_t>(1) << 46;
  d |= static_cast<uint64_t>(base_offset & 7u) << 49;
  d |= layout << 61;
  return d;
}

// kind::tf32 instruction descriptor: F32 accumulate, TF32 A/B, M=128 (m=256: CTA pair).
__host__ __device__ constexpr uint32_t idesc_tf32(uint32_t n, bool a_mn_major, bool b_mn_major, uint32_t m = 128) {
  return (1u << 4)                               // c_format = F32
         | (2u << 7)                             // a_format = TF32
         | (2u << 10)                            // b_format = TF32
         | ((a_mn_major ? 1u : 0u) << 15)        // a_major
         | ((b_mn_major ? 1u : 0u) << 16)        // b_major
         | ((n >> 3) << 17)                      // N >> 3
         | ((m >> 4) << 24);                     // M >> 4
}

}  // namespace cgb
