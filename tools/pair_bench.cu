// pair_bench.cu -- what does one filter tap cost the MMA issuer in the shifted-window
// kernel's CTA-pair (cta_group::2) pattern? (round-2 diagnosis tool, not product code)
//
// Each cluster of 2 CTAs runs `taps` taps; per tap the leader issues MT x 4 UMMAs
// (M = 256 across the pair, N = BN, K = 8) exactly as sw_conv_kernel does: A K-major
// SW128 window rows (optionally shifted per tap like a 3x3 stencil), B half tiles per
// CTA (MN-major SW128 32-byte atoms like the filters, or K-major), accumulators MT x BN.
// mode bits:
//   1  commit (multicast to both CTAs) per tap onto a B_STAGES ring
//   2  full ring handshake: a "TMA" thread per CTA waits its b_empty (the commit) and
//      arrives on the leader's b_full (remote for the peer); the issuer spin-waits b_full
//   4  row-shifted A per tap (3x3 taps over a 58-row plane)
//   8  B K-major instead of MN-major
//  16  "TMA" threads spin (test_wait) instead of suspending try_wait
//  32  leader-only handshake (b_full count 1, the peer never arrives)
//  64  leader-only handshake with a CTA-scope local arrive (what the real kernel's
//      expect_tx arrive costs) instead of the release.cluster one
// 128  real filter TMA per stage (as sw_conv_kernel: leader expect_tx, both CTAs issue
//      2-SM TMA boxes completing on the leader's barrier)
// Reports issuer cycles per tap and per UMMA against the ideal (BN/2 cycles per UMMA).
#include <cstdio>
#include <cstdlib>
#include <vector>

#include <cudaTypedefs.h>

#include "../paper_2005_06410_b200/csrc/common.cuh"

using namespace cgb;

constexpr int BS = 8;  // B ring stages

template <int BN, int MT>
__global__ void __launch_bounds__(128, 1) bench(const __grid_constant__ CUtensorMap tm, int taps, int mode, long long* out) {
  extern __shared__ uint8_t raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  // A window: MT*128 + 128 rows x 128 B; B ring: BS x (BN/2 x 32 x 4) bytes
  constexpr int A_BYTES = (MT * 128 + 128) * 128;
  constexpr int NB = BN / 2;
  constexpr int B_TILE = NB * 32 * 4;
  uint8_t* sa = smem;
  uint8_t* sb = smem + A_BYTES;
  __shared__ uint64_t b_full[BS], b_empty[BS], done;
  __shared__ uint32_t tmem_holder;
  const int tid = threadIdx.x, warp = tid / 32;
  const uint32_t rank = cluster_ctarank();
  for (int i = tid; i < (A_BYTES + BS * B_TILE) / 4; i += blockDim.x)
    reinterpret_cast<float*>(smem)[i] = 1.0f / (1 + (i & 7));
  fence_proxy_async_smem();
  if (tid == 0) {
    for (int s = 0; s < BS; ++s) {
      mbar_init(&b_full[s], (mode & (32 | 64 | 128)) ? 1 : 2);
      mbar_init(&b_empty[s], 1);
    }
    mbar_init(&done, 1);
    fence_mbar_init();
  }
  cluster_sync();
  if (warp == 0) tmem_alloc2(&tmem_holder, MT * BN <= 256 ? 2 * MT * BN : 512);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = tmem_holder;
  const uint32_t lead_b_full = mapa_shared(b_full, 0);
  if (warp == 1 && (mode & 2) && elect_one()) {
    // "TMA" thread: frees stage s for the issuer once the MMAs that read it completed
    if (mode & 128) {
      for (int t = 0; t < taps; ++t) {
        const int s = t % BS;
        const uint32_t ph = (t / BS) & 1;
        mbar_wait(&b_empty[s], ph ^ 1);
        if (rank == 0) mbar_arrive_expect_tx(&b_full[s], 2 * B_TILE);
        const uint32_t dst = smem_u32(sb) + s * B_TILE;
#pragma unroll
        for (int j = 0; j < NB / 32; ++j)
          tma_load_3d_2sm(dst + j * 4096, &tm, lead_b_full + s * 8, (int)rank * NB + 32 * j, t % 9, 0);
      }
    } else if (!((mode & (32 | 64)) && rank != 0)) {
      for (int t = 0; t < taps; ++t) {
        const int s = t % BS;
        const uint32_t ph = (t / BS) & 1;
        if (mode & 16) mbar_wait_spin(&b_empty[s], ph ^ 1);
        else mbar_wait(&b_empty[s], ph ^ 1);
        if (mode & 64) mbar_arrive(&b_full[s]);
        else mbar_arrive_cluster(lead_b_full + s * 8);
      }
    }
  }
  if (warp == 0 && rank == 0 && elect_one()) {
    constexpr uint32_t UN = BN > 256 ? 256 : BN;
    const bool bk = (mode & 8) != 0;
    const uint32_t idesc = idesc_tf32(UN, false, !bk, 256);
    const uint64_t a0 = smem_desc(smem_u32(sa), 16, 1024);
    const uint64_t b0 = bk ? smem_desc(smem_u32(sb), 16, 1024) : smem_desc(smem_u32(sb), 4096, 512, 0, kLayoutSW128_32B);
    const uint32_t b_kstep = bk ? 2 : 64;
    long long t0 = clock64();
    for (int t = 0; t < taps; ++t) {
      const int s = t % BS;
      const uint32_t ph = (t / BS) & 1;
      if (mode & 2) {
        mbar_wait_spin(&b_full[s], ph);
        tc_fence_after();
      }
      const int tap = t % 9;
      const uint64_t shift = (mode & 4) ? (uint64_t)((tap % 3) + 58 * (tap / 3)) * 8 : 0;
      const uint64_t at = a0 + shift;
      const uint64_t bt = b0 + (uint64_t)s * (B_TILE >> 4);
#pragma unroll
      for (int kk = 0; kk < 4; ++kk)
#pragma unroll
        for (int hf = 0; hf < BN / (int)UN; ++hf)
#pragma unroll
          for (int mt = 0; mt < MT; ++mt)
            mma_tf32_2cta(tmem + mt * BN + hf * UN, at + mt * 1024 + kk * 2,
                          bt + hf * (UN / 32) * 256 + kk * b_kstep, idesc, (t | kk) ? 1u : 0u);
      if (mode & 1) mma_commit_mc2(&b_empty[s], 3);
    }
    mma_commit_mc2(&done, 3);
    mbar_wait(&done, 0);
    out[blockIdx.x] = clock64() - t0;
  } else if (warp == 0 && rank == 1 && elect_one()) {
    mbar_wait(&done, 0);
  }
  __syncwarp();
  tc_fence_before();
  cluster_sync();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc2(tmem, MT * BN <= 256 ? 2 * MT * BN : 512);
  }
}

template <int BN, int MT>
void run(int mode, int taps = 2000) {
  long long* d;
  cudaMalloc(&d, 148 * sizeof(long long));
  cudaMemset(d, 0, 148 * sizeof(long long));
  auto k = bench<BN, MT>;
  const int smem = (MT * 128 + 128) * 128 + BS * (BN / 2) * 128 + 2048;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(148);
  cfg.blockDim = dim3(128);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  // filters (k_n = BN, 9 taps, 32 channels), tap-major 3-D map like make_filter_tmap_tapmajor
  static float* f = nullptr;
  if (!f) cudaMalloc(&f, 512 * 9 * 32 * 4);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  CUtensorMap tm;
  cuuint64_t dims[3] = {(cuuint64_t)BN, 9, 32};
  cuuint64_t strides[2] = {(cuuint64_t)BN * 4, (cuuint64_t)BN * 9 * 4};
  cuuint32_t box[3] = {32, 1, 32}, estr[3] = {1, 1, 1};
  reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn)(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, f, dims, strides, box,
      estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  cudaError_t e = cudaLaunchKernelEx(&cfg, k, tm, taps, mode, d);
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  std::vector<long long> h(148);
  cudaMemcpy(h.data(), d, 148 * 8, cudaMemcpyDeviceToHost);
  double avg = 0;
  int n = 0;
  for (auto x : h)
    if (x > 0) { avg += x; ++n; }
  avg /= n > 0 ? n : 1;
  const double per_tap = avg / taps, per_mma = per_tap / (MT * 4 * (BN > 256 ? BN / 256 : 1));
  const double ideal = (BN > 256 ? 256 : BN) / 2.0;
  printf("BN=%3d MT=%d mode=%2d %s cycles/tap %7.1f  cycles/UMMA %6.1f (ideal %5.1f, %.0f%%)\n", BN, MT, mode,
         e ? cudaGetErrorString(e) : "", per_tap, per_mma, ideal, 100.0 * ideal / per_mma);
  cudaFree(d);
}

int main(int argc, char** argv) {
  const int modes[] = {1, 3, 67, 131, 135};
  for (int m : modes) {
    run<64, 1>(m); run<64, 2>(m); run<64, 4>(m);
    run<128, 1>(m); run<128, 2>(m);
    run<256, 1>(m);
  }
  return 0;
}
