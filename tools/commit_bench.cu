// commit_bench.cu -- does tcgen05.commit between MMA groups stall the MMA pipeline?
#include <cstdio>
#include <vector>
#include "../paper_2005_06410_b200/csrc/common.cuh"
using namespace cgb;

template <int N, int G, int MODE>
__global__ void __launch_bounds__(384, 1) bench(int groups, long long* cycles) {
  extern __shared__ uint8_t raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar, bars[8], pre, stop;
  __shared__ uint32_t tmem_holder;
  const int tid = threadIdx.x;
  for (int i = tid; i < 98304 / 4; i += blockDim.x) reinterpret_cast<float*>(smem)[i] = 0.5f;
  fence_proxy_async_smem();
  if (tid == 0) {
    mbar_init(&bar, 1);
    for (int i = 0; i < 8; ++i) mbar_init(&bars[i], 1);
    mbar_init(&pre, 1);
    mbar_init(&stop, 1);
    mbar_arrive(&pre);
    fence_mbar_init();
  }
  if (tid < 32) tmem_alloc(&tmem_holder, MODE == 6 ? (4 * N > 256 ? 512 : 256) : 2 * N);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_holder;
  if (tid < 32 && elect_one()) {
    const uint32_t idesc = idesc_tf32(N, false, false);
    const uint64_t ad = smem_desc(smem_u32(smem), 16, 1024);
    const uint64_t bd = smem_desc(smem_u32(smem) + 81920, 16, 1024);
    long long t0 = clock64();
    for (int g = 0; g < groups; ++g) {
      if (MODE == 6) {  // the shifted-window issue pattern: 4 k-steps x 4 accumulators, row-shifted A
        const uint64_t at = ad + (uint64_t)((g % 9) % 3 + 58 * ((g % 9) / 3)) * 8;
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
#pragma unroll
          for (int mt = 0; mt < 4; ++mt)
            mma_tf32(tmem + mt * N, at + mt * 1024 + kk * 2, bd + kk * 64, idesc, g | kk);
        mma_commit(&bars[g & 7]);
        continue;
      }
#pragma unroll
      for (int i = 0; i < G; ++i) mma_tf32(tmem + (i & 1) * N, ad + (i & 3) * 2, bd + (i & 3) * 2, idesc, g | i);
      if (MODE >= 1) mma_commit(&bars[g & 7]);
      if (MODE == 2) {  // wait on an mbarrier that completes immediately (like b_full with the TMA far ahead)
        mbar_wait(&pre, 0);
        tc_fence_after();
      }
      if (MODE == 3) {  // wait for the MMAs committed 4 groups ago (a 4-deep ring)
        if (g >= 4) { mbar_wait(&bars[(g - 4) & 7], ((g - 4) >> 3) & 1); tc_fence_after(); }
      }
    }
    mma_commit(&bar);
    mbar_wait(&bar, 0);
    cycles[blockIdx.x] = clock64() - t0;
    mbar_arrive(&stop);
  } else if (MODE >= 4 && tid >= 128) {
    // pollers: MODE 4 = every lane polls, MODE 5 = one lane per warp polls
    if (MODE == 4 || (tid & 31) == 0) mbar_wait(&stop, 0);
    __syncwarp();
  }
  __syncwarp();
  tc_fence_before();
  __syncthreads();
  if (tid < 32) {
    tc_fence_after();
    tmem_dealloc(tmem, MODE == 6 ? (4 * N > 256 ? 512 : 256) : 2 * N);
  }
}

template <int N, int G, int MODE>
void run() {
  long long* d;
  cudaMalloc(&d, 148 * 8);
  cudaFuncSetAttribute(bench<N, G, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  const int groups = MODE == 6 ? 4096 / 16 : 4096 / G;
  bench<N, G, MODE><<<148, MODE >= 4 ? 384 : 128, 100 * 1024>>>(groups, d);
  cudaError_t e = cudaDeviceSynchronize();
  std::vector<long long> h(148);
  cudaMemcpy(h.data(), d, 148 * 8, cudaMemcpyDeviceToHost);
  double avg = 0;
  for (auto x : h) avg += x / 148.0;
  printf("N=%3d G=%2d commit=%d %s cycles/MMA %.1f (ideal %.0f)\n", N, G, MODE, e ? cudaGetErrorString(e) : "",
         avg / (groups * (MODE == 6 ? 16 : G)), N / 2.0);
}

int main() {
  run<64, 16, 6>();
  run<128, 16, 6>();
  run<128, 8, 4>();
  run<64, 16, 4>();
  run<128, 8, 5>();
  run<64, 16, 5>();
  run<128, 8, 2>();
  run<64, 16, 2>();
  run<128, 8, 3>();
  run<64, 16, 3>();
  run<128, 8, 0>();
  run<128, 8, 1>();
  run<128, 16, 1>();
  run<128, 32, 1>();
  run<64, 16, 1>();
  run<256, 4, 1>();
  run<256, 8, 1>();
  return 0;
}
