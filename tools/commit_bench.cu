// commit_bench.cu -- does tcgen05.commit between MMA groups stall the MMA pipeline?
#include <cstdio>
#include <vector>
#include "../paper_2005_06410_b200/csrc/common.cuh"
using namespace cgb;

template <int N, int G, int MODE>
__global__ void __launch_bounds__(128, 1) bench(int groups, long long* cycles) {
  extern __shared__ uint8_t raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar, bars[8];
  __shared__ uint32_t tmem_holder;
  const int tid = threadIdx.x;
  for (int i = tid; i < 65536 / 4; i += blockDim.x) reinterpret_cast<float*>(smem)[i] = 0.5f;
  fence_proxy_async_smem();
  if (tid == 0) {
    mbar_init(&bar, 1);
    for (int i = 0; i < 8; ++i) mbar_init(&bars[i], 1);
    fence_mbar_init();
  }
  if (tid < 32) tmem_alloc(&tmem_holder, 2 * N);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_holder;
  if (tid < 32 && elect_one()) {
    const uint32_t idesc = idesc_tf32(N, false, false);
    const uint64_t ad = smem_desc(smem_u32(smem), 16, 1024);
    const uint64_t bd = smem_desc(smem_u32(smem) + 32768, 16, 1024);
    long long t0 = clock64();
    for (int g = 0; g < groups; ++g) {
#pragma unroll
      for (int i = 0; i < G; ++i) mma_tf32(tmem + (i & 1) * N, ad + (i & 3) * 2, bd + (i & 3) * 2, idesc, g | i);
      if (MODE == 1) mma_commit(&bars[g & 7]);
    }
    mma_commit(&bar);
    mbar_wait(&bar, 0);
    cycles[blockIdx.x] = clock64() - t0;
  }
  __syncwarp();
  tc_fence_before();
  __syncthreads();
  if (tid < 32) {
    tc_fence_after();
    tmem_dealloc(tmem, 2 * N);
  }
}

template <int N, int G, int MODE>
void run() {
  long long* d;
  cudaMalloc(&d, 148 * 8);
  cudaFuncSetAttribute(bench<N, G, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  const int groups = 4096 / G;
  bench<N, G, MODE><<<148, 128, 100 * 1024>>>(groups, d);
  cudaError_t e = cudaDeviceSynchronize();
  std::vector<long long> h(148);
  cudaMemcpy(h.data(), d, 148 * 8, cudaMemcpyDeviceToHost);
  double avg = 0;
  for (auto x : h) avg += x / 148.0;
  printf("N=%3d G=%2d commit=%d %s cycles/MMA %.1f (ideal %.0f)\n", N, G, MODE, e ? cudaGetErrorString(e) : "",
         avg / (groups * G), N / 2.0);
}

int main() {
  run<128, 8, 0>();
  run<128, 8, 1>();
  run<128, 16, 1>();
  run<128, 32, 1>();
  run<64, 16, 1>();
  run<256, 4, 1>();
  run<256, 8, 1>();
  return 0;
}
