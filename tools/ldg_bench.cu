// ldg_bench.cu -- throughput of the window-staging access pattern (debug tool).
// I is h x w x c x b (h fastest). Each warp stages units of 32 rows: lane l loads C
// channels (plane-strided) of V consecutive pixels (V = 1, 2, 4 -> LDG.32/64/128), then
// writes them to shared memory. 148 CTAs x W warps, `smem_kb` of dynamic shared memory
// allocated (sets the L1 carve-out). Reports achieved GB/s of input staged.
#include <cstdio>
#include <vector>
#include <cuda_runtime.h>

template <int V, int C>
__global__ void __launch_bounds__(1024, 1) stage(const float* __restrict__ I, long plane, long nunits, int reps,
                                                 float* sink) {
  extern __shared__ float sm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  float acc = 0.f;
  for (int r = 0; r < reps; ++r)
    for (long u = (long)blockIdx.x * nw + warp; u < nunits; u += (long)gridDim.x * nw) {
      // unit u: 32*V consecutive pixels of image (u % 64), channel group (u / 64) % (cpi/C)
      const long px = (u * 32 * V) % plane;
      const long img = (u * 32 * V) / plane;
      const float* src = I + img * plane * 64 + px + lane * V;
      float v[C * V];
#pragma unroll
      for (int c = 0; c < C; ++c) {
        if (V == 1) v[c] = __ldg(src + c * plane);
        if (V == 2) { float2 t = __ldg(reinterpret_cast<const float2*>(src + c * plane)); v[2 * c] = t.x; v[2 * c + 1] = t.y; }
        if (V == 4) { float4 t = __ldg(reinterpret_cast<const float4*>(src + c * plane));
                      v[4 * c] = t.x; v[4 * c + 1] = t.y; v[4 * c + 2] = t.z; v[4 * c + 3] = t.w; }
      }
      const unsigned base = (unsigned)__cvta_generic_to_shared(sm) + (unsigned)(((warp * 32 + lane) * 16) % 24576) * 4;
#pragma unroll
      for (int i = 0; i < C * V; i += 4)  // volatile 16-byte stores: nothing can be elided
        asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(base + (unsigned)(i % 16) * 4),
                     "f"(v[i]), "f"(v[i + 1]), "f"(v[i + 2]), "f"(v[i + 3]) : "memory");
      acc += v[0];
    }
  if (acc == 12345.f) sink[0] = acc;
}

template <int V, int C>
void run(const float* I, long plane, long bytes, int warps, int smem_kb) {
  const long nunits = bytes / 4 / 64 / (32 * V) / 1;  // units per channel-group sweep (64 channels/image)
  float* sink; cudaMalloc(&sink, 4);
  cudaFuncSetAttribute(stage<V, C>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_kb * 1024);
  stage<V, C><<<148, warps * 32, smem_kb * 1024>>>(I, plane, nunits, 1, sink);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  stage<V, C><<<148, warps * 32, smem_kb * 1024>>>(I, plane, nunits, 3, sink);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  const double staged = 3.0 * nunits * 32 * V * C * 4;
  printf("V=%d C=%2d warps=%2d smem=%3d KB: %7.1f GB/s  (%s)\n", V, C, warps, smem_kb, staged / (ms * 1e-3) / 1e9,
         cudaGetErrorString(cudaGetLastError()));
  cudaFree(sink);
}

int main() {
  const long plane = 56 * 56, imgs = 256;  // 64 channels per image -> 205 MB; half is touched: L2-resident
  const long bytes = plane * 64 * imgs * 4;
  float* I; cudaMalloc(&I, bytes + 4096);
  cudaMemset(I, 0, bytes);
  for (int w : {4, 8, 12, 16, 24, 32}) run<1, 32>(I, plane, bytes, w, 100);
  for (int w : {12, 24}) run<1, 16>(I, plane, bytes, w, 100);
  return 0;
}
