// tma_rate.cu -- per-SM TMA tensor-load throughput vs box shape (debug tool).
// 148 CTAs; one thread streams boxes from an L2-resident buffer into a ring of RS slots;
// one consumer warp only waits and frees the slot. Reports bytes/clk/SM and GB/s.
#include <cstdio>
#include <cstdlib>
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include "../paper_2005_06410_b200/csrc/common.cuh"
using namespace cgb;

template <int RS>
__global__ void __launch_bounds__(64, 1) rate(const __grid_constant__ CUtensorMap tm, int nbox, int box_bytes,
                                             int rows_total, int row_step, long long* cyc) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + RS * 16384);
  uint64_t* empty = full + RS;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    for (int i = 0; i < RS; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 1); }
    fence_mbar_init();
  }
  __syncthreads();
  long long t0 = clock64();
  if (warp == 0) {
    if (lane == 0)
      for (int k = 0; k < nbox; ++k) {
        const int slot = k % RS;
        mbar_wait(&empty[slot], ((k / RS) & 1) ^ 1);
        mbar_arrive_expect_tx(&full[slot], box_bytes);
        const int r = ((blockIdx.x * 7 + k) * row_step) % rows_total;
        tma_load_2d(smem_u32(smem + slot * 16384), &tm, &full[slot], 0, r);
      }
  } else {
    for (int k = 0; k < nbox; ++k) {
      const int slot = k % RS;
      mbar_wait(&full[slot], (k / RS) & 1);
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[slot]);
    }
    if (lane == 0) cyc[blockIdx.x] = clock64() - t0;
  }
}

int main() {
  void* fn = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  if (!fn) { printf("no encoder\n"); return 1; }
  auto enc = (PFN_cuTensorMapEncodeTiled_v12000)fn;
  const size_t bytes = 64ull << 20;  // 64 MB: L2-resident
  float* buf; cudaMalloc(&buf, bytes); cudaMemset(buf, 0, bytes);
  long long* cyc; cudaMalloc(&cyc, 148 * 8);
  struct Shape { const char* name; int row_floats, pitch_floats, rows, start; };
  Shape shapes[] = {
      {"32 rows x 128B aligned (filter box)", 32, 4096, 32, 0},
      {"32 rows x 128B, rows 128B apart (contiguous 4KB)", 32, 32, 32, 0},
      {"16 rows x 256B aligned", 64, 4096, 16, 0},
      {"8 rows x 512B aligned", 128, 4096, 8, 0},
      {"32 rows x 144B (input box, s=1)", 36, 3136, 32, 0},
      {"32 rows x 272B (input box, s=2)", 68, 3136, 32, 0},
      {"64 rows x 128B aligned (8KB)", 32, 4096, 64, 0},
      {"128 rows x 128B aligned (16KB)", 32, 4096, 128, 0},
      {"32 rows x 256B aligned (8KB)", 64, 4096, 32, 0},
  };
  for (auto& sh : shapes) {
    CUtensorMap tm;
    const cuuint64_t rows_total = bytes / 4 / sh.pitch_floats;
    cuuint64_t dims[2] = {(cuuint64_t)sh.pitch_floats, rows_total};
    cuuint64_t strides[1] = {(cuuint64_t)sh.pitch_floats * 4};
    cuuint32_t box[2] = {(cuuint32_t)sh.row_floats, (cuuint32_t)sh.rows}, es[2] = {1, 1};
    CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, buf, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r) { printf("%s: encode %d\n", sh.name, (int)r); continue; }
    const int box_bytes = sh.row_floats * sh.rows * 4;
    const int nbox = 2000;
    const size_t smem = 8 * 16384 + 1024 + 256;
    cudaFuncSetAttribute(rate<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    for (int it = 0; it < 2; ++it) {
      cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
      cudaEventRecord(e0);
      rate<8><<<148, 64, smem>>>(tm, nbox, box_bytes, (int)(rows_total - sh.rows), 97, cyc);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      long long h[148]; cudaMemcpy(h, cyc, sizeof h, cudaMemcpyDeviceToHost);
      double mc = 0; for (int i = 0; i < 148; ++i) mc += h[i]; mc /= 148;
      if (it == 1)
        printf("%-50s box %5d B: %6.1f B/clk/SM  %7.1f GB/s total  %5.1f clk/row (%s)\n", sh.name, box_bytes,
               (double)box_bytes * nbox / mc, (double)box_bytes * nbox * 148 / (ms * 1e-3) / 1e9,
               mc / nbox / sh.rows, cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
