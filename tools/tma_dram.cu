// tma_dram.cu -- TMA tensor-load throughput from DRAM for the raw-input pattern (debug tool).
// I viewed as (pixels = 3136, channel rows = c*b): CTA i streams "chunks" of NB consecutive
// boxes (box_px pixels x box_rows channel rows) into a ring of RS 8 KB slots; a consumer
// warp frees slots as they land. Reports GB/s. Pattern knobs: box shape, ring depth.
#include <cstdio>
#include <cstdlib>
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include "../paper_2005_06410_b200/csrc/common.cuh"
using namespace cgb;

__global__ void __launch_bounds__(64, 1) stream(const __grid_constant__ CUtensorMap tm, int nchunks, int nb, int box_px,
                                               int box_rows, int rows_total, int rs) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + rs * 8192);
  uint64_t* empty = full + rs;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    for (int i = 0; i < rs; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 1); }
    fence_mbar_init();
  }
  __syncthreads();
  const int total = nchunks * nb;
  if (warp == 0) {
    if (lane == 0)
      for (int k = 0; k < total; ++k) {
        const int slot = k % rs;
        mbar_wait(&empty[slot], ((k / rs) & 1) ^ 1);
        mbar_arrive_expect_tx(&full[slot], box_px * box_rows * 4);
        const int chunk = blockIdx.x + gridDim.x * (k / nb);
        const int row0 = (chunk * box_rows * 4) % (rows_total - box_rows);  // channel-row block of this chunk
        const int px0 = ((chunk * 5) % 40) * 64 + (k % nb) * box_px;
        tma_load_2d(smem_u32(smem + slot * 8192), &tm, &full[slot], px0, row0);
      }
  } else {
    for (int k = 0; k < total; ++k) {
      const int slot = k % rs;
      mbar_wait(&full[slot], (k / rs) & 1);
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[slot]);
    }
  }
}

int main() {
  void* fn = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  if (!fn) { printf("no encoder\n"); return 1; }
  auto enc = (PFN_cuTensorMapEncodeTiled_v12000)fn;
  const int plane = 3136, rows = 128 * 128 * 4;  // 822 MB: DRAM-resident
  float* buf; cudaMalloc(&buf, (size_t)plane * rows * 4); cudaMemset(buf, 0, (size_t)plane * rows * 4);
  struct S { int px, rows, nb, rs; };
  S shapes[] = {{64, 32, 13, 16}, {64, 32, 13, 24}, {64, 32, 26, 24}, {128, 16, 13, 24}, {256, 8, 13, 24},
                {32, 64, 13, 24}, {64, 32, 13, 8}};
  for (auto& sh : shapes) {
    CUtensorMap tm;
    cuuint64_t dims[2] = {(cuuint64_t)plane, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)plane * 4};
    cuuint32_t box[2] = {(cuuint32_t)sh.px, (cuuint32_t)sh.rows}, es[2] = {1, 1};
    CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, buf, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r) { printf("encode %d\n", (int)r); continue; }
    const int nchunks = 40;
    const size_t smem = (size_t)sh.rs * 8192 + 1024 + 512;
    cudaFuncSetAttribute(stream, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    float best = 1e9;
    for (int it = 0; it < 3; ++it) {
      cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
      cudaEventRecord(e0);
      stream<<<148, 64, smem>>>(tm, nchunks, sh.nb, sh.px, sh.rows, rows, sh.rs);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1); best = ms < best ? ms : best;
    }
    const double bytes = 148.0 * nchunks * sh.nb * sh.px * sh.rows * 4;
    printf("box %3d px x %2d rows, %2d boxes/chunk, ring %2d: %7.1f GB/s  %.1f GB/s/SM (%s)\n", sh.px, sh.rows, sh.nb,
           sh.rs, bytes / (best * 1e-3) / 1e9, bytes / (best * 1e-3) / 1e9 / 148, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
