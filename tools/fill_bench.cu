// fill_bench.cu -- window-fill throughput: register-staged LDG producers vs a TMA-fed
// raw ring + shared-memory transpose (debug tool, not product code).
//
// Work item = one 32-row box of one phase plane of one padded column x 32 channels: rows
// hq = 0..31 hold input (h = s*hq + a - p, w = s*wq + c - p) of image bb, channels
// 32*cc..+32. Each item ends as 32 K-major, 128B-swizzled 128-byte rows in a window
// buffer (what the shifted-window kernel's producers write).
//   mode 0: warp per item, lane = row, 32 LDG.32 (channel planes) then 8 STS.128.
//   mode 1: one thread streams the items' boxes by TMA (4-D map, element strides s,s,1,1,
//           zero fill = the padding) into a ring of RS 4 KB slots; warp (slot % NW) reads
//           its row across the 32 channel rows (32 LDS.32) and writes 8 STS.128.
//   mode 2: mode 0 plus prefetch.global.L2 of the item the warp handles next.
// Checks that modes 0 and 1 produce the same window checksum.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include "../paper_2005_06410_b200/csrc/common.cuh"

using namespace cgb;
constexpr int SLOT = 9216;  // raw slot: 32 channels x (64 + 4) floats, 128-byte aligned

struct P {
  int h_i, w_i, c_i, b, s, p, Hq, Wq, nph, CC;
  int ncol;        // padded columns per window (one CTA tile's window)
  int nb_ldg;      // 32-lane units per column and phase (LDG mode)
  int nb_tma;      // TMA boxes per column and phase (32*s + 4 rows each)
  int windows;     // total windows
  long items;      // total LDG items (for the byte count)
};

// Window-major order like the conv kernel: a CTA stages window w (ncol consecutive
// padded columns) for chunk cc, items in row order within each w-phase plane.
__device__ __forceinline__ void item_ldg(const P& a, int w, int j, int& col, int& pc, int& bx) {
  bx = j % a.nb_ldg; j /= a.nb_ldg;
  col = w * a.ncol + j % a.ncol; j /= a.ncol;
  pc = j;
}
__device__ __forceinline__ void item_tma(const P& a, int w, int j, int& col, int& pc, int& bx) {
  bx = j % a.nb_tma; j /= a.nb_tma;
  col = w * a.ncol + j % a.ncol; j /= a.ncol;
  pc = j;
}

template <int NW, int RS>
__global__ void __launch_bounds__((NW + 1) * 32, 1)
    fill(const __grid_constant__ CUtensorMap tm, const float* __restrict__ I, P a, int mode,
         unsigned long long* sum) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* ring = smem;                       // RS x 4 KB
  uint8_t* win = smem + RS * SLOT;            // NW x 4 KB window rows
  uint64_t* full = reinterpret_cast<uint64_t*>(win + NW * 4096);
  uint64_t* empty = full + RS;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  constexpr int SPW = RS / NW;
  static_assert(RS % NW == 0, "each consumer warp owns RS / NW slots");
  if (threadIdx.x == 0) {
    for (int i = 0; i < RS; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 1); }
    fence_mbar_init();
  }
  __syncthreads();
  const long first = blockIdx.x, step = gridDim.x;
  const int plane = a.h_i * a.w_i;
  unsigned long long acc = 0;
  if (mode == 1) {
    if (warp == NW) {
      if (lane == 0) {
        int k = 0;
        const int ipw = a.nph * a.ncol * a.nb_tma;
        for (int w = blockIdx.x; w < a.windows; w += gridDim.x)
          for (int cc = 0; cc < a.CC; ++cc)
            for (int jj = 0; jj < ipw; ++jj, ++k) {
              const int j = k / NW, slot = (k % NW) * SPW + j % SPW;
              mbar_wait(&empty[slot], ((j / SPW) & 1) ^ 1);
              int col, pc, bx;
              item_tma(a, w, jj, col, pc, bx);
              const int wq = col % a.Wq, bb = col / a.Wq;
              // dim-0 box starts must be 16-byte aligned: start 4-aligned below, 4 extra rows
              const int h0 = 32 * a.s * bx - a.p, h0a = h0 >= 0 ? h0 & ~3 : -((-h0 + 3) & ~3);
              mbar_arrive_expect_tx(&full[slot], 32 * (32 * a.s + 4) * 4);
              tma_load_4d(smem_u32(ring + slot * SLOT), &tm, &full[slot], h0a, a.s * wq + pc - a.p, 32 * cc, bb);
            }
      }
    } else {
      int k = 0;
      const int ipw = a.nph * a.ncol * a.nb_tma;
      for (int w = blockIdx.x; w < a.windows; w += gridDim.x)
        for (int cc = 0; cc < a.CC; ++cc)
          for (int jj = 0; jj < ipw; ++jj, ++k) {
        if (k % NW != warp) continue;
        const int j = k / NW, slot = warp * SPW + j % SPW;
        mbar_wait(&full[slot], (j / SPW) & 1);
        const uint32_t dst = smem_u32(win + warp * 4096);
        int col, pc, bx;
        item_tma(a, w, jj, col, pc, bx);
        const int h0 = 32 * a.s * bx - a.p, h0a = h0 >= 0 ? h0 & ~3 : -((-h0 + 3) & ~3);
        const int RW = 32 * a.s + 4;  // raw row (one channel) in floats
        const uint32_t src = smem_u32(ring + slot * SLOT) + (h0 - h0a) * 4;
        if (a.s == 1) {
          float v[32];
#pragma unroll
          for (int c = 0; c < 32; ++c) v[c] = lds_f32(src + (c * RW + lane) * 4);
#pragma unroll
          for (int ch = 0; ch < 8; ++ch)
            st_shared_v4(dst + lane * 128 + ((ch ^ (lane & 7)) << 4), v[4 * ch], v[4 * ch + 1], v[4 * ch + 2],
                         v[4 * ch + 3]);
          acc += __float_as_uint(v[lane]) + __float_as_uint(v[(lane + 7) & 31]);
        } else {
#pragma unroll
          for (int half = 0; half < 2; ++half) {
            float v0[16], v1[16];
#pragma unroll
            for (int c = 0; c < 16; ++c) {
              v0[c] = lds_f32(src + ((16 * half + c) * RW + 2 * lane) * 4);
              v1[c] = lds_f32(src + ((16 * half + c) * RW + 2 * lane + 1) * 4);
            }
#pragma unroll
            for (int ch = 0; ch < 4; ++ch) {
              const int q = 4 * half + ch;
              st_shared_v4(dst + lane * 128 + ((q ^ (lane & 7)) << 4), v0[4 * ch], v0[4 * ch + 1], v0[4 * ch + 2],
                           v0[4 * ch + 3]);
              st_shared_v4(dst + lane * 128 + ((q ^ (lane & 7)) << 4), v1[4 * ch], v1[4 * ch + 1],
                           v1[4 * ch + 2], v1[4 * ch + 3]);
            }
            acc += __float_as_uint(v0[lane & 15]) + __float_as_uint(v1[(lane + 7) & 15]);
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[slot]);
      }
    }
  } else if (warp < NW) {  // modes 0, 2, 3
    int k = 0;
    const int ipw = a.nph * a.ncol * a.nb_ldg;
    for (int w = blockIdx.x; w < a.windows; w += gridDim.x)
      for (int cc = 0; cc < a.CC; ++cc)
        for (int jj = warp; jj < ipw; jj += NW, ++k) {
      int col, pc, bx;
      item_ldg(a, w, jj, col, pc, bx);
      const int wq = col % a.Wq, bb = col / a.Wq;
      // kernel lane mapping: stride 2 -> lanes cover 16 rows x both h phases = 32 consecutive h
      const int row = a.s == 2 ? (lane & 7) + 8 * (lane >> 4) + 16 * bx : lane + 32 * bx;
      const int pa = a.s == 2 ? (lane >> 3) & 1 : 0;
      const int h = a.s * row + pa - (mode == 3 ? 0 : a.p), wi = a.s * wq + pc - a.p;  // mode 3: 128B-aligned runs
      const bool ok = row < a.Hq && (unsigned)h < (unsigned)a.h_i && (unsigned)wi < (unsigned)a.w_i;
      const float* src = I + ((long)bb * a.c_i + 32L * cc) * plane + (long)wi * a.h_i + h;
      float v[32];
#pragma unroll
      for (int c = 0; c < 32; ++c) v[c] = ok ? __ldg(src + (long)c * plane) : 0.0f;
      const uint32_t dst = smem_u32(win + warp * 4096);
#pragma unroll
      for (int ch = 0; ch < 8; ++ch)
        st_shared_v4(dst + lane * 128 + ((ch ^ (lane & 7)) << 4), v[4 * ch], v[4 * ch + 1], v[4 * ch + 2],
                     v[4 * ch + 3]);
      acc += __float_as_uint(v[lane]) + __float_as_uint(v[(lane + 7) & 31]);
    }
  }
  atomicAdd(sum, acc);
}

static PFN_cuTensorMapEncodeTiled_v12000 encoder() {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  if (e != cudaSuccess || !fn) { printf("no cuTensorMapEncodeTiled: %s\n", cudaGetErrorString(e)); exit(1); }
  return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
}

template <int NW, int RS>
void run(const char* name, const float* I, P a, int mode, int mtimes) {
  CUtensorMap tm;
  cuuint64_t dims[4] = {(cuuint64_t)a.h_i, (cuuint64_t)a.w_i, (cuuint64_t)a.c_i, (cuuint64_t)a.b};
  cuuint64_t strides[3] = {(cuuint64_t)a.h_i * 4, (cuuint64_t)a.h_i * a.w_i * 4,
                           (cuuint64_t)a.c_i * a.h_i * a.w_i * 4};
  cuuint32_t box[4] = {(cuuint32_t)(32 * a.s + 4), 1, 32, 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = encoder()(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<float*>(I), dims, strides, box, estr,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                         CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) { printf("%s: tensor map encode failed %d\n", name, (int)r); return; }
  // pad to 200 KB like the conv kernel (sets the same L1 carve-out)
  const size_t smem = std::max<size_t>(RS * SLOT + NW * 4096 + 2 * RS * 8 + 1024, 200 * 1024);
  auto k = fill<NW, RS>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  unsigned long long* sum;
  cudaMalloc(&sum, 8);
  cudaMemset(sum, 0, 8);
  k<<<148, (NW + 1) * 32, smem>>>(tm, I, a, mode, sum);  // warm
  if (cudaDeviceSynchronize() != cudaSuccess) { printf("%s: %s\n", name, cudaGetErrorString(cudaGetLastError())); exit(1); }
  unsigned long long h0 = 0;
  cudaMemcpy(&h0, sum, 8, cudaMemcpyDeviceToHost);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  float best = 1e30f;
  for (int t = 0; t < mtimes; ++t) {
    cudaEventRecord(e0);
    k<<<148, (NW + 1) * 32, smem>>>(tm, I, a, mode, sum);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    best = ms < best ? ms : best;
  }
  const double bytes = (double)a.items * a.nph * a.Hq * 128;  // useful window rows
  printf("%-28s NW=%2d RS=%2d smem=%3zu KB: %8.1f us  %7.1f GB/s of window  checksum %llx  (%s)\n", name, NW, RS,
         smem / 1024, best * 1e3, bytes / (best * 1e-3) / 1e9, h0, cudaGetErrorString(cudaGetLastError()));
  cudaFree(sum);
}

int main(int argc, char** argv) {
  const bool only_tma = argc > 2;
  // default: the stride-2 56->28 c128 layer at b=128; "s1" selects 56x56 c64 stride 1
  setvbuf(stdout, nullptr, _IONBF, 0);
  const bool s1 = argc > 1 && argv[1][0] == 's' && argv[1][1] == '1';
  const int batch = getenv("FB_BATCH") ? atoi(getenv("FB_BATCH")) : 128;
  P a;
  if (s1) { a.h_i = a.w_i = 56; a.c_i = 64; a.b = batch; a.s = 1; a.p = 1; a.Hq = 57; a.Wq = 57; a.ncol = 11;
             a.nb_ldg = 2; a.nb_tma = 2; }
  else    { a.h_i = a.w_i = 56; a.c_i = 128; a.b = batch; a.s = 2; a.p = 1; a.Hq = 29; a.Wq = 29; a.ncol = 6;
             a.nb_ldg = 2; a.nb_tma = 1; }
  a.nph = a.s; a.CC = a.c_i / 32;
  a.windows = a.b * a.Wq / a.ncol;
  a.items = (long)a.windows * a.CC * a.nph * a.ncol;  // (column, w-phase, chunk) triples
  const size_t n = (size_t)a.h_i * a.w_i * a.c_i * a.b;
  float* I;
  cudaMalloc(&I, n * 4);
  std::vector<float> h(n);
  for (size_t i = 0; i < n; ++i) h[i] = (float)((i * 2654435761u) % 1000) * 1e-3f;
  cudaMemcpy(I, h.data(), n * 4, cudaMemcpyHostToDevice);
  printf("geometry %s: input %.1f MB, %.1f MB of window\n", s1 ? "56x56 c64 s1" : "56->28 c128 s2", n * 4 / 1e6,
         a.items * a.nph * a.Hq * 128 / 1e6);
  if (!only_tma) {
    run<12, 12>("LDG aligned (mode 3)", I, a, 3, 5);
    run<12, 12>("LDG (mode 0)", I, a, 0, 5);
    run<16, 16>("LDG (mode 0)", I, a, 0, 5);
  }
  run<12, 12>("TMA ring (mode 1)", I, a, 1, 5);
  run<8, 8>("TMA ring (mode 1)", I, a, 1, 5);
  run<8, 16>("TMA ring (mode 1)", I, a, 1, 5);
  run<6, 18>("TMA ring (mode 1)", I, a, 1, 5);
  run<4, 16>("TMA ring (mode 1)", I, a, 1, 5);
  run<4, 20>("TMA ring (mode 1)", I, a, 1, 5);
  return 0;
}
