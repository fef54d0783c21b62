// umma_bench.cu -- throughput of tcgen05.mma kind::tf32 per shape / operand layout (debug tool).
// One CTA per SM, each issues `iters` MMAs into TMEM from fixed smem operands; reports
// cycles per MMA and the implied chip TFLOPS.
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_2005_06410_b200/csrc/common.cuh"

using namespace cgb;

template <int N>
__global__ void __launch_bounds__(128, 1) bench(int iters, int a_shift_rows, int b_kmajor, int a_tmem_unused,
                                                 long long* cycles) {
  extern __shared__ uint8_t raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sa = smem;          // 64 KB of A rows
  uint8_t* sb = smem + 65536;  // B
  __shared__ uint64_t bar, bar2, rot[16];
  __shared__ uint32_t tmem_holder;
  const int tid = threadIdx.x;
  for (int i = tid; i < (65536 + N * 128) / 4; i += blockDim.x) reinterpret_cast<float*>(smem)[i] = 1.0f / (1 + (i & 7));
  fence_proxy_async_smem();
  if (tid == 0) {
    mbar_init(&bar, 1);
    mbar_init(&bar2, 1);
    for (int i = 0; i < 16; ++i) mbar_init(&rot[i], 1);
    fence_mbar_init();
  }
  if (tid < 32) tmem_alloc(&tmem_holder, N < 32 ? 64 : 2 * N);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_holder;
  if (tid < 32 && elect_one()) {
    const uint32_t idesc = idesc_tf32(N, false, !b_kmajor);
    const uint64_t bd = b_kmajor ? smem_desc(smem_u32(sb), 16, 1024)
                                 : smem_desc(smem_u32(sb), 4096, 512, 0, kLayoutSW128_32B);
    long long t0 = clock64();
    const int bvary = a_tmem_unused & 1, dvary = (a_tmem_unused >> 1) & 1, afix = (a_tmem_unused >> 2) & 1;
    for (int it = 0; it < iters; ++it) {
      const uint32_t row = (it * a_shift_rows) & 127;
      const uint64_t ad = afix ? smem_desc(smem_u32(sa), 16, 1024)
                               : smem_desc(smem_u32(sa) + row * 128 + (it & 3) * 32, 16, 1024);
      const uint64_t bdd = bvary ? bd + (uint64_t)((it & 3) * 2) : bd;
      const uint32_t dd = dvary ? tmem + (it & 1) * N : tmem;
      mma_tf32(dd, ad, bdd, idesc, it > 1);
      const int cevery = (a_tmem_unused >> 4) & 255, nrot = a_tmem_unused >> 12;
      if (cevery && (it % cevery) == cevery - 1) mma_commit(nrot ? &rot[(it / cevery) % nrot] : &bar2);
    }
    mma_commit(&bar);
    mbar_wait(&bar, 0);
    long long t1 = clock64();
    cycles[blockIdx.x] = t1 - t0;
  }
  __syncwarp();
  tc_fence_before();
  __syncthreads();
  if (tid < 32) {
    tc_fence_after();
    tmem_dealloc(tmem, N < 32 ? 64 : 2 * N);
  }
}

template <int N>
void run(int iters, int shift, int bk, const char* name, int mode = 0) {
  long long* d;
  cudaMalloc(&d, 148 * sizeof(long long));
  cudaFuncSetAttribute(bench<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  bench<N><<<148, 128, 200 * 1024>>>(iters, shift, bk, mode, d);
  cudaError_t e = cudaDeviceSynchronize();
  std::vector<long long> h(148);
  cudaMemcpy(h.data(), d, 148 * 8, cudaMemcpyDeviceToHost);
  long long mx = 0;
  double avg = 0;
  for (auto x : h) { mx = x > mx ? x : mx; avg += x / 148.0; }
  const double cyc = avg / iters;
  const double flops_per_mma = 2.0 * 128 * N * 8;
  // chip TFLOPS at 1.9 GHz
  printf("%-40s N=%3d  %s  cycles/MMA %.2f  (ideal %.1f)  -> %.0f TFLOPS @1.9GHz\n", name, N,
         e == cudaSuccess ? "ok " : cudaGetErrorString(e), cyc, 128.0 * N / 256.0,
         flops_per_mma / cyc * 1.9e9 * 148 / 1e12);
  cudaFree(d);
}

int main() {
  const int it = 4096;
  run<64>(it, 1, 1, "A,B vary, D alternates 2 accs", 3);
  run<128>(it, 1, 1, "A,B vary, D alternates 2 accs", 3);
  run<128>(it, 1, 1, "A,B vary, commit every 8", 1 | (8 << 4));
  run<128>(it, 1, 1, "A,B vary, D alt, commit every 8", 3 | (8 << 4));
  run<64>(it, 1, 1, "A,B vary, D alt, commit every 16", 3 | (16 << 4));
  run<256>(it, 1, 1, "A,B vary, commit every 4", 1 | (4 << 4));
  // commit every 8 MMAs (N=128): same barrier vs a ring of 2/3/4/8 barriers
  for (int nrot : {0, 2, 3, 4, 8, 16})
    run<128>(it, 1, 0, nrot ? "commit every 8, ring of barriers" : "commit every 8, one barrier", 3 | (8 << 4) | (nrot << 12));
  for (int nrot : {0, 3, 8})
    run<256>(it, 1, 0, nrot ? "commit every 4, ring" : "commit every 4, one barrier", 3 | (4 << 4) | (nrot << 12));
  return 0;
}
