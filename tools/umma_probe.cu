// umma_probe.cu -- standalone probe of tcgen05 kind::tf32 operand layouts (debug tool).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 tools/umma_probe.cu -o /tmp/umma_probe
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>

#include "../paper_2005_06410_b200/csrc/common.cuh"

using namespace cgb;

// A: 128 x 32 (K-major SW128). B: N x 32. mode 0: B K-major SW128, mode 1: B MN-major SW128.
// a_row_shift: A descriptor starts `shift` rows later (tests row-shifted descriptors),
// base_off_mode: 0 = base offset 0, 1 = (addr >> 7) & 7.
template <int N>
__global__ void probe(const float* A, const float* B, float* D, int mode, int a_row_shift, int base_off_mode,
                      int use_idesc_m) {
  extern __shared__ uint8_t raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sa = smem;                 // 256 rows * 128 B = 32 KB (room for shifts)
  uint8_t* sb = smem + 32768;         // N * 128 B
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_holder;
  const int tid = threadIdx.x;
  // fill A rows 0..255 (row r holds A[(r - a_row_shift)] for r >= shift)
  for (int i = tid; i < 256 * 32; i += blockDim.x) {
    const int r = i / 32, k = i % 32;
    const int src = r - a_row_shift;
    const float v = (src >= 0 && src < 128) ? A[src * 32 + k] : 0.0f;
    const uint32_t off = r * 128 + (((k / 4) ^ (r & 7)) << 4) + (k % 4) * 4;
    *reinterpret_cast<float*>(sa + off) = v;
  }
  // fill B
  for (int i = tid; i < N * 32; i += blockDim.x) {
    const int n = i / 32, k = i % 32;
    const float v = B[n * 32 + k];
    uint32_t off;
    if (mode == 0) {  // K-major: row n, 32 k per row
      off = n * 128 + (((k / 4) ^ (n & 7)) << 4) + (k % 4) * 4;
    } else if (mode == 1) {  // MN-major: row k (128 B = 32 n), 32-n blocks 4096 B apart
      const int nb = n / 32, nn = n % 32;
      off = nb * 4096 + k * 128 + (((nn / 4) ^ (k & 7)) << 4) + (nn % 4) * 4;
    } else {  // MN-major, 128B swizzle with 32-byte atoms: Swizzle<2,5,2>
      const int nb = n / 32, nn = n % 32;
      const uint32_t lin = nb * 4096 + k * 128 + nn * 4;
      off = lin ^ (((lin >> 7) & 3) << 5);
    }
    *reinterpret_cast<float*>(sb + off) = v;
  }
  fence_proxy_async_smem();
  if (tid == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  if (tid < 32) tmem_alloc(&tmem_holder, N < 32 ? 32 : N);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_holder;
  if (tid < 32 && elect_one()) {
    uint32_t idesc = idesc_tf32(N, false, mode >= 1);
    if (!use_idesc_m) idesc &= ~(0x1Fu << 24);
    for (int kk = 0; kk < 4; ++kk) {
      const uint32_t a_addr = smem_u32(sa) + a_row_shift * 128 + kk * 32;
      const uint32_t bo = base_off_mode ? ((a_addr >> 7) & 7) : 0;
      const uint64_t ad = smem_desc(a_addr, 16, 1024, bo);
      uint64_t bd;
      if (mode == 0) bd = smem_desc(smem_u32(sb) + kk * 32, 16, 1024);
      else if (mode == 1) bd = smem_desc(smem_u32(sb) + kk * 1024, 4096, 1024);
      else if (mode == 2) bd = smem_desc(smem_u32(sb) + kk * 1024, 4096, 512, 0, kLayoutSW128_32B);
      else bd = smem_desc(smem_u32(sb) + kk * 1024, 512, 4096, 0, kLayoutSW128_32B);
      mma_tf32(tmem, ad, bd, idesc, kk > 0);
    }
    mma_commit(&bar);
  }
  __syncwarp();
  mbar_wait(&bar, 0);
  tc_fence_after();
  const int w = tid / 32;
  for (int cb = 0; cb < N / 32; ++cb) {
    uint32_t r[32];
    tmem_ld_32x32b_x32(tmem + ((uint32_t)(w * 32) << 16) + cb * 32, r);
    tmem_ld_wait();
    for (int j = 0; j < 32; ++j) D[(w * 32 + (tid % 32)) * N + cb * 32 + j] = __uint_as_float(r[j]);
  }
  tc_fence_before();
  __syncthreads();
  if (tid < 32) {
    tc_fence_after();
    tmem_dealloc(tmem, N < 32 ? 32 : N);
  }
}

int main() {
  constexpr int N = 64;
  std::vector<float> A(128 * 32), B(N * 32), D(128 * N), R(128 * N);
  srand(1);
  for (auto& x : A) x = (float)(rand() % 17 - 8);
  for (auto& x : B) x = (float)(rand() % 13 - 6);
  for (int m = 0; m < 128; ++m)
    for (int n = 0; n < N; ++n) {
      double s = 0;
      for (int k = 0; k < 32; ++k) s += (double)A[m * 32 + k] * B[n * 32 + k];
      R[m * N + n] = (float)s;
    }
  float *dA, *dB, *dD;
  cudaMalloc(&dA, A.size() * 4);
  cudaMalloc(&dB, B.size() * 4);
  cudaMalloc(&dD, D.size() * 4);
  cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(probe<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, 80 * 1024);
  struct T { int mode, shift, bom, m; };
  T tests[] = {{0, 0, 0, 1}, {1, 0, 0, 1}, {2, 0, 0, 1}, {3, 0, 0, 1}, {2, 13, 0, 1}};
  for (auto t : tests) {
    cudaMemset(dD, 0, D.size() * 4);
    probe<N><<<1, 128, 80 * 1024>>>(dA, dB, dD, t.mode, t.shift, t.bom, t.m);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("mode %d: CUDA error %s\n", t.mode, cudaGetErrorString(e)); return 1; }
    cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
    int bad = 0, zeros = 0;
    double maxerr = 0;
    for (int i = 0; i < 128 * N; ++i) {
      maxerr = fmax(maxerr, fabs(D[i] - R[i]));
      bad += D[i] != R[i];
      zeros += D[i] == 0;
    }
    printf("B %s  a_row_shift=%2d base_off=%d : mismatches %d/%d zeros %d maxerr %g  D[0..3]=%g %g %g %g ref %g %g %g %g\n",
           t.mode == 0 ? "K-major   " : (t.mode == 1 ? "MN-major16" : (t.mode == 2 ? "MN-32B-a  " : "MN-32B-b  ")), t.shift, t.bom, bad, 128 * N, zeros, maxerr, D[0], D[1], D[2], D[3],
           R[0], R[1], R[2], R[3]);
  }
  return 0;
}
