// simt_kernels.cu -- CUDA-core kernels of the B200 convolution operator:
//   K1 im2col_kernel      explicit lowering (replaces im2col<float>, im2col.hpp:77-120)
//   K4 ffma_conv_kernel   fp32 FFMA implicit/explicit GEMM for degenerate low-K layers
//                         (replaces microkernel_generic's role, microkernel.hpp:40-59)
//   K5 filter_prep_kernel TF32 hi/lo split of the filters for 3xTF32 (no reference equivalent)
#include <algorithm>

#include "internal.h"

namespace cgb {

// ============================================================================ K1
// One thread writes 4 consecutive rows r..r+3 of one lowered column c (a float4 when
// ldb % 4 == 0). Column c = i_h + i_w*h_o + i_b*h_o*w_o, row r = i_kh + i_kw*k_h +
// i_c*k_h*k_w; the value is I(i_h*s+i_kh-p, i_w*s+i_kw-p, i_c, i_b) or +0 in the
// padding (im2col.hpp:71-76). Pure data movement, hence bit-exact. Writes are fully
// coalesced along r (the column is contiguous, ld = ldb); reads hit L1/L2 since the
// k_h*k_w taps of neighbouring columns overlap.
struct Im2colArgs {
  int32_t k_h, k_w, c_i, h_i, w_i, s, p, h_o, w_o, K;
  int64_t n, ldb, plane;
};

template <bool VEC>
__global__ void __launch_bounds__(256) im2col_kernel(const float* __restrict__ I, float* __restrict__ B,
                                                     Im2colArgs a) {
  const int64_t chunks = (a.ldb + 3) / 4;
  const int64_t total = chunks * a.n;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t col = idx / chunks;
    const int32_t r0 = static_cast<int32_t>(idx - col * chunks) * 4;
    const int32_t hw = a.h_o * a.w_o;
    const int32_t i_b = static_cast<int32_t>(col / hw);
    const int32_t rem = static_cast<int32_t>(col - (int64_t)i_b * hw);
    const int32_t i_w = rem / a.h_o, i_h = rem - i_w * a.h_o;
    const int32_t h0 = i_h * a.s - a.p, w0 = i_w * a.s - a.p;
    int32_t kh = r0 % a.k_h;
    int32_t t = r0 / a.k_h;
    int32_t kw = t % a.k_w;
    int32_t c = t / a.k_w;
    const float* img = I + (int64_t)i_b * a.c_i * a.plane;
    float v[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int32_t r = r0 + e;
      const int32_t hh = h0 + kh, ww = w0 + kw;
      float x = 0.0f;
      if (r < a.K && (unsigned)hh < (unsigned)a.h_i && (unsigned)ww < (unsigned)a.w_i)
        x = __ldg(img + c * a.plane + (int64_t)ww * a.h_i + hh);
      v[e] = x;
      if (++kh == a.k_h) {
        kh = 0;
        if (++kw == a.k_w) { kw = 0; ++c; }
      }
    }
    float* dst = B + col * a.ldb + r0;
    if (VEC) {
      *reinterpret_cast<float4*>(dst) = make_float4(v[0], v[1], v[2], v[3]);
    } else {
#pragma unroll
      for (int e = 0; e < 4; ++e)
        if (r0 + e < a.ldb) dst[e] = v[e];
    }
  }
}

cudaError_t launch_im2col(const float* I, float* B, int64_t ldb, const ConvGeom& g, cudaStream_t st) {
  Im2colArgs a;
  a.k_h = (int32_t)g.k_h; a.k_w = (int32_t)g.k_w; a.c_i = (int32_t)g.c_i; a.h_i = (int32_t)g.h_i;
  a.w_i = (int32_t)g.w_i; a.s = (int32_t)g.s; a.p = (int32_t)g.p; a.h_o = (int32_t)g.h_o; a.w_o = (int32_t)g.w_o;
  a.K = (int32_t)g.k; a.n = g.n; a.ldb = ldb; a.plane = g.h_i * g.w_i;
  const int64_t total = ((ldb + 3) / 4) * g.n;
  const int64_t blocks = std::min<int64_t>((total + 255) / 256, 148 * 16);
  const bool vec = (ldb % 4 == 0) && (reinterpret_cast<uintptr_t>(B) % 16 == 0);
  if (vec)
    im2col_kernel<true><<<(unsigned)blocks, 256, 0, st>>>(I, B, a);
  else
    im2col_kernel<false><<<(unsigned)blocks, 256, 0, st>>>(I, B, a);
  count_launch();
  return cudaGetLastError();
}

// ============================================================================ K4
// Tile: 128 output pixels x 64 filters x 16 rows of K per step, 256 threads,
// 8 pixels x 4 filters of fp32 FMA accumulators per thread. The A operand (lowered
// matrix) is gathered from I (implicit) or read from B (explicit) into shared
// memory; the filter block is read coalesced along k_n. O is written k_n-fastest
// (tensor.hpp:108-113: Chat = O as k_n x n, ld = k_n).
namespace ffma {
constexpr int BM = 128, BN = 64, BK = 16, THREADS = 256;

struct Args {
  int32_t k_n, k_h, k_w, c_i, h_i, w_i, s, p, h_o, w_o, K;
  int64_t n, ldb, plane;
};

// Min blocks per SM: unset for the implicit kernel (80 registers, unchanged SASS); 2 for
// the explicit one, which needs 96 (at the default 64-register allocation it spilled).
template <bool EXPLICIT>
__global__ void __launch_bounds__(THREADS, EXPLICIT ? 2 : 0) ffma_conv_kernel(const float* __restrict__ F,
                                                            const float* __restrict__ I,
                                                            const float* __restrict__ Bexp,
                                                            float* __restrict__ O, Args a) {
  __shared__ float As[BK][BM + 4];
  __shared__ __align__(16) float Bs[BK][BN + 4];
  const int tid = threadIdx.x;
  const int64_t m0 = (int64_t)blockIdx.x * BM;
  const int n0 = blockIdx.y * BN;

  // A loader: pixel row pl, k rows kr0..kr0+7
  const int pl = tid % BM;
  const int kr0 = (tid / BM) * 8;
  const int64_t P = m0 + pl;
  const bool p_ok = P < a.n;
  int32_t h0 = 0, w0 = 0;
  const float* img = I;
  if (!EXPLICIT && p_ok) {
    const int32_t hw = a.h_o * a.w_o;
    const int32_t i_b = (int32_t)(P / hw);
    const int32_t rem = (int32_t)(P - (int64_t)i_b * hw);
    const int32_t i_w = rem / a.h_o, i_h = rem - i_w * a.h_o;
    h0 = i_h * a.s - a.p;
    w0 = i_w * a.s - a.p;
    img = I + (int64_t)i_b * a.c_i * a.plane;
  }
  // B loader: filter column bn, k rows bk0..bk0+3
  const int bn = tid % BN;
  const int bk0 = (tid / BN) * 4;

  // compute mapping
  const int tx = tid % 16;  // 4 filters: tx*4 .. +3
  const int ty = tid / 16;  // 8 pixels: ty + 16*i

  float acc[8][4];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.0f;

  float av[8], bv[4];
  auto load_tile = [&](int k0) {
    if (EXPLICIT) {
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const int r = k0 + kr0 + e;
        av[e] = (p_ok && r < a.K) ? __ldg(Bexp + P * a.ldb + r) : 0.0f;
      }
    } else {
      int32_t r = k0 + kr0;
      int32_t kh = r % a.k_h;
      int32_t t = r / a.k_h;
      int32_t kw = t % a.k_w;
      int32_t c = t / a.k_w;
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const int32_t hh = h0 + kh, ww = w0 + kw;
        float x = 0.0f;
        if (p_ok && r + e < a.K && (unsigned)hh < (unsigned)a.h_i && (unsigned)ww < (unsigned)a.w_i)
          x = __ldg(img + c * a.plane + (int64_t)ww * a.h_i + hh);
        av[e] = x;
        if (++kh == a.k_h) {
          kh = 0;
          if (++kw == a.k_w) { kw = 0; ++c; }
        }
      }
    }
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int r = k0 + bk0 + e;
      const int nn = n0 + bn;
      bv[e] = (r < a.K && nn < a.k_n) ? __ldg(F + (int64_t)r * a.k_n + nn) : 0.0f;
    }
  };

  load_tile(0);
  for (int k0 = 0; k0 < a.K; k0 += BK) {
    __syncthreads();
#pragma unroll
    for (int e = 0; e < 8; ++e) As[kr0 + e][pl] = av[e];
#pragma unroll
    for (int e = 0; e < 4; ++e) Bs[bk0 + e][bn] = bv[e];
    __syncthreads();
    if (k0 + BK < a.K) load_tile(k0 + BK);
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      const float4 b4 = *reinterpret_cast<const float4*>(&Bs[kk][tx * 4]);
      const float bb[4] = {b4.x, b4.y, b4.z, b4.w};
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float x = As[kk][ty + 16 * i];
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(x, bb[j], acc[i][j]);
      }
    }
  }

  const int nb = n0 + tx * 4;
  const bool vec = (a.k_n % 4 == 0) && (nb + 3 < a.k_n);
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int64_t PP = m0 + ty + 16 * i;
    if (PP >= a.n) continue;
    float* dst = O + PP * a.k_n + nb;
    if (vec) {
      *reinterpret_cast<float4*>(dst) = make_float4(acc[i][0], acc[i][1], acc[i][2], acc[i][3]);
    } else {
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (nb + j < a.k_n) dst[j] = acc[i][j];
    }
  }
}
}  // namespace ffma

cudaError_t launch_ffma_conv(const float* F, const float* I, const float* explicit_src, int64_t ldb, float* O,
                             const ConvGeom& g, cudaStream_t st) {
  ffma::Args a;
  a.k_n = (int32_t)g.k_n; a.k_h = (int32_t)g.k_h; a.k_w = (int32_t)g.k_w; a.c_i = (int32_t)g.c_i;
  a.h_i = (int32_t)g.h_i; a.w_i = (int32_t)g.w_i; a.s = (int32_t)g.s; a.p = (int32_t)g.p;
  a.h_o = (int32_t)g.h_o; a.w_o = (int32_t)g.w_o; a.K = (int32_t)g.k;
  a.n = g.n; a.ldb = ldb; a.plane = g.h_i * g.w_i;
  dim3 grid((unsigned)((g.n + ffma::BM - 1) / ffma::BM), (unsigned)((g.k_n + ffma::BN - 1) / ffma::BN));
  if (explicit_src)
    ffma::ffma_conv_kernel<true><<<grid, ffma::THREADS, 0, st>>>(F, I, explicit_src, O, a);
  else
    ffma::ffma_conv_kernel<false><<<grid, ffma::THREADS, 0, st>>>(F, I, nullptr, O, a);
  count_launch();
  return cudaGetLastError();
}

// ============================================================================ K5
__global__ void __launch_bounds__(256) filter_prep_kernel(const float* __restrict__ F, float* __restrict__ hi,
                                                          float* __restrict__ lo, int64_t k_n, int64_t K,
                                                          int64_t ldf) {
  const int64_t total = ldf * K;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = idx / ldf;
    const int64_t nn = idx - r * ldf;
    const float f = nn < k_n ? __ldg(F + r * k_n + nn) : 0.0f;
    if (lo) {
      const float h = to_tf32(f);
      hi[idx] = h;
      lo[idx] = to_tf32(f - h);
    } else {
      hi[idx] = f;
    }
  }
}

cudaError_t launch_filter_prep(const float* F, float* hi, float* lo, int64_t ldf, const ConvGeom& g,
                               cudaStream_t st) {
  const int64_t total = ldf * g.k;
  const int64_t blocks = std::min<int64_t>((total + 255) / 256, 148 * 8);
  filter_prep_kernel<<<(unsigned)std::max<int64_t>(blocks, 1), 256, 0, st>>>(F, hi, lo, g.k_n, g.k, ldf);
  count_launch();
  return cudaGetLastError();
}

// w-im2col filters for the low-channel shifted-window mode: F'(n, kh, j) with
// j = c + c_i*kw (< k_w*c_i <= 32), zero for j >= k_w*c_i, as a (k_n, k_h, 32) array
// (the tap-major TMA map with k_h taps of 32 channels). 3xTF32: hi/lo split.
__global__ void __launch_bounds__(256) wim_filter_prep_kernel(const float* __restrict__ F, float* __restrict__ hi,
                                                              float* __restrict__ lo, int64_t k_n, int64_t k_h,
                                                              int64_t k_w, int64_t c_i) {
  const int64_t total = k_n * k_h * 32;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t n = idx % k_n, kh = (idx / k_n) % k_h, j = idx / (k_n * k_h);
    const int64_t kw = j / c_i, c = j - kw * c_i;
    const float f = kw < k_w ? __ldg(F + n + k_n * (kh + k_h * (kw + k_w * c))) : 0.0f;
    if (lo) {
      const float h = to_tf32(f);
      hi[idx] = h;
      lo[idx] = to_tf32(f - h);
    } else {
      hi[idx] = f;
    }
  }
}

cudaError_t launch_wim_filter_prep(const float* F, float* hi, float* lo, const ConvGeom& g, cudaStream_t st) {
  const int64_t total = g.k_n * g.k_h * 32;
  const int64_t blocks = std::min<int64_t>((total + 255) / 256, 148 * 8);
  wim_filter_prep_kernel<<<(unsigned)std::max<int64_t>(blocks, 1), 256, 0, st>>>(F, hi, lo, g.k_n, g.k_h, g.k_w,
                                                                                 g.c_i);
  count_launch();
  return cudaGetLastError();
}

}  // namespace cgb
