// ref_order.cu -- the reference's own arithmetic, bit for bit, on CUDA cores.
//
// Three entry points whose results are bit-identical to the reference's CPU templates
// for T = float and T = double, because each output is accumulated in exactly the
// reference's order with the product rounded before the add (the reference is built with
// -ffp-contract=off; __fmul_rn/__fadd_rn, __dmul_rn/__dadd_rn keep nvcc from fusing):
//
//   conv_direct   conv.hpp:24-55     O starts at +0; O += F*x over channel, filter
//                                    column, filter row; padding taps skipped.
//   gemm order    gemm.hpp:46-97,    per kc block [p_c, p_c + kc): acc = 0, acc += a*b
//                 microkernel.hpp    for p ascending (padding zeros included, as the
//                 :20-38             packed panels hold them); then C = C + acc. With C
//                                    zero-filled first (conv.hpp:71,89) this is
//                                    conv_gemm / conv_im2col_gemm / gemm.
//   im2col<T>     im2col.hpp:77-120  pure data movement.
//
// These are the checkers and the float64 path (the reference's f64 instantiations,
// bindings.cpp:58-65, README.md:38-40), not the performance path: one thread per output,
// a warp on 32 consecutive filters of one output pixel (coalesced F and O, broadcast x).
#include <algorithm>

#include "internal.h"

namespace cgb {

template <typename T>
CGB_DEV T mul_rn(T a, T b);
template <>
CGB_DEV float mul_rn<float>(float a, float b) { return __fmul_rn(a, b); }
template <>
CGB_DEV double mul_rn<double>(double a, double b) { return __dmul_rn(a, b); }
template <typename T>
CGB_DEV T add_rn(T a, T b);
template <>
CGB_DEV float add_rn<float>(float a, float b) { return __fadd_rn(a, b); }
template <>
CGB_DEV double add_rn<double>(double a, double b) { return __dadd_rn(a, b); }

template <typename T>
__global__ void __launch_bounds__(256) direct_kernel(const T* __restrict__ F, const T* __restrict__ I,
                                                     T* __restrict__ O, ConvGeom g) {
  const int64_t total = g.h_o * g.w_o * g.b * g.k_n;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = idx % g.k_n, pix = idx / g.k_n;
    const int64_t i_h = pix % g.h_o, t = pix / g.h_o;
    const int64_t i_w = t % g.w_o, i_b = t / g.w_o;
    T acc = T(0);
    for (int64_t i_c = 0; i_c < g.c_i; ++i_c) {
      const T* plane = I + (i_c + i_b * g.c_i) * g.h_i * g.w_i;
      for (int64_t i_kw = 0; i_kw < g.k_w; ++i_kw) {
        const int64_t w_in = i_w * g.s + i_kw - g.p;
        if (w_in < 0 || w_in >= g.w_i) continue;
        for (int64_t i_kh = 0; i_kh < g.k_h; ++i_kh) {
          const int64_t h_in = i_h * g.s + i_kh - g.p;
          if (h_in < 0 || h_in >= g.h_i) continue;
          const T x = plane[w_in * g.h_i + h_in];
          const T f = F[k + g.k_n * (i_kh + g.k_h * (i_kw + g.k_w * i_c))];
          acc = add_rn(acc, mul_rn(f, x));
        }
      }
    }
    O[idx] = acc;
  }
}

// C (m x n, ldc) = sum over kc blocks of (A * B restricted to the block), A (m x K,
// lda), B either the caller's matrix (K x n, ldb) or, when B == nullptr, the lowered
// matrix of the convolution g read straight from I (element r, c of im2col.hpp:71-76).
template <typename T>
__global__ void __launch_bounds__(256) refgemm_kernel(const T* __restrict__ A, int64_t lda, const T* __restrict__ B,
                                                      int64_t ldb, const T* __restrict__ I, ConvGeom g,
                                                      T* __restrict__ C, int64_t ldc, int64_t m, int64_t n,
                                                      int64_t K, int64_t kc, bool accumulate) {
  const int64_t total = m * n;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = idx % m, col = idx / m;
    // implicit source: decompose the column once (decompose_col, im2col.hpp:24-29)
    int64_t h0 = 0, w0 = 0;
    const T* img = nullptr;
    if (!B) {
      const int64_t i_h = col % g.h_o, t = col / g.h_o;
      const int64_t i_w = t % g.w_o, i_b = t / g.w_o;
      h0 = i_h * g.s - g.p;
      w0 = i_w * g.s - g.p;
      img = I + i_b * g.c_i * g.h_i * g.w_i;
    }
    T c = accumulate ? C[row + col * ldc] : T(0);  // gemm is C += A*B (callers zero C first)
    for (int64_t p0 = 0; p0 < K; p0 += kc) {
      const int64_t p1 = min(K, p0 + kc);
      T acc = T(0);
      // row p -> (i_kh, i_kw, i_c) by carry counters (decompose_row, im2col.hpp:17-22)
      int64_t kh = 0, kw = 0, ch = 0;
      if (!B) {
        kh = p0 % g.k_h;
        const int64_t q = p0 / g.k_h;
        kw = q % g.k_w;
        ch = q / g.k_w;
      }
      for (int64_t p = p0; p < p1; ++p) {
        T b;
        if (B) {
          b = B[p + col * ldb];
        } else {
          const int64_t hh = h0 + kh, ww = w0 + kw;
          b = (hh >= 0 && hh < g.h_i && ww >= 0 && ww < g.w_i) ? img[(ch * g.w_i + ww) * g.h_i + hh] : T(0);
          if (++kh == g.k_h) {
            kh = 0;
            if (++kw == g.k_w) {
              kw = 0;
              ++ch;
            }
          }
        }
        acc = add_rn(acc, mul_rn(A[row + p * lda], b));
      }
      c = add_rn(c, acc);
    }
    C[row + col * ldc] = c;
  }
}

template <typename T>
__global__ void __launch_bounds__(256) im2col_kernel_t(const T* __restrict__ I, T* __restrict__ B, int64_t ldb,
                                                       ConvGeom g) {
  const int64_t total = ldb * g.n;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = idx % ldb, col = idx / ldb;
    T v = T(0);
    if (r < g.k) {
      const int64_t kh = r % g.k_h, q = r / g.k_h, kw = q % g.k_w, ch = q / g.k_w;
      const int64_t i_h = col % g.h_o, t = col / g.h_o;
      const int64_t i_w = t % g.w_o, i_b = t / g.w_o;
      const int64_t hh = i_h * g.s + kh - g.p, ww = i_w * g.s + kw - g.p;
      if (hh >= 0 && hh < g.h_i && ww >= 0 && ww < g.w_i)
        v = I[((i_b * g.c_i + ch) * g.w_i + ww) * g.h_i + hh];
    }
    B[idx] = v;
  }
}

static unsigned grid_for(int64_t total) {
  return (unsigned)std::max<int64_t>(1, std::min<int64_t>((total + 255) / 256, 148 * 16));
}

template <typename T>
cudaError_t launch_direct_t(const T* F, const T* I, T* O, const ConvGeom& g, cudaStream_t st) {
  direct_kernel<T><<<grid_for(g.h_o * g.w_o * g.b * g.k_n), 256, 0, st>>>(F, I, O, g);
  count_launch();
  return cudaGetLastError();
}

template <typename T>
cudaError_t launch_refgemm_t(const T* A, int64_t lda, const T* B, int64_t ldb, const T* I, const ConvGeom& g, T* C,
                             int64_t ldc, int64_t m, int64_t n, int64_t K, int64_t kc, bool accumulate,
                             cudaStream_t st) {
  refgemm_kernel<T><<<grid_for(m * n), 256, 0, st>>>(A, lda, B, ldb, I, g, C, ldc, m, n, K, kc, accumulate);
  count_launch();
  return cudaGetLastError();
}

template <typename T>
cudaError_t launch_im2col_t(const T* I, T* B, int64_t ldb, const ConvGeom& g, cudaStream_t st) {
  im2col_kernel_t<T><<<grid_for(ldb * g.n), 256, 0, st>>>(I, B, ldb, g);
  count_launch();
  return cudaGetLastError();
}

cudaError_t launch_direct_conv(const float* F, const float* I, float* O, const ConvGeom& g, cudaStream_t st) {
  return launch_direct_t<float>(F, I, O, g, st);
}
cudaError_t launch_direct_conv_f64(const double* F, const double* I, double* O, const ConvGeom& g, cudaStream_t st) {
  return launch_direct_t<double>(F, I, O, g, st);
}
cudaError_t launch_refgemm_f64(const double* A, int64_t lda, const double* B, int64_t ldb, const double* I,
                               const ConvGeom& g, double* C, int64_t ldc, int64_t m, int64_t n, int64_t K, int64_t kc,
                               bool accumulate, cudaStream_t st) {
  return launch_refgemm_t<double>(A, lda, B, ldb, I, g, C, ldc, m, n, K, kc, accumulate, st);
}
cudaError_t launch_im2col_f64(const double* I, double* B, int64_t ldb, const ConvGeom& g, cudaStream_t st) {
  return launch_im2col_t<double>(I, B, ldb, g, st);
}

}  // namespace cgb
