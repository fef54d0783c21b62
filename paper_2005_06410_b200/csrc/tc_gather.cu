// tc_gather.cu -- K3 (fused) tcgen05 implicit GEMM with a tap-major K order.
//
// The reference packs the lowered matrix B-hat in row order r = i_kh + i_kw*k_h +
// i_c*k_h*k_w (im2col.hpp:71-76, pack_b_im2col im2col.hpp:177-262). A dot product is
// order-independent up to rounding, so this kernel walks K as (channel chunk cc, tap)
// instead: one K step = 32 consecutive channels of one filter tap. Then
//   * the A producer does one padding test and one address setup per (pixel, tap)
//     and gathers 32 channels at the plane stride -- warps read 32 consecutive output
//     pixels per channel, i.e. coalesced 128-byte lines for stride 1;
//   * the 9 taps of one channel chunk are consecutive K steps, so the input window is
//     re-read from L1 rather than L2;
//   * the filter block for (tap, cc) is a 3-D TMA box (32 filters x 1 tap x 32
//     channels) read straight from F (k_n fastest is the MN-major UMMA B layout).
//
// Tile: 128 pixels x BN filters (BN up to 512 = two UMMA N=256 halves sharing A),
// K step 32. Roles (320 threads): warps 0-7 A producers (register-staged, two steps
// of lookahead; TF32 rounding or 3xTF32 hi/lo split in registers), warp 8 TMA + TMEM
// allocation, warp 9 MMA issue; warps 0-3 then drain TMEM to O.
#include <algorithm>

#include "internal.h"

namespace cgb {
namespace tg {

constexpr int BM = 128;
constexpr int BK = 32;
constexpr int PRODUCER_WARPS = 8;
constexpr int TMA_WARP = 8;
constexpr int MMA_WARP = 9;
constexpr int THREADS = 320;
constexpr int A_TILE = BM * BK * 4;  // 16 KB

template <int BN, bool SPLIT>
struct Cfg {
  static constexpr int NS = SPLIT ? 2 : 1;
  static constexpr int B_TILE = BN * BK * 4;
  static constexpr int STAGE = NS * (A_TILE + B_TILE);
  static constexpr int BUDGET = 200 * 1024;
  static constexpr int STAGES_RAW = BUDGET / STAGE;
  static constexpr int STAGES = STAGES_RAW > 8 ? 8 : (STAGES_RAW < 2 ? 2 : STAGES_RAW);
  static constexpr int TMEM_COLS = BN;  // 64..512, power of two
  static constexpr int SMEM = STAGES * STAGE + 1024 + 256;
  static constexpr int UMMA_N = BN > 256 ? 256 : BN;
  static constexpr int NHALF = BN / UMMA_N;
};

struct Args {
  int32_t k_n, k_h, k_w, c_i, h_i, w_i, s, p, h_o, w_o;
  int32_t CC;   // channel chunks of 32
  int32_t KS;   // K steps = k_h*k_w*CC
  int64_t n, plane;
};

struct Row {
  const float* img;  // image base
  int32_t h0, w0;
  bool ok;
};

// 4 channels (c..c+3) of pixel row at tap (kh, kw)
CGB_DEV void gather4(const Args& a, const Row& rw, int32_t kh, int32_t kw, int32_t c, float (&v)[4]) {
  const int32_t hh = rw.h0 + kh, ww = rw.w0 + kw;
  const bool ok = rw.ok && (unsigned)hh < (unsigned)a.h_i && (unsigned)ww < (unsigned)a.w_i;
  const float* src = rw.img + (int64_t)c * a.plane + ww * a.h_i + hh;
#pragma unroll
  for (int e = 0; e < 4; ++e) v[e] = (ok && c + e < a.c_i) ? __ldg(src + e * a.plane) : 0.0f;
}

template <int BN, bool SPLIT>
__global__ void __launch_bounds__(THREADS, 1)
    tc_gather_kernel(const __grid_constant__ CUtensorMap tmap_hi, const __grid_constant__ CUtensorMap tmap_lo,
                     const float* __restrict__ I, float* __restrict__ O, Args a) {
  using C = Cfg<BN, SPLIT>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  auto a_tile = [&](int s, int part) { return smem + s * C::STAGE + part * A_TILE; };
  auto b_tile = [&](int s, int part) { return smem + s * C::STAGE + C::NS * A_TILE + part * C::B_TILE; };
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::STAGES * C::STAGE);
  uint64_t* empty = full + C::STAGES;
  uint64_t* tmem_full = empty + C::STAGES;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(tmem_full + 1);

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const int64_t m0 = (int64_t)blockIdx.x * BM;
  const int n0 = blockIdx.y * BN;

  if (warp == TMA_WARP) {
    if (lane == 0) {
      for (int s = 0; s < C::STAGES; ++s) {
        mbar_init(&full[s], PRODUCER_WARPS + 1);
        mbar_init(&empty[s], 1);
      }
      mbar_init(tmem_full, 1);
      fence_mbar_init();
      tma_prefetch_desc(&tmap_hi);
      if (SPLIT) tma_prefetch_desc(&tmap_lo);
    }
    __syncwarp();
    tmem_alloc(tmem_holder, C::TMEM_COLS);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;

  if (warp < PRODUCER_WARPS) {
    // -------------------------------------------------------------- A producers
    Row rw[2];
    int rows[2];
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      rows[q] = (lane % 8) + 8 * (warp + 8 * q);
      const int64_t P = m0 + rows[q];
      rw[q].ok = P < a.n;
      rw[q].h0 = 0; rw[q].w0 = 0; rw[q].img = I;
      if (rw[q].ok) {
        const int32_t hw = a.h_o * a.w_o;
        const int32_t i_b = (int32_t)(P / hw);
        const int32_t rem = (int32_t)(P - (int64_t)i_b * hw);
        const int32_t i_w = rem / a.h_o, i_h = rem - i_w * a.h_o;
        rw[q].h0 = i_h * a.s - a.p;
        rw[q].w0 = i_w * a.s - a.p;
        rw[q].img = I + (int64_t)i_b * a.c_i * a.plane;
      }
    }
    const int chunk0 = lane / 8;  // swizzle chunks chunk0 and chunk0 + 4 -> channels 4*chunk
    // K-step walk: ks = cc * taps + tap (taps inner, for L1 reuse of the input window)
    const int32_t taps = a.k_h * a.k_w;
    float buf[2][2][2][4];  // [lookahead slot][row][chunk][e]
    auto load = [&](int ks, float (&v)[2][2][4]) {
      const int32_t cc = ks / taps, tap = ks - cc * taps;
      const int32_t kw = tap / a.k_h, kh = tap - kw * a.k_h;
#pragma unroll
      for (int q = 0; q < 2; ++q)
#pragma unroll
        for (int u = 0; u < 2; ++u) gather4(a, rw[q], kh, kw, cc * BK + 4 * (chunk0 + 4 * u), v[q][u]);
    };
    auto store = [&](int ks, const float (&v)[2][2][4]) {
      const int s = ks % C::STAGES;
      const uint32_t ph = (ks / C::STAGES) & 1;
      mbar_wait(&empty[s], ph ^ 1);
#pragma unroll
      for (int q = 0; q < 2; ++q)
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int ch = chunk0 + 4 * u;
          const uint32_t off = rows[q] * 128 + ((ch ^ (rows[q] & 7)) << 4);
          float4 hi, lo;
          float* h = &hi.x;
          float* l = &lo.x;
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float x = v[q][u][e];
            const float t = to_tf32(x);
            h[e] = t;
            if (SPLIT) l[e] = to_tf32(x - t);
          }
          *reinterpret_cast<float4*>(a_tile(s, 0) + off) = hi;
          if (SPLIT) *reinterpret_cast<float4*>(a_tile(s, 1) + off) = lo;
        }
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(&full[s]);
    };
    // two register slots of lookahead, statically indexed (manual unroll by 2)
    load(0, buf[0]);
    if (a.KS > 1) load(1, buf[1]);
    for (int ks = 0; ks < a.KS; ks += 2) {
      store(ks, buf[0]);
      if (ks + 2 < a.KS) load(ks + 2, buf[0]);
      if (ks + 1 < a.KS) {
        store(ks + 1, buf[1]);
        if (ks + 3 < a.KS) load(ks + 3, buf[1]);
      }
    }
  } else if (warp == TMA_WARP) {
    // -------------------------------------------------------------- filter TMA
    if (elect_one()) {
      constexpr uint32_t bytes = C::NS * C::B_TILE;
      const int32_t taps = a.k_h * a.k_w;
      for (int ks = 0; ks < a.KS; ++ks) {
        const int s = ks % C::STAGES;
        const uint32_t ph = (ks / C::STAGES) & 1;
        const int32_t cc = ks / taps, tap = ks - cc * taps;
        mbar_wait(&empty[s], ph ^ 1);
        mbar_arrive_expect_tx(&full[s], bytes);
#pragma unroll
        for (int j = 0; j < BN / 32; ++j) {
          tma_load_3d(smem_u32(b_tile(s, 0)) + j * 4096, &tmap_hi, &full[s], n0 + 32 * j, tap, cc * BK);
          if (SPLIT) tma_load_3d(smem_u32(b_tile(s, 1)) + j * 4096, &tmap_lo, &full[s], n0 + 32 * j, tap, cc * BK);
        }
      }
    }
  } else if (warp == MMA_WARP) {
    // -------------------------------------------------------------- MMA issue
    constexpr uint32_t idesc = idesc_tf32(C::UMMA_N, false, true);
    if (elect_one()) {
      for (int ks = 0; ks < a.KS; ++ks) {
        const int s = ks % C::STAGES;
        const uint32_t ph = (ks / C::STAGES) & 1;
        mbar_wait(&full[s], ph);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < BK / 8; ++kk) {
          const uint64_t ad = smem_desc(smem_u32(a_tile(s, 0)) + kk * 32, 16, 1024);
          const uint64_t ad_lo = SPLIT ? smem_desc(smem_u32(a_tile(s, 1)) + kk * 32, 16, 1024) : 0;
          const uint32_t acc = (ks | kk) != 0;
#pragma unroll
          for (int hf = 0; hf < C::NHALF; ++hf) {
            const uint32_t boff = hf * (C::UMMA_N / 32) * 4096 + kk * 1024;
            const uint64_t bd = smem_desc(smem_u32(b_tile(s, 0)) + boff, 4096, 512, 0, kLayoutSW128_32B);
            const uint32_t d = tmem_base + hf * C::UMMA_N;
            if (SPLIT) {
              const uint64_t bd_lo = smem_desc(smem_u32(b_tile(s, 1)) + boff, 4096, 512, 0, kLayoutSW128_32B);
              mma_tf32(d, ad_lo, bd, idesc, acc);
              mma_tf32(d, ad, bd_lo, idesc, 1);
              mma_tf32(d, ad, bd, idesc, 1);
            } else {
              mma_tf32(d, ad, bd, idesc, acc);
            }
          }
        }
        mma_commit(&empty[s]);
      }
      mma_commit(tmem_full);
    }
  }

  // -------------------------------------------------------------- epilogue (warps 0-3)
  if (warp < 4) {
    mbar_wait(tmem_full, 0);
    tc_fence_after();
    const int64_t P = m0 + warp * 32 + lane;
    const bool vec = (a.k_n % 4) == 0 && reinterpret_cast<uintptr_t>(O) % 16 == 0;
#pragma unroll 1
    for (int cb = 0; cb < BN / 32; ++cb) {
      uint32_t r[32];
      tmem_ld_32x32b_x32(tmem_base + ((uint32_t)(warp * 32) << 16) + cb * 32, r);
      tmem_ld_wait();
      const int nb = n0 + cb * 32;
      if (P < a.n && nb < a.k_n) {
        float* dst = O + P * a.k_n + nb;
        if (vec && nb + 32 <= a.k_n) {
#pragma unroll
          for (int j = 0; j < 32; j += 4)
            *reinterpret_cast<float4*>(dst + j) = make_float4(__uint_as_float(r[j]), __uint_as_float(r[j + 1]),
                                                              __uint_as_float(r[j + 2]), __uint_as_float(r[j + 3]));
        } else {
#pragma unroll
          for (int j = 0; j < 32; ++j)
            if (nb + j < a.k_n) dst[j] = __uint_as_float(r[j]);
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == TMA_WARP) {
    __syncwarp();
    tc_fence_after();
    tmem_dealloc(tmem_base, C::TMEM_COLS);
  }
}

template <int BN, bool SPLIT>
cudaError_t launch_cfg(const CUtensorMap& th, const CUtensorMap& tl, const float* I, float* O, const Args& a,
                       cudaStream_t st) {
  using C = Cfg<BN, SPLIT>;
  auto kern = tc_gather_kernel<BN, SPLIT>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
  if (e != cudaSuccess) return e;
  dim3 grid((unsigned)((a.n + BM - 1) / BM), (unsigned)((a.k_n + BN - 1) / BN));
  kern<<<grid, THREADS, C::SMEM, st>>>(th, tl, I, O, a);
  count_launch();
  return cudaGetLastError();
}

}  // namespace tg

bool gather_supported(const ConvGeom& g) { return g.c_i >= 16 && g.k_n % 4 == 0; }

cudaError_t launch_tc_gather(const float* f_hi, const float* f_lo, const float* I, float* O, const ConvGeom& g,
                             bool split, cudaStream_t st) {
  tg::Args a;
  a.k_n = (int32_t)g.k_n; a.k_h = (int32_t)g.k_h; a.k_w = (int32_t)g.k_w; a.c_i = (int32_t)g.c_i;
  a.h_i = (int32_t)g.h_i; a.w_i = (int32_t)g.w_i; a.s = (int32_t)g.s; a.p = (int32_t)g.p;
  a.h_o = (int32_t)g.h_o; a.w_o = (int32_t)g.w_o;
  a.CC = (int32_t)((g.c_i + tg::BK - 1) / tg::BK);
  a.KS = (int32_t)(g.k_h * g.k_w) * a.CC;
  a.n = g.n; a.plane = g.h_i * g.w_i;
  CUtensorMap th, tl;
  cudaError_t e = make_filter_tmap_tapmajor(&th, f_hi, g);
  if (e != cudaSuccess) return e;
  if (split) {
    if ((e = make_filter_tmap_tapmajor(&tl, f_lo, g)) != cudaSuccess) return e;
  } else {
    tl = th;
  }
  const int64_t kn = g.k_n;
#define CGB_TG(BN)                                                                                  \
  return split ? tg::launch_cfg<BN, true>(th, tl, I, O, a, st) : tg::launch_cfg<BN, false>(th, tl, I, O, a, st);
  if (kn <= 64) { CGB_TG(64) }
  if (kn <= 128) { CGB_TG(128) }
  if (kn <= 256 || split) { CGB_TG(256) }
#undef CGB_TG
  return tg::launch_cfg<512, false>(th, tl, I, O, a, st);  // 3xTF32 stages do not fit at BN = 512
}

}  // namespace cgb
