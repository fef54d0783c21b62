// tc_conv.cu -- K3: tcgen05 (kind::tf32) implicit-GEMM convolution for sm_100a in the
// reference's row order (any geometry; the fallback of the fused path).
//
// Replaces the reference's five-loop BLIS GEMM driven by pack_b_im2col
// (gemm.hpp:46-97, im2col.hpp:177-262) and its 8x12 micro-kernel
// (microkernel.hpp:20-38). The explicit path's GEMM over B-hat is k2_gemm.cu.
//
// GEMM orientation: M = output pixels (column c of the lowered matrix,
// c = i_h + i_w*h_o + i_b*h_o*w_o), N = filters (k_n), K = k_h*k_w*c_i in the
// reference's row order r = i_kh + i_kw*k_h + i_c*k_h*k_w. D[pixel][filter] lands in
// TMEM as 128 lanes x BN fp32 columns, so each epilogue thread owns one pixel and
// writes BN contiguous filters of O (k_n fastest, tensor.hpp:108-113).
//
// Operands:
//   A (pixels x K, K-major, 128B swizzle): gathered by 8 producer warps
//     (register-staged: LDG -> [TF32 rounding | 3xTF32 hi/lo split] -> STS into the
//     canonical swizzled layout). The lowered matrix never reaches HBM.
//   B (K x filters, MN-major, 128B swizzle of 32-byte atoms): TMA boxes of 32 filters x 32 rows
//     straight from F (k_n fastest is already MN-major), or from the hi/lo split.
// Roles (320 threads): warps 0-7 A producers (warps 0-3 then run the epilogue on
// TMEM lanes 0-127), warp 8 TMA producer + TMEM allocator, warp 9 MMA issuer.
// Pipeline: STAGES slots, full[] (8 producer-warp arrivals + TMA tx bytes) and
// empty[] (tcgen05.commit) mbarriers; tmem_full signals the epilogue.
#include <algorithm>
#include <cstdio>

#include "internal.h"

namespace cgb {
namespace tc {

constexpr int BM = 128;
constexpr int BK = 32;  // one 128-byte swizzle row of fp32
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
  static constexpr int BUDGET = SPLIT ? 200 * 1024 : 100 * 1024;
  static constexpr int STAGES_RAW = BUDGET / STAGE;
  static constexpr int STAGES = STAGES_RAW > 6 ? 6 : (STAGES_RAW < 2 ? 2 : STAGES_RAW);
  static constexpr int TMEM_COLS = BN < 32 ? 32 : BN;
  static constexpr int SMEM = STAGES * STAGE + 1024 /*align*/ + 256 /*barriers*/;
};

struct Args {
  int32_t k_n, k_h, k_w, c_i, h_i, w_i, s, p, h_o, w_o, K;
  int32_t KT;  // number of BK steps
  int64_t n, plane;
  // mixed-radix decomposition of BK in (c, kw, kh) digits
  int32_t d_c, d_kw, d_kh;
};

// Per producer thread: 2 pixel rows x 2 swizzle chunks x 4 consecutive K.
struct RowState {
  const float* base;  // I + image offset + w0*h_i + h0 (may point outside; only read when valid)
  int32_t h0, w0;
  bool ok;
};
struct ChunkState {
  int32_t c, kw, kh, r;  // decomposition of the chunk's first row at the current stage
};

CGB_DEV void gather_chunk(const Args& a, const RowState& rs, const ChunkState& cs, float (&v)[4]) {
  int32_t c = cs.c, kw = cs.kw, kh = cs.kh;
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const int32_t hh = rs.h0 + kh, ww = rs.w0 + kw;
    float x = 0.0f;
    if (rs.ok && cs.r + e < a.K && (unsigned)hh < (unsigned)a.h_i && (unsigned)ww < (unsigned)a.w_i)
      x = __ldg(rs.base + c * a.plane + kw * a.h_i + kh);
    v[e] = x;
    if (++kh == a.k_h) {
      kh = 0;
      if (++kw == a.k_w) { kw = 0; ++c; }
    }
  }
}

CGB_DEV void advance_chunk(const Args& a, ChunkState& cs) {
  cs.r += BK;
  int32_t kh = cs.kh + a.d_kh;
  int32_t carry = kh >= a.k_h;
  kh -= carry ? a.k_h : 0;
  int32_t kw = cs.kw + a.d_kw + carry;
  carry = kw >= a.k_w;
  kw -= carry ? a.k_w : 0;
  cs.c += a.d_c + carry;
  cs.kw = kw;
  cs.kh = kh;
}

template <int BN, bool SPLIT>
__global__ void __launch_bounds__(THREADS, 1)
    tc_conv_kernel(const __grid_constant__ CUtensorMap tmap_hi, const __grid_constant__ CUtensorMap tmap_lo,
                   const float* __restrict__ I, float* __restrict__ O, Args a) {
  using C = Cfg<BN, SPLIT>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  // stage s: [A_hi][A_lo?][B_hi][B_lo?]
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
    // ------------------------------------------------------------ A producers
    RowState rs[2];
    int rows[2];
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      rows[q] = (lane % 8) + 8 * (warp + 8 * q);
      const int64_t P = m0 + rows[q];
      rs[q].ok = P < a.n;
      rs[q].h0 = 0; rs[q].w0 = 0; rs[q].base = I;
      if (rs[q].ok) {
        const int32_t hw = a.h_o * a.w_o;
        const int32_t i_b = (int32_t)(P / hw);
        const int32_t rem = (int32_t)(P - (int64_t)i_b * hw);
        const int32_t i_w = rem / a.h_o, i_h = rem - i_w * a.h_o;
        rs[q].h0 = i_h * a.s - a.p;
        rs[q].w0 = i_w * a.s - a.p;
        rs[q].base = I + (int64_t)i_b * a.c_i * a.plane + (int64_t)rs[q].w0 * a.h_i + rs[q].h0;
      }
    }
    ChunkState cs[2];
    int chunks[2];
#pragma unroll
    for (int v = 0; v < 2; ++v) {
      chunks[v] = (lane / 8) + 4 * v;
      const int32_t r = 4 * chunks[v];
      cs[v].r = r;
      cs[v].kh = r % a.k_h;
      const int32_t t = r / a.k_h;
      cs[v].kw = t % a.k_w;
      cs[v].c = t / a.k_w;
    }
    float vals[2][2][4];
    auto load_stage = [&]() {
#pragma unroll
      for (int q = 0; q < 2; ++q)
#pragma unroll
        for (int v = 0; v < 2; ++v) gather_chunk(a, rs[q], cs[v], vals[q][v]);
    };
    load_stage();
    for (int kt = 0; kt < a.KT; ++kt) {
      const int s = kt % C::STAGES;
      const uint32_t ph = (kt / C::STAGES) & 1;
      mbar_wait(&empty[s], ph ^ 1);
#pragma unroll
      for (int q = 0; q < 2; ++q)
#pragma unroll
        for (int v = 0; v < 2; ++v) {
          const uint32_t off = rows[q] * 128 + ((chunks[v] ^ (rows[q] & 7)) << 4);
          float4 hi, lo;
          float* h = &hi.x;
          float* l = &lo.x;
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float x = vals[q][v][e];
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
      if (kt + 1 < a.KT) {
#pragma unroll
        for (int v = 0; v < 2; ++v) advance_chunk(a, cs[v]);
        load_stage();
      }
    }
  } else if (warp == TMA_WARP) {
    // ------------------------------------------------------------ B (filter) TMA producer
    if (elect_one()) {
      constexpr uint32_t bytes = C::NS * C::B_TILE;
      for (int kt = 0; kt < a.KT; ++kt) {
        const int s = kt % C::STAGES;
        const uint32_t ph = (kt / C::STAGES) & 1;
        mbar_wait(&empty[s], ph ^ 1);
        mbar_arrive_expect_tx(&full[s], bytes);
#pragma unroll
        for (int j = 0; j < BN / 32; ++j) {
          tma_load_2d(smem_u32(b_tile(s, 0)) + j * 4096, &tmap_hi, &full[s], n0 + 32 * j, kt * BK);
          if (SPLIT) tma_load_2d(smem_u32(b_tile(s, 1)) + j * 4096, &tmap_lo, &full[s], n0 + 32 * j, kt * BK);
        }
      }
    }
  } else if (warp == MMA_WARP) {
    // ------------------------------------------------------------ MMA issuer
    constexpr uint32_t idesc = idesc_tf32(BN < 32 ? 32 : BN, /*a_mn=*/false, /*b_mn=*/true);
    if (elect_one()) {
      for (int kt = 0; kt < a.KT; ++kt) {
        const int s = kt % C::STAGES;
        const uint32_t ph = (kt / C::STAGES) & 1;
        mbar_wait(&full[s], ph);
        tc_fence_after();
        const uint32_t a_hi = smem_u32(a_tile(s, 0)), b_hi = smem_u32(b_tile(s, 0));
#pragma unroll
        for (int kk = 0; kk < BK / 8; ++kk) {
          // A: K-major SW128, k-step = +32 B inside the swizzle row; 8-row groups 1024 B apart.
          // B: MN-major SW128 with 32-byte atoms (the only MN-major layout kind::tf32 takes):
          //    k-step = +1024 B (8 rows of 128 B), 4-row groups 512 B apart, 32-filter blocks 4096 B apart.
          const uint64_t ad = smem_desc(a_hi + kk * 32, 16, 1024);
          const uint64_t bd = smem_desc(b_hi + kk * 1024, 4096, 512, 0, kLayoutSW128_32B);
          const uint32_t acc = (kt | kk) != 0;
          if (SPLIT) {
            const uint64_t ad_lo = smem_desc(smem_u32(a_tile(s, 1)) + kk * 32, 16, 1024);
            const uint64_t bd_lo = smem_desc(smem_u32(b_tile(s, 1)) + kk * 1024, 4096, 512, 0, kLayoutSW128_32B);
            mma_tf32(tmem_base, ad_lo, bd, idesc, acc);
            mma_tf32(tmem_base, ad, bd_lo, idesc, 1);
            mma_tf32(tmem_base, ad, bd, idesc, 1);
          } else {
            mma_tf32(tmem_base, ad, bd, idesc, acc);
          }
        }
        mma_commit(&empty[s]);
      }
      mma_commit(tmem_full);
    }
  }

  // ------------------------------------------------------------ epilogue (warps 0-3)
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
                       int64_t n, int64_t k_n, cudaStream_t st) {
  using C = Cfg<BN, SPLIT>;
  auto kern = tc_conv_kernel<BN, SPLIT>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
  if (e != cudaSuccess) return e;
  dim3 grid((unsigned)((n + BM - 1) / BM), (unsigned)((k_n + BN - 1) / BN));
  kern<<<grid, THREADS, C::SMEM, st>>>(th, tl, I, O, a);
  count_launch();
  return cudaGetLastError();
}

}  // namespace tc

cudaError_t launch_tc_conv(const float* f_hi, const float* f_lo, int64_t ldf, const float* I, float* O,
                           const ConvGeom& g, bool split, cudaStream_t st) {
  tc::Args a;
  a.k_n = (int32_t)g.k_n; a.k_h = (int32_t)g.k_h; a.k_w = (int32_t)g.k_w; a.c_i = (int32_t)g.c_i;
  a.h_i = (int32_t)g.h_i; a.w_i = (int32_t)g.w_i; a.s = (int32_t)g.s; a.p = (int32_t)g.p;
  a.h_o = (int32_t)g.h_o; a.w_o = (int32_t)g.w_o; a.K = (int32_t)g.k;
  a.KT = (int32_t)((g.k + tc::BK - 1) / tc::BK);
  a.n = g.n; a.plane = g.h_i * g.w_i;
  {
    const int32_t khw = a.k_h * a.k_w;
    a.d_c = tc::BK / khw;
    const int32_t rem = tc::BK % khw;
    a.d_kw = rem / a.k_h;
    a.d_kh = rem % a.k_h;
  }
  CUtensorMap th, tl;
  cudaError_t e = make_filter_tmap(&th, f_hi, g.k_n, g.k, ldf);
  if (e != cudaSuccess) return e;
  if (split) {
    e = make_filter_tmap(&tl, f_lo, g.k_n, g.k, ldf);
    if (e != cudaSuccess) return e;
  } else {
    tl = th;
  }
  const int64_t kn = g.k_n;
#define CGB_TC_DISPATCH(BN)                                                      \
  return split ? tc::launch_cfg<BN, true>(th, tl, I, O, a, g.n, kn, st)          \
               : tc::launch_cfg<BN, false>(th, tl, I, O, a, g.n, kn, st);
  if (kn <= 32) { CGB_TC_DISPATCH(32) }
  if (kn <= 64) { CGB_TC_DISPATCH(64) }
  if (kn <= 128) { CGB_TC_DISPATCH(128) }
  CGB_TC_DISPATCH(256)
#undef CGB_TC_DISPATCH
}

}  // namespace cgb
