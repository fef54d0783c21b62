// k2_gemm.cu -- K2: the explicit path's GEMM over the lowered matrix, TMA-fed on both
// operands (tcgen05 kind::tf32, sm_100a).
//
// Replaces the reference's gemm() over a MatrixSource (gemm.hpp:46-105) and
// MatrixSource::pack_block (packing.hpp:89-113): where the reference packs kc x nc
// blocks of B-hat into Bc panels, the TMA unit here loads 128-column x 32-row tiles of
// B-hat straight into the 128B-swizzled K-major UMMA layout (B-hat is K-fastest with
// ld % 4 == 0, i.e. already K-major for the M operand). Filters (k_n fastest =
// MN-major) come in by TMA as in the fused kernels. No thread touches an operand
// element in TF32 mode.
//
// GEMM orientation as in tc_conv.cu: M = lowered columns (output pixels), N = filters,
// K = lowered rows; D[pixel][filter] in TMEM, so one epilogue thread owns one pixel and
// writes BN contiguous filters of O.
//
// Roles: warp 0 TMA producer (+TMEM alloc), warp 1 MMA issuer, warps 2-5 epilogue
// (TMEM lane quadrant = warp % 4), 3xTF32 only: warps 6-13 "lo" warps. Persistent
// grid, one ring of STAGES (A tile, filter tile) slots filled by TMA -- as deep as shared
// memory allows, since it has to cover the HBM latency -- plus, in 3xTF32, a short ring
// of LOS lo slots written by the lo warps (they are consumed within one stage time);
// two TMEM accumulator sets so the epilogue of one tile overlaps the main loop of the
// next.
//
// 3xTF32: the tensor core truncates raw fp32 operands to TF32 (pinned by
// tests/test_parity_gpu.py::test_tf32_truncates_raw_operands), so the TMA'd raw tile IS
// the hi operand; the lo warps write lo = rna_tf32(x - trunc_tf32(x)) element for
// element at the same (swizzled) offsets into a second tile -- for the A tile always,
// for the filter tile when no pre-split lo filters were passed (large static weights,
// e.g. fc layers: no per-call split pass over them, no workspace).
//
// Few-tile shapes (fc layers: n = batch <= 128 columns against 10^2 MB of weights):
// split-K over S pieces per tile so every SM streams its share of the weights; pieces
// write partial tiles to a workspace and k2_reduce_kernel sums them in piece order
// (bitwise deterministic; no CTA waits on another).
#include <algorithm>
#include <cstdio>

#include "internal.h"

namespace cgb {
namespace k2 {

constexpr int BM = 128;
constexpr int BK = 32;  // one 128-byte swizzle row of fp32
constexpr int A_TILE = BM * BK * 4;
constexpr int TMA_WARP = 0, MMA_WARP = 1, EPI_WARP0 = 2, LO_WARP0 = 6, LO_WARPS = 8;

// MODE 0: TF32. 1: 3xTF32, pre-split filter lo tiles arrive by TMA. 2: 3xTF32, the filter
// lo tile is split in the kernel (FLO).
template <int BN, int MODE>
struct Cfg {
  static constexpr bool SPLIT = MODE != 0;
  static constexpr bool FLO = MODE == 2;
  static constexpr int B_TILE = BN * BK * 4;
  static constexpr int STAGE = A_TILE + B_TILE * (MODE == 1 ? 2 : 1);  // TMA-filled: A raw, F raw[, F lo]
  static constexpr int LO_SLOT = !SPLIT ? 0 : A_TILE + (FLO ? B_TILE : 0);  // lo-warp-filled: A lo[, F lo]
  static constexpr int BUDGET = 216 * 1024;
  // lo slots: a slot is busy from the split to the end of its stage's MMAs, about two
  // stage times -- three slots where five TMA stages still fit beside them, else two
  // while two stages fit (a third TMA stage instead of the second lo slot measured
  // slower: fc6 3xTF32 216 vs 190 us), else one
  static constexpr int LOS = !SPLIT ? 0
                             : (BUDGET - 3 * LO_SLOT) / STAGE >= 5 ? 3
                             : (BUDGET - 2 * LO_SLOT) / STAGE >= 2 ? 2 : 1;
  static constexpr int STAGES_RAW = (BUDGET - LOS * LO_SLOT) / STAGE;
  static constexpr int STAGES = STAGES_RAW > 8 ? 8 : STAGES_RAW;
  static constexpr int TMEM_COLS = 2 * BN < 32 ? 32 : 2 * BN;
  static constexpr int THREADS = 32 * (SPLIT ? LO_WARP0 + LO_WARPS : LO_WARP0);
  static constexpr int SMEM = STAGES * STAGE + LOS * LO_SLOT + 1024 /*align*/ + 256 /*barriers*/;
  static_assert(STAGES >= 2, "ring too shallow");
};

struct Args {
  float* O;
  float* ws;        // split-K partial tiles: [tile][piece][128][BN]
  int64_t n;        // lowered columns (output pixels)
  int64_t items;    // tiles * S
  int32_t k_n, KT;  // filters, 32-row chunks of K
  int32_t m_tiles, n_tiles, S;
  int32_t nt_fast;  // work order: filter tile fastest (B-hat tile shared through L2) or pixel tile fastest
  int32_t vec;      // O rows can take 32-byte (2) / 16-byte (1) vector stores
};

struct Item {
  int32_t mt, nt, piece, kt0, kt1;
};

CGB_DEV Item decode(const Args& a, int64_t w) {
  Item x;
  if (a.nt_fast) {
    x.nt = (int32_t)(w % a.n_tiles);
    const int64_t r = w / a.n_tiles;
    x.piece = (int32_t)(r % a.S);
    x.mt = (int32_t)(r / a.S);
  } else {
    x.mt = (int32_t)(w % a.m_tiles);
    const int64_t r = w / a.m_tiles;
    x.piece = (int32_t)(r % a.S);
    x.nt = (int32_t)(r / a.S);
  }
  x.kt0 = (int32_t)((int64_t)x.piece * a.KT / a.S);
  x.kt1 = (int32_t)((int64_t)(x.piece + 1) * a.KT / a.S);
  return x;
}

// One accumulator row segment (32 fp32 columns) to global memory; ncols = valid columns.
CGB_DEV void store_row32(float* dst, const uint32_t (&r)[32], int ncols, int vec) {
  if (ncols >= 32 && vec == 2) {
#pragma unroll
    for (int j = 0; j < 32; j += 8) st_global_v8(dst + j, &r[j]);
  } else if (ncols >= 32 && vec == 1) {
#pragma unroll
    for (int j = 0; j < 32; j += 4)
      *reinterpret_cast<float4*>(dst + j) = make_float4(__uint_as_float(r[j]), __uint_as_float(r[j + 1]),
                                                        __uint_as_float(r[j + 2]), __uint_as_float(r[j + 3]));
  } else {
#pragma unroll
    for (int j = 0; j < 32; ++j)
      if (j < ncols) dst[j] = __uint_as_float(r[j]);
  }
}

template <int BN, int MODE>
__global__ void __launch_bounds__(Cfg<BN, MODE>::THREADS, 1)
    k2_gemm_kernel(const __grid_constant__ CUtensorMap tmap_a, const __grid_constant__ CUtensorMap tmap_hi,
                   const __grid_constant__ CUtensorMap tmap_lo, Args a) {
  using C = Cfg<BN, MODE>;
  constexpr bool SPLIT = C::SPLIT, FLO = C::FLO;
  constexpr int LOS = C::LOS > 0 ? C::LOS : 1;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  // stage s: [A raw][F raw][F lo (MODE 1)]; lo slot l: [A lo][F lo (MODE 2)]
  auto a_tile = [&](int s) { return smem + s * C::STAGE; };
  auto b_tile = [&](int s) { return smem + s * C::STAGE + A_TILE; };
  auto b_lo_tma = [&](int s) { return smem + s * C::STAGE + A_TILE + C::B_TILE; };
  auto a_lo = [&](int l) { return smem + C::STAGES * C::STAGE + l * C::LO_SLOT; };
  auto b_lo_flo = [&](int l) { return smem + C::STAGES * C::STAGE + l * C::LO_SLOT + A_TILE; };
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::STAGES * C::STAGE + C::LOS * C::LO_SLOT);
  uint64_t* empty = full + C::STAGES;
  uint64_t* lo_full = empty + C::STAGES;      // [LOS]
  uint64_t* lo_empty = lo_full + 3;           // [LOS]
  uint64_t* tmem_full = lo_empty + 3;         // [2]
  uint64_t* tmem_empty = tmem_full + 2;       // [2]
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(tmem_empty + 2);

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;

  if (warp == TMA_WARP) {
    if (lane == 0) {
      for (int s = 0; s < C::STAGES; ++s) {
        mbar_init(&full[s], 1);
        mbar_init(&empty[s], 1);
      }
      for (int i = 0; i < 3; ++i) {
        mbar_init(&lo_full[i], LO_WARPS);
        mbar_init(&lo_empty[i], 1);
      }
      for (int i = 0; i < 2; ++i) {
        mbar_init(&tmem_full[i], 1);
        mbar_init(&tmem_empty[i], 4);
      }
      fence_mbar_init();
      tma_prefetch_desc(&tmap_a);
      tma_prefetch_desc(&tmap_hi);
      if (MODE == 1) tma_prefetch_desc(&tmap_lo);
    }
    __syncwarp();
    tmem_alloc(tmem_holder, C::TMEM_COLS);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;
  griddep_wait();  // B-hat is the previous kernel's output (K1)

  if (warp == TMA_WARP) {
    // ------------------------------------------------------------ TMA producer: B-hat tile + filter tile per stage
    if (elect_one()) {
      constexpr uint32_t bytes = C::STAGE;
      uint32_t it = 0;
      for (int64_t w = blockIdx.x; w < a.items; w += gridDim.x) {
        const Item x = decode(a, w);
        for (int kt = x.kt0; kt < x.kt1; ++kt, ++it) {
          const int s = it % C::STAGES;
          const uint32_t ph = (it / C::STAGES) & 1;
          mbar_wait(&empty[s], ph ^ 1);
          mbar_arrive_expect_tx(&full[s], bytes);
          tma_load_2d(smem_u32(a_tile(s)), &tmap_a, &full[s], kt * BK, x.mt * BM);
#pragma unroll
          for (int j = 0; j < (BN + 31) / 32; ++j) {
            tma_load_2d(smem_u32(b_tile(s)) + j * 4096, &tmap_hi, &full[s], x.nt * BN + 32 * j, kt * BK);
            if (MODE == 1)
              tma_load_2d(smem_u32(b_lo_tma(s)) + j * 4096, &tmap_lo, &full[s], x.nt * BN + 32 * j, kt * BK);
          }
        }
      }
    }
  } else if (warp == MMA_WARP) {
    // ------------------------------------------------------------ MMA issuer
    constexpr uint32_t idesc = idesc_tf32(BN < 32 ? 32 : BN, /*a_mn=*/false, /*b_mn=*/true);
    if (elect_one()) {
      uint32_t it = 0, ti = 0;
      for (int64_t w = blockIdx.x; w < a.items; w += gridDim.x, ++ti) {
        const Item x = decode(a, w);
        const uint32_t as = ti & 1, aph = (ti >> 1) & 1;
        mbar_wait_spin(&tmem_empty[as], aph ^ 1);
        tc_fence_after();
        const uint32_t d = tmem_base + as * BN;
        for (int kt = x.kt0; kt < x.kt1; ++kt, ++it) {
          const int s = it % C::STAGES;
          const uint32_t ph = (it / C::STAGES) & 1;
          mbar_wait_spin(&full[s], ph);
          tc_fence_after();
          const uint32_t a_hi = smem_u32(a_tile(s)), b_hi = smem_u32(b_tile(s));
          // A: K-major SW128, k-step = +32 B inside the swizzle row; 8-row groups 1024 B apart.
          // F: MN-major SW128 with 32-byte atoms: k-step = +1024 B, 4-row groups 512 B apart,
          //    32-filter blocks 4096 B apart.
#pragma unroll
          for (int kk = 0; kk < BK / 8; ++kk) {
            const uint64_t ad = smem_desc(a_hi + kk * 32, 16, 1024);
            const uint64_t bd = smem_desc(b_hi + kk * 1024, 4096, 512, 0, kLayoutSW128_32B);
            mma_tf32(d, ad, bd, idesc, (kt != x.kt0 || kk != 0) ? 1u : 0u);
          }
          if (SPLIT) {
            if (MODE == 1) {  // pre-split filter lo arrived with the stage
              const uint32_t b_lo = smem_u32(b_lo_tma(s));
#pragma unroll
              for (int kk = 0; kk < BK / 8; ++kk)
                mma_tf32(d, smem_desc(a_hi + kk * 32, 16, 1024),
                         smem_desc(b_lo + kk * 1024, 4096, 512, 0, kLayoutSW128_32B), idesc, 1);
            }
            const int l = it % LOS;
            mbar_wait_spin(&lo_full[l], (it / LOS) & 1);
            tc_fence_after();
            const uint32_t al = smem_u32(a_lo(l));
#pragma unroll
            for (int kk = 0; kk < BK / 8; ++kk) {
              const uint64_t bd = smem_desc(b_hi + kk * 1024, 4096, 512, 0, kLayoutSW128_32B);
              mma_tf32(d, smem_desc(al + kk * 32, 16, 1024), bd, idesc, 1);
              if (FLO)
                mma_tf32(d, smem_desc(a_hi + kk * 32, 16, 1024),
                         smem_desc(smem_u32(b_lo_flo(l)) + kk * 1024, 4096, 512, 0, kLayoutSW128_32B), idesc, 1);
            }
            mma_commit(&lo_empty[l]);
          }
          mma_commit(&empty[s]);
        }
        mma_commit(&tmem_full[as]);
      }
    }
  } else if (warp < LO_WARP0) {
    // ------------------------------------------------------------ epilogue: TMEM -> registers -> O (or partial tile)
    const int q = warp % 4;
    const int row = q * 32 + lane;
    uint32_t ti = 0;
    for (int64_t w = blockIdx.x; w < a.items; w += gridDim.x, ++ti) {
      const Item x = decode(a, w);
      const uint32_t as = ti & 1, aph = (ti >> 1) & 1;
      mbar_wait_warp(&tmem_full[as], aph);
      tc_fence_after();
      const int64_t P = (int64_t)x.mt * BM + row;
      const int n0 = x.nt * BN;
      float* dst_row;
      int vec = a.vec;
      if (a.S > 1) {
        const int64_t tile = (int64_t)x.mt * a.n_tiles + x.nt;
        dst_row = a.ws + ((tile * a.S + x.piece) * BM + row) * BN;
        vec = 2;
      } else {
        dst_row = a.O + P * a.k_n + n0;
      }
#pragma unroll 1
      for (int cb = 0; cb < (BN + 31) / 32; ++cb) {
        uint32_t r[32];
        tmem_ld_32x32b_x32(tmem_base + ((uint32_t)(q * 32) << 16) + as * BN + cb * 32, r);
        tmem_ld_wait();
        const int ncols = a.S > 1 ? 32 : min(32, a.k_n - (n0 + cb * 32));
        if (P < a.n && ncols > 0) store_row32(dst_row + cb * 32, r, ncols, vec);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tmem_empty[as]);
    }
  } else if (SPLIT) {
    // ------------------------------------------------------------ lo warps: lo = rna_tf32(x - trunc_tf32(x))
    const int t = (warp - LO_WARP0) * 32 + lane;
    uint32_t it = 0;
    // explicit shared-space accesses (through generic pointers the compiler emitted
    // LD.E/ST.E and serialised every load behind the previous store), four 16-byte loads
    // in flight per lane before the first store
    auto split_tile = [&](const uint8_t* src, uint8_t* dst, int bytes) {
      const uint32_t s0 = smem_u32(src) + t * 16, d0 = smem_u32(dst) + t * 16;
      constexpr int STEP = LO_WARPS * 32 * 16;  // 4 KB per pass of the 8 warps
      for (int off = 0; off < bytes; off += 4 * STEP) {
        float v[4][4];
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (off + u * STEP < bytes)
          asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                       : "=f"(v[u][0]), "=f"(v[u][1]), "=f"(v[u][2]), "=f"(v[u][3])
                       : "r"(s0 + off + u * STEP));
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (off + u * STEP < bytes)
          st_shared_v4(d0 + off + u * STEP, to_tf32(v[u][0] - tf32_trunc(v[u][0])),
                       to_tf32(v[u][1] - tf32_trunc(v[u][1])), to_tf32(v[u][2] - tf32_trunc(v[u][2])),
                       to_tf32(v[u][3] - tf32_trunc(v[u][3])));
      }
    };
    for (int64_t w = blockIdx.x; w < a.items; w += gridDim.x) {
      const Item x = decode(a, w);
      for (int kt = x.kt0; kt < x.kt1; ++kt, ++it) {
        const int s = it % C::STAGES;
        const uint32_t ph = (it / C::STAGES) & 1;
        const int l = it % LOS;
        // suspending try_wait, one polling lane per warp: spinning test_wait lanes measured
        // 1.6x slower on the N = 64 shapes (their polls compete with the shared-memory-bound
        // UMMAs) and no faster elsewhere
        mbar_wait_warp(&lo_empty[l], ((it / LOS) & 1) ^ 1);
        mbar_wait_warp(&full[s], ph);
        split_tile(a_tile(s), a_lo(l), A_TILE);
        if (FLO) split_tile(b_tile(s), b_lo_flo(l), C::B_TILE);
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(&lo_full[l]);
      }
    }
  }
  griddep_launch_dependents();
  tc_fence_before();
  __syncthreads();
  if (warp == TMA_WARP) {
    __syncwarp();
    tc_fence_after();
    tmem_dealloc(tmem_base, C::TMEM_COLS);
  }
}

// Ordered sum of the S partial tiles of every output element (split-K shapes).
template <int BN>
__global__ void __launch_bounds__(256) k2_reduce_kernel(Args a) {
  griddep_wait();
  const int64_t q4 = a.k_n / 4;  // float4 groups per output row (k_n % 4 == 0 on this path)
  const int64_t total = a.n * q4;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t P = i / q4;
    const int32_t col = (int32_t)(i - P * q4) * 4;
    const int32_t mt = (int32_t)(P / BM), row = (int32_t)(P % BM);
    const int32_t nt = col / BN, cc = col % BN;
    const float* src = a.ws + ((((int64_t)mt * a.n_tiles + nt) * a.S) * BM + row) * BN + cc;
    float acc[4];
    ld_global_cg_v4(src, acc);
    for (int sp = 1; sp < a.S; ++sp) {
      float v[4];
      ld_global_cg_v4(src + (int64_t)sp * BM * BN, v);
#pragma unroll
      for (int e = 0; e < 4; ++e) acc[e] += v[e];
    }
    float* dst = a.O + P * a.k_n + col;
    if (a.vec) {  // O 16-byte aligned
      *reinterpret_cast<float4*>(dst) = make_float4(acc[0], acc[1], acc[2], acc[3]);
    } else {
#pragma unroll
      for (int e = 0; e < 4; ++e) dst[e] = acc[e];
    }
  }
}

template <int BN, int MODE>
cudaError_t launch_cfg(const CUtensorMap& ta, const CUtensorMap& th, const CUtensorMap& tl, Args a, int sms,
                       cudaStream_t st) {
  using C = Cfg<BN, MODE>;
  auto kern = k2_gemm_kernel<BN, MODE>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
  if (e != cudaSuccess) return e;
  const Tuning tu = tuning();
  a.n_tiles = (a.k_n + BN - 1) / BN;
  const int64_t tiles = (int64_t)a.m_tiles * a.n_tiles;
  // split-K when the tiles cannot occupy half the SMs: S pieces of >= 4 chunks each
  a.S = 1;
  if (a.k_n % 4 == 0 && tu.splitk >= 0) {
    int S = 1;
    if (tu.splitk > 0) S = std::min(tu.splitk, a.KT);
    else if (2 * tiles <= sms) S = (int)std::min<int64_t>(std::max(a.KT / 4, 1), sms / tiles);
    if (S > 1) {
      int* counters = nullptr;
      float* ws = nullptr;
      const size_t ws_bytes = (size_t)tiles * S * BM * BN * sizeof(float);
      if (sw::sk_buffers(st, 0, ws_bytes, &counters, &ws) && ws) {
        a.S = S;
        a.ws = ws;
      }
    }
  }
  a.items = tiles * a.S;
  const unsigned grid = (unsigned)std::min<int64_t>(a.items, sms);
  cudaLaunchConfig_t lc{};
  lc.gridDim = dim3(grid);
  lc.blockDim = dim3(C::THREADS);
  lc.dynamicSmemBytes = C::SMEM;
  lc.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  lc.attrs = at;
  lc.numAttrs = tu.pdl ? 1 : 0;
  if ((e = cudaLaunchKernelEx(&lc, kern, ta, th, tl, a)) != cudaSuccess) return e;
  count_launch();
  if (a.S > 1) {
    cudaLaunchConfig_t rc = lc;
    const int64_t total = a.n * (a.k_n / 4);
    rc.gridDim = dim3((unsigned)std::min<int64_t>((total + 255) / 256, (int64_t)sms * 8));
    rc.blockDim = dim3(256);
    rc.dynamicSmemBytes = 0;
    if ((e = cudaLaunchKernelEx(&rc, k2_reduce_kernel<BN>, a)) != cudaSuccess) return e;
    count_launch();
  }
  return cudaGetLastError();
}

}  // namespace k2

cudaError_t launch_k2_gemm(const float* f_hi, const float* f_lo, int64_t ldf, const float* Bhat, int64_t ldb,
                           float* O, const ConvGeom& g, bool split, cudaStream_t st) {
  if (ldb % 4 != 0 || reinterpret_cast<uintptr_t>(Bhat) % 16 != 0) return cudaErrorNotSupported;
  k2::Args a{};
  a.O = O;
  a.ws = nullptr;
  a.n = g.n;
  a.k_n = (int32_t)g.k_n;
  a.KT = (int32_t)((g.k + k2::BK - 1) / k2::BK);
  a.m_tiles = (int32_t)((g.n + k2::BM - 1) / k2::BM);
  a.nt_fast = g.n >= g.k_n;
  a.vec = 0;
  if (g.k_n % 8 == 0 && reinterpret_cast<uintptr_t>(O) % 32 == 0) a.vec = 2;
  else if (g.k_n % 4 == 0 && reinterpret_cast<uintptr_t>(O) % 16 == 0) a.vec = 1;
  CUtensorMap ta, th, tl;
  cudaError_t e = make_bhat_tmap(&ta, Bhat, g.k, g.n, ldb);
  if (e != cudaSuccess) return e;
  if ((e = make_filter_tmap(&th, f_hi, g.k_n, g.k, ldf)) != cudaSuccess) return e;
  if (split && f_lo) {
    if ((e = make_filter_tmap(&tl, f_lo, g.k_n, g.k, ldf)) != cudaSuccess) return e;
  } else {
    tl = th;
  }
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t kn = g.k_n;
  const int mode = !split ? 0 : (f_lo ? 1 : 2);
#define CGB_K2_DISPATCH(BN)                                                   \
  return mode == 0   ? k2::launch_cfg<BN, 0>(ta, th, tl, a, sms, st)          \
         : mode == 1 ? k2::launch_cfg<BN, 1>(ta, th, tl, a, sms, st)          \
                     : k2::launch_cfg<BN, 2>(ta, th, tl, a, sms, st);
  if (kn <= 32) { CGB_K2_DISPATCH(32) }
  if (kn <= 64) { CGB_K2_DISPATCH(64) }
  if (kn <= 128) { CGB_K2_DISPATCH(128) }
  CGB_K2_DISPATCH(256)
#undef CGB_K2_DISPATCH
}

}  // namespace cgb
