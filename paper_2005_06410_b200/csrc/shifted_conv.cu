// shifted_conv.cu -- V2: "shifted window" tcgen05 implicit GEMM for stride-1 convolutions.
//
// The reference materialises (explicit path, im2col.hpp:77-120) or packs on the fly
// (fused path, pack_b_im2col im2col.hpp:177-262) k_h*k_w shifted copies of every
// input element. On B200 the copies are unnecessary: index output pixels in the
// *padded* plane, m' = i_h + H_q*(i_w + W_q*i_b) with H_q = h_i + 2p, W_q = w_i + 2p
// (rows with i_h >= h_o or i_w >= w_o are computed and discarded), and the A operand
// of filter tap (kh, kw) is the padded input window shifted by d = kh + H_q*kw rows.
// A K-major, 128B-swizzled shared-memory window (one 128-byte row = 32 channels of one
// padded pixel) is therefore staged ONCE per 32-channel chunk, and each tap's UMMA
// reads it through a descriptor whose start address is moved by d rows. Swizzling is
// applied on absolute shared addresses, so arbitrary row shifts are legal with
// base_offset 0 (measured on B200: tools/umma_probe.cu).
//
// Per tile (MT x 128 padded pixels, BN filters), per channel chunk cc:
//   producers stage rows [m0, m0 + MT*128 + dmax) x 32 channels (LDG -> TF32 round or
//   3xTF32 split -> STS, zero rows for padding / past the batch),
//   the TMA warp streams F[n0:n0+BN, tap, cc*32:+32] boxes (3-D map, MN-major),
//   the MMA warp issues taps x 4 k-steps x MT UMMAs (M=128, N=BN, K=8) per chunk.
// Persistent: grid = #SMs, static round-robin tiles, two TMEM accumulator sets so the
// epilogue of tile i overlaps the main loop of tile i+1.
//
// Roles (448 threads): warps 0-7 A producers, warp 8 filter TMA + TMEM alloc,
// warp 9 MMA issue, warps 10-13 epilogue (TMEM lanes 64*... per warp%4).
#include <algorithm>

#include "internal.h"

namespace cgb {
namespace sw {

constexpr int BK = 32;
constexpr int PRODUCER_WARPS = 8;
constexpr int TMA_WARP = 8;
constexpr int MMA_WARP = 9;
constexpr int EPI_WARP0 = 10;
constexpr int THREADS = 14 * 32;

struct Args {
  int32_t k_n, k_h, k_w, c_i, h_i, w_i, p, h_o, w_o, b;
  int32_t Hq, Wq;     // padded plane
  int32_t dmax;       // (k_h-1) + Hq*(k_w-1)
  int32_t R;          // staged rows per chunk = MT*128 + dmax
  int32_t CC;         // channel chunks
  int32_t taps;
  int32_t m_tiles, n_tiles;
  int64_t Mp;         // padded output rows Hq*Wq*b
  int64_t plane;      // h_i*w_i
};

template <int MT, int BN, bool SPLIT, int A_SLOTS, int B_STAGES>
struct Cfg {
  static constexpr int NS = SPLIT ? 2 : 1;
  static constexpr int B_TILE = BN * BK * 4;
  static constexpr int ACC_COLS = MT * BN;  // per accumulator set
  static constexpr int TMEM_COLS = 2 * ACC_COLS <= 512 ? 2 * ACC_COLS : ACC_COLS;
  static constexpr int ACC_SETS = 2 * ACC_COLS <= 512 ? 2 : 1;
  static constexpr int UMMA_N = BN > 256 ? 256 : BN;
};

template <int MT, int BN, bool SPLIT, int A_SLOTS, int B_STAGES>
__global__ void __launch_bounds__(THREADS, 1)
    sw_conv_kernel(const __grid_constant__ CUtensorMap tmap_hi, const __grid_constant__ CUtensorMap tmap_lo,
                   const float* __restrict__ I, float* __restrict__ O, Args a, uint32_t a_slot_bytes) {
  using C = Cfg<MT, BN, SPLIT, A_SLOTS, B_STAGES>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  // [A slots: A_SLOTS x NS x a_slot_bytes][B stages: B_STAGES x NS x B_TILE][barriers]
  auto a_slot = [&](int s, int part) { return smem + (s * C::NS + part) * a_slot_bytes; };
  uint8_t* b_base = smem + A_SLOTS * C::NS * a_slot_bytes;
  auto b_slot = [&](int s, int part) { return b_base + (s * C::NS + part) * C::B_TILE; };
  uint64_t* bars = reinterpret_cast<uint64_t*>(b_base + B_STAGES * C::NS * C::B_TILE);
  uint64_t* a_full = bars;
  uint64_t* a_empty = a_full + A_SLOTS;
  uint64_t* b_full = a_empty + A_SLOTS;
  uint64_t* b_empty = b_full + B_STAGES;
  uint64_t* t_full = b_empty + B_STAGES;
  uint64_t* t_empty = t_full + 2;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(t_empty + 2);

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const int total_tiles = a.m_tiles * a.n_tiles;

  if (warp == TMA_WARP) {
    if (lane == 0) {
      for (int s = 0; s < A_SLOTS; ++s) {
        mbar_init(&a_full[s], PRODUCER_WARPS);
        mbar_init(&a_empty[s], 1);
      }
      for (int s = 0; s < B_STAGES; ++s) {
        mbar_init(&b_full[s], 1);
        mbar_init(&b_empty[s], 1);
      }
      for (int s = 0; s < 2; ++s) {
        mbar_init(&t_full[s], 1);
        mbar_init(&t_empty[s], 4);
      }
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
    // ---------------------------------------------------------------- window producers
    // warp w stages row blocks rb = w, w+8, ...: lane = row within the block (32
    // consecutive padded pixels -> coalesced reads per channel), 32 channels per row.
    const int row_blocks = (a.R + 31) / 32;
    const int32_t hw_q = a.Hq * a.Wq;
    int it = 0;  // chunk counter across tiles (slot ring position)
    for (int tile = blockIdx.x; tile < total_tiles; tile += gridDim.x) {
      const int64_t m0 = (int64_t)(tile % a.m_tiles) * (MT * 128);
      for (int cc = 0; cc < a.CC; ++cc, ++it) {
        const int s = it % A_SLOTS;
        const uint32_t ph = (it / A_SLOTS) & 1;
        mbar_wait(&a_empty[s], ph ^ 1);
        uint8_t* dst_hi = a_slot(s, 0);
        uint8_t* dst_lo = a_slot(s, SPLIT ? 1 : 0);
        for (int rb = warp; rb < row_blocks; rb += PRODUCER_WARPS) {
          const int row = rb * 32 + lane;
          const int64_t Q = m0 + row;
          bool ok = row < a.R && Q < a.Mp;
          const float* src = I;
          if (ok) {
            const int32_t bb = (int32_t)(Q / hw_q);
            const int32_t rem = (int32_t)(Q - (int64_t)bb * hw_q);
            const int32_t wq = rem / a.Hq, hq = rem - wq * a.Hq;
            const int32_t h = hq - a.p, w = wq - a.p;
            ok = (unsigned)h < (unsigned)a.h_i && (unsigned)w < (unsigned)a.w_i;
            src = I + ((int64_t)bb * a.c_i + (int64_t)cc * BK) * a.plane + (int64_t)w * a.h_i + h;
          }
          const int cmax = a.c_i - cc * BK;  // channels available in this chunk
          float v[BK];
#pragma unroll
          for (int c = 0; c < BK; ++c) v[c] = (ok && c < cmax) ? __ldg(src + c * a.plane) : 0.0f;
          if (row < a.R) {
#pragma unroll
            for (int ch = 0; ch < 8; ++ch) {
              const uint32_t off = row * 128 + ((ch ^ (row & 7)) << 4);
              float4 hi, lo;
              float* h = &hi.x;
              float* l = &lo.x;
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                const float x = v[4 * ch + e];
                const float t = to_tf32(x);
                h[e] = t;
                if (SPLIT) l[e] = to_tf32(x - t);
              }
              *reinterpret_cast<float4*>(dst_hi + off) = hi;
              if (SPLIT) *reinterpret_cast<float4*>(dst_lo + off) = lo;
            }
          }
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(&a_full[s]);
      }
    }
  } else if (warp == TMA_WARP) {
    // ---------------------------------------------------------------- filter TMA
    if (elect_one()) {
      constexpr uint32_t bytes = C::NS * C::B_TILE;
      int it = 0;
      for (int tile = blockIdx.x; tile < total_tiles; tile += gridDim.x) {
        const int n0 = (tile / a.m_tiles) * BN;
        for (int cc = 0; cc < a.CC; ++cc)
          for (int tap = 0; tap < a.taps; ++tap, ++it) {
            const int s = it % B_STAGES;
            const uint32_t ph = (it / B_STAGES) & 1;
            mbar_wait(&b_empty[s], ph ^ 1);
            mbar_arrive_expect_tx(&b_full[s], bytes);
#pragma unroll
            for (int j = 0; j < BN / 32; ++j) {
              tma_load_3d(smem_u32(b_slot(s, 0)) + j * 4096, &tmap_hi, &b_full[s], n0 + 32 * j, tap, cc * BK);
              if (SPLIT)
                tma_load_3d(smem_u32(b_slot(s, 1)) + j * 4096, &tmap_lo, &b_full[s], n0 + 32 * j, tap, cc * BK);
            }
          }
      }
    }
  } else if (warp == MMA_WARP) {
    // ---------------------------------------------------------------- MMA issue
    constexpr uint32_t idesc = idesc_tf32(C::UMMA_N, false, true);
    if (elect_one()) {
      int ait = 0, bit = 0, t = 0;
      for (int tile = blockIdx.x; tile < total_tiles; tile += gridDim.x, ++t) {
        const int acc_set = C::ACC_SETS == 2 ? (t & 1) : 0;
        const uint32_t acc_ph = C::ACC_SETS == 2 ? ((t >> 1) & 1) : (t & 1);
        mbar_wait(&t_empty[acc_set], acc_ph ^ 1);
        tc_fence_after();
        const uint32_t d_base = tmem_base + acc_set * C::ACC_COLS;
        for (int cc = 0; cc < a.CC; ++cc, ++ait) {
          const int as = ait % A_SLOTS;
          mbar_wait(&a_full[as], (ait / A_SLOTS) & 1);
          tc_fence_after();
          const uint32_t a_hi = smem_u32(a_slot(as, 0));
          const uint32_t a_lo = smem_u32(a_slot(as, SPLIT ? 1 : 0));
          for (int tap = 0; tap < a.taps; ++tap, ++bit) {
            const int bs = bit % B_STAGES;
            mbar_wait(&b_full[bs], (bit / B_STAGES) & 1);
            tc_fence_after();
            const int kh = tap % a.k_h, kw = tap / a.k_h;
            const uint32_t d_rows = kh + a.Hq * kw;
            const uint32_t b_hi = smem_u32(b_slot(bs, 0));
            const uint32_t b_lo = smem_u32(b_slot(bs, SPLIT ? 1 : 0));
#pragma unroll
            for (int kk = 0; kk < BK / 8; ++kk) {
#pragma unroll
              for (int hf = 0; hf < BN / C::UMMA_N; ++hf) {
                const uint32_t boff = hf * (C::UMMA_N / 32) * 4096 + kk * 1024;
                const uint64_t bd = smem_desc(b_hi + boff, 4096, 512, 0, kLayoutSW128_32B);
                const uint64_t bd_lo = SPLIT ? smem_desc(b_lo + boff, 4096, 512, 0, kLayoutSW128_32B) : 0;
#pragma unroll
                for (int mt = 0; mt < MT; ++mt) {
                  const uint32_t aoff = (mt * 128 + d_rows) * 128 + kk * 32;
                  const uint64_t ad = smem_desc(a_hi + aoff, 16, 1024);
                  const uint32_t d = d_base + mt * BN + hf * C::UMMA_N;
                  const uint32_t acc = (cc | tap | kk) != 0;
                  if (SPLIT) {
                    const uint64_t ad_lo = smem_desc(a_lo + aoff, 16, 1024);
                    mma_tf32(d, ad_lo, bd, idesc, acc);
                    mma_tf32(d, ad, bd_lo, idesc, 1);
                    mma_tf32(d, ad, bd, idesc, 1);
                  } else {
                    mma_tf32(d, ad, bd, idesc, acc);
                  }
                }
              }
            }
            mma_commit(&b_empty[bs]);
          }
          mma_commit(&a_empty[as]);
        }
        mma_commit(&t_full[acc_set]);
      }
    }
  } else {
    // ---------------------------------------------------------------- epilogue
    const int ew = warp - EPI_WARP0;      // 0..3
    const int sub = warp % 4;             // TMEM lane quadrant this warp may access
    const int32_t hw_q = a.Hq * a.Wq;
    const bool vec = (a.k_n % 4) == 0;
    int t = 0;
    for (int tile = blockIdx.x; tile < total_tiles; tile += gridDim.x, ++t) {
      const int acc_set = C::ACC_SETS == 2 ? (t & 1) : 0;
      const uint32_t acc_ph = C::ACC_SETS == 2 ? ((t >> 1) & 1) : (t & 1);
      const int64_t m0 = (int64_t)(tile % a.m_tiles) * (MT * 128);
      const int n0 = (tile / a.m_tiles) * BN;
      mbar_wait(&t_full[acc_set], acc_ph);
      tc_fence_after();
#pragma unroll 1
      for (int mt = 0; mt < MT; ++mt) {
        const int64_t Q = m0 + mt * 128 + sub * 32 + lane;
        int64_t P = -1;
        if (Q < a.Mp) {
          const int32_t bb = (int32_t)(Q / hw_q);
          const int32_t rem = (int32_t)(Q - (int64_t)bb * hw_q);
          const int32_t wq = rem / a.Hq, hq = rem - wq * a.Hq;
          if (hq < a.h_o && wq < a.w_o) P = hq + (int64_t)a.h_o * (wq + (int64_t)a.w_o * bb);
        }
#pragma unroll 1
        for (int cb = 0; cb < BN / 32; ++cb) {
          uint32_t r[32];
          tmem_ld_32x32b_x32(tmem_base + ((uint32_t)(sub * 32) << 16) + acc_set * C::ACC_COLS + mt * BN + cb * 32,
                             r);
          tmem_ld_wait();
          const int nb = n0 + cb * 32;
          if (P >= 0 && nb < a.k_n) {
            float* dst = O + P * a.k_n + nb;
            if (vec && nb + 32 <= a.k_n) {
#pragma unroll
              for (int j = 0; j < 32; j += 4)
                *reinterpret_cast<float4*>(dst + j) =
                    make_float4(__uint_as_float(r[j]), __uint_as_float(r[j + 1]), __uint_as_float(r[j + 2]),
                                __uint_as_float(r[j + 3]));
            } else {
#pragma unroll
              for (int j = 0; j < 32; ++j)
                if (nb + j < a.k_n) dst[j] = __uint_as_float(r[j]);
            }
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&t_empty[acc_set]);
      (void)ew;
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

template <int MT, int BN, bool SPLIT, int A_SLOTS, int B_STAGES>
cudaError_t launch_cfg(const CUtensorMap& th, const CUtensorMap& tl, const float* I, float* O, Args a,
                       cudaStream_t st) {
  using C = Cfg<MT, BN, SPLIT, A_SLOTS, B_STAGES>;
  a.R = MT * 128 + a.dmax;
  const uint32_t a_slot_bytes = (uint32_t)(((a.R + 7) / 8) * 8 * 128);
  const size_t smem = (size_t)A_SLOTS * C::NS * a_slot_bytes + (size_t)B_STAGES * C::NS * C::B_TILE + 1024 + 256;
  if (smem > 227 * 1024) return cudaErrorNotSupported;
  a.m_tiles = (int32_t)((a.Mp + MT * 128 - 1) / (MT * 128));
  a.n_tiles = (a.k_n + BN - 1) / BN;
  auto kern = sw_conv_kernel<MT, BN, SPLIT, A_SLOTS, B_STAGES>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int tiles = a.m_tiles * a.n_tiles;
  kern<<<std::min(tiles, sms), THREADS, smem, st>>>(th, tl, I, O, a, a_slot_bytes);
  count_launch();
  return cudaGetLastError();
}

static Args make_args(const ConvGeom& g) {
  Args a;
  a.k_n = (int32_t)g.k_n; a.k_h = (int32_t)g.k_h; a.k_w = (int32_t)g.k_w; a.c_i = (int32_t)g.c_i;
  a.h_i = (int32_t)g.h_i; a.w_i = (int32_t)g.w_i; a.p = (int32_t)g.p; a.h_o = (int32_t)g.h_o;
  a.w_o = (int32_t)g.w_o; a.b = (int32_t)g.b;
  a.Hq = (int32_t)(g.h_o + g.k_h - 1);
  a.Wq = (int32_t)(g.w_o + g.k_w - 1);
  a.dmax = (a.k_h - 1) + a.Hq * (a.k_w - 1);
  a.CC = (a.c_i + BK - 1) / BK;
  a.taps = a.k_h * a.k_w;
  a.Mp = (int64_t)a.Hq * a.Wq * g.b;
  a.plane = g.h_i * g.w_i;
  a.R = 0; a.m_tiles = 0; a.n_tiles = 0;
  return a;
}

}  // namespace sw

// Domain: stride 1, filters through the tap-major TMA map (k_n % 4 == 0), enough
// channels per chunk to be worth a window, and little garbage from the padded plane.
bool shifted_supported(const ConvGeom& g) {
  if (g.s != 1 || g.k_n % 4 != 0 || g.c_i < 16 || g.k_n > 256) return false;
  const double waste = (double)((g.h_o + g.k_h - 1) * (g.w_o + g.k_w - 1)) / (double)(g.h_o * g.w_o);
  if (waste > 1.2) return false;
  const int64_t dmax = (g.k_h - 1) + (g.h_o + g.k_h - 1) * (g.k_w - 1);
  return dmax <= 512;
}

cudaError_t launch_tc_conv_shifted(const float* f_hi, const float* f_lo, int64_t ldf, const float* I, float* O,
                                   const ConvGeom& g, bool split, cudaStream_t st) {
  (void)ldf;
  sw::Args a = sw::make_args(g);
  CUtensorMap th, tl;
  cudaError_t e = make_filter_tmap_tapmajor(&th, f_hi, g);
  if (e != cudaSuccess) return e;
  if (split) {
    if ((e = make_filter_tmap_tapmajor(&tl, f_lo, g)) != cudaSuccess) return e;
  } else {
    tl = th;
  }
  const int64_t kn = g.k_n;
  if (kn <= 64) {
    if (split) {
      e = sw::launch_cfg<2, 64, true, 1, 4>(th, tl, I, O, a, st);
      if (e != cudaErrorNotSupported) return e;
      return sw::launch_cfg<1, 64, true, 1, 4>(th, tl, I, O, a, st);
    }
    e = sw::launch_cfg<4, 64, false, 2, 6>(th, tl, I, O, a, st);
    if (e != cudaErrorNotSupported) return e;
    return sw::launch_cfg<2, 64, false, 2, 6>(th, tl, I, O, a, st);
  }
  if (kn <= 128) {
    if (split) {
      e = sw::launch_cfg<2, 128, true, 1, 3>(th, tl, I, O, a, st);
      if (e != cudaErrorNotSupported) return e;
      return sw::launch_cfg<1, 128, true, 1, 3>(th, tl, I, O, a, st);
    }
    e = sw::launch_cfg<2, 128, false, 2, 4>(th, tl, I, O, a, st);
    if (e != cudaErrorNotSupported) return e;
    return sw::launch_cfg<1, 128, false, 2, 4>(th, tl, I, O, a, st);
  }
  if (split) return sw::launch_cfg<1, 256, true, 1, 2>(th, tl, I, O, a, st);
  return sw::launch_cfg<1, 256, false, 2, 3>(th, tl, I, O, a, st);
}

}  // namespace cgb
