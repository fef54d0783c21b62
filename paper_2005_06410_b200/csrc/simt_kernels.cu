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

// Slab version for 16-byte-aligned B (the explicit path's workspace): a CTA stages the
// input slab of one (image, h tile, w tile, channel block) in shared memory -- padding
// zeros included, filled by cp.async with lanes along h (coalesced, every load of the CTA
// in flight at once) -- then writes its piece of every lowered column with lanes along
// r: one 16-byte store per lane, 512 contiguous bytes per warp instruction. The r ->
// slab offset map is pixel-independent: it is built once per CTA and each lane keeps the
// offsets of its chunks in registers, so the write loop is 4 LDS + 1 STG per 16 bytes
// with no bounds checks and no divisions. The kernel is issue-bound (ncu: 78% of the
// issue slots), hence the care about instruction counts.
//   V   elements per cp.async (2 needs an even h_i and an 8-byte aligned I)
//   NCL chunks (16 B) per lane held in registers; 0 = any count (offsets re-read per pixel)
struct SlabArgs {
  int32_t k_h, k_w, c_i, h_i, w_i, s, p, h_o, w_o, K;
  int32_t CB, NCB, HT, NHT, WT, NWT, HP, HPpad, WS, RB;
  int64_t ldb, plane;
  // flat write phase (short columns: K <= ~100 rows would leave most lanes of the
  // chunk-per-lane loop idle): one channel block, one output column per CTA, so the CTA's
  // piece of B is one contiguous run and item = pixel * chunks + chunk indexes it directly
  int32_t flat;
  uint32_t nch_m, nch_p;  // item / chunks as a multiply-shift
  uint32_t ho_m, ho_p;    // pixel / h_o likewise (several whole output columns per CTA)
};

template <int V, int NCL>
__global__ void __launch_bounds__(256) im2col_slab_kernel(const float* __restrict__ I, float* __restrict__ B,
                                                         SlabArgs a) {
  extern __shared__ float slab_smem[];
  const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
  int64_t item = blockIdx.x;
  const int cb = (int)(item % a.NCB); item /= a.NCB;
  const int wt = (int)(item % a.NWT); item /= a.NWT;
  const int ht = (int)(item % a.NHT);
  const int i_b = (int)(item / a.NHT);
  const int cbn = min(a.CB, a.c_i - cb * a.CB);                        // channels of this block
  const int nrows = cb == a.NCB - 1 ? (int)a.ldb - cb * a.RB : a.RB;   // lowered rows of this block (% 4 == 0)
  const int slab_floats = (a.CB * a.WS * a.HPpad + 3) & ~3;  // the table is read as int4
  int32_t* table = reinterpret_cast<int32_t*>(slab_smem + slab_floats);
  const int h_base = ht * a.HT, w_base = wt * a.WT;
  const int htn = min(a.HT, a.h_o - h_base), wtn = min(a.WT, a.w_o - w_base);
  const int hp = (htn - 1) * a.s + a.k_h;  // input rows the tile reads
  const int h_first = h_base * a.s - a.p;  // input row of the tile's first tap (may be negative)
  // slab column jj holds input row A0 + jj; A0 is V-aligned so that a cp.async never
  // straddles the image edge and source and destination share their alignment
  const int A0 = h_first & ~(V - 1);
  const int j0 = h_first - A0;
  const int khw = a.k_h * a.k_w;
  for (int r = tid; r < nrows; r += 256) {
    int32_t off = -1;  // rows >= K (zero fill up to ldb)
    if (cb * a.RB + r < a.K) {
      const int c = r / khw, t = r - c * khw;
      const int kw = t / a.k_h, kh = t - kw * a.k_h;
      off = (c * a.WS + kw) * a.HPpad + kh + j0;
    }
    table[r] = off;
  }
  const float* img = I + ((int64_t)i_b * a.c_i + (int64_t)cb * a.CB) * a.plane;
  const uint32_t slab_s = smem_u32(slab_smem);
  {
    const int nv = (j0 + hp + V - 1) / V;  // cp.async per slab row
    const int q8 = 8 / a.WS, r8 = 8 - q8 * a.WS;
    int c = warp / a.WS, wl = warp - c * a.WS;
    for (int row = warp; row < cbn * a.WS; row += 8) {
      const int ww = w_base * a.s - a.p + wl;
      const uint32_t dst = slab_s + (uint32_t)(row * a.HPpad) * 4u;
      if ((unsigned)ww < (unsigned)a.w_i) {
        const float* src = img + (int64_t)c * a.plane + (int64_t)ww * a.h_i + A0;
        for (int q = lane; q < nv; q += 32) {
          const bool ok = (unsigned)(A0 + V * q) < (unsigned)a.h_i;
          const float* sp = src + (ok ? V * q : -A0);  // a valid address either way
          if (V == 2)
            asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(dst + 8u * q), "l"(sp), "r"(ok ? 8u : 0u)
                         : "memory");
          else
            cp_async_4(dst + 4u * q, sp, ok ? 4u : 0u);
        }
      } else {  // a padding column: zeros
        for (int q = lane; q < nv * V; q += 32) slab_smem[row * a.HPpad + q] = 0.0f;
      }
      c += q8;
      wl += r8;
      if (wl >= a.WS) { wl -= a.WS; ++c; }
    }
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
  __syncthreads();

  const int npix = htn * wtn;
  const int nch = nrows / 4;
  const int4* table4 = reinterpret_cast<const int4*>(table);
  float* const Bblk = B + ((int64_t)h_base + (int64_t)w_base * a.h_o + (int64_t)i_b * a.h_o * a.w_o) * a.ldb +
                      (int64_t)cb * a.RB + 4 * lane;
  const int q8 = 8 / htn, r8 = 8 - q8 * htn;
  int wl = warp / htn, hl = warp - wl * htn;
  if (a.flat) {
    const int items = npix * nch;
    float* const Bcta = B + ((int64_t)h_base + (int64_t)w_base * a.h_o + (int64_t)i_b * a.h_o * a.w_o) * a.ldb;
    for (int it = tid; it < items; it += 256) {
      const int pix = (int)(((uint64_t)(uint32_t)it * a.nch_m) >> a.nch_p);
      const int ch = it - pix * nch;
      const int4 o = table4[ch];
      // WT > 1 only with whole output columns (htn == h_o): the pixels stay one contiguous run
      const int wl = a.WT == 1 ? 0 : (int)(((uint64_t)(uint32_t)pix * a.ho_m) >> a.ho_p);
      const float* sp = slab_smem + (wl * a.s) * a.HPpad + (pix - wl * htn) * a.s;
      float4 v;
      v.x = o.x < 0 ? 0.0f : sp[o.x];
      v.y = o.y < 0 ? 0.0f : sp[o.y];
      v.z = o.z < 0 ? 0.0f : sp[o.z];
      v.w = o.w < 0 ? 0.0f : sp[o.w];
      *reinterpret_cast<float4*>(Bcta + 4 * (int64_t)it) = v;
    }
    return;
  }
  if constexpr (NCL > 0) {
    // pixel-outer: the lane's chunk offsets live in registers
    int4 o[NCL];
#pragma unroll
    for (int i = 0; i < NCL; ++i) {
      const int ch = lane + 32 * i;
      o[i] = ch < nch ? table4[ch] : make_int4(-2, -2, -2, -2);
    }
    for (int pix = warp; pix < npix; pix += 8) {
      const float* sp = slab_smem + (wl * a.s) * a.HPpad + hl * a.s;
      float* dst = Bblk + (int64_t)(hl + wl * a.h_o) * a.ldb;
#pragma unroll
      for (int i = 0; i < NCL; ++i) {
        if (o[i].w >= 0) {  // offsets grow with r: the common, fully valid chunk
          *reinterpret_cast<float4*>(dst + 128 * i) = make_float4(sp[o[i].x], sp[o[i].y], sp[o[i].z], sp[o[i].w]);
        } else if (o[i].x != -2) {  // the chunk that crosses K (zero fill up to ldb)
          float4 v;
          v.x = o[i].x < 0 ? 0.0f : sp[o[i].x];
          v.y = o[i].y < 0 ? 0.0f : sp[o[i].y];
          v.z = o[i].z < 0 ? 0.0f : sp[o[i].z];
          v.w = 0.0f;
          *reinterpret_cast<float4*>(dst + 128 * i) = v;
        }
      }
      wl += q8;
      hl += r8;
      if (hl >= htn) { hl -= htn; ++wl; }
    }
  } else {
    for (int pix = warp; pix < npix; pix += 8) {
      const float* sp = slab_smem + (wl * a.s) * a.HPpad + hl * a.s;
      float* dst = Bblk + (int64_t)(hl + wl * a.h_o) * a.ldb;
      for (int ch = lane; ch < nch; ch += 32) {
        const int4 o = table4[ch];
        float4 v;
        v.x = o.x < 0 ? 0.0f : sp[o.x];
        v.y = o.y < 0 ? 0.0f : sp[o.y];
        v.z = o.z < 0 ? 0.0f : sp[o.z];
        v.w = o.w < 0 ? 0.0f : sp[o.w];
        *reinterpret_cast<float4*>(dst + 4 * (ch - lane)) = v;
      }
      wl += q8;
      hl += r8;
      if (hl >= htn) { hl -= htn; ++wl; }
    }
  }
}

// Row stride of the slab (>= need, a multiple of V) with the fewest shared-memory bank
// conflicts in the write phase: lanes read the slab at table offsets of rows r = 4*lane + e.
static int best_slab_stride(const SlabArgs& a, int need, int V, int rows) {
  const int khw = a.k_h * a.k_w;
  int best = (need + V - 1) / V * V, best_cost = 1 << 30;
  for (int hp = best; hp < need + 34; hp += V) {
    int cost = 0;
    for (int g0 = 0; g0 < std::min(rows, 512); g0 += 128)
      for (int e = 0; e < 4; ++e) {
        int banks[32] = {0};
        for (int l = 0; l < 32; ++l) {
          const int r = g0 + 4 * l + e;
          if (r >= rows) break;
          const int c = r / khw, t = r - c * khw, kw = t / a.k_h, kh = t - kw * a.k_h;
          ++banks[((c * a.WS + kw) * hp + kh) & 31];
        }
        int mx = 0;
        for (int b = 0; b < 32; ++b) mx = std::max(mx, banks[b]);
        cost += mx;
      }
    if (cost < best_cost) { best_cost = cost; best = hp; }
  }
  return best;
}

template <int V>
static cudaError_t launch_slab_v(int ncl, unsigned blocks, size_t smem, const float* I, float* B, const SlabArgs& a,
                                 cudaStream_t st) {
#define CGB_SLAB_CASE(N)                                                                                     \
  case N: {                                                                                                  \
    auto kern = im2col_slab_kernel<V, N>;                                                                    \
    if (smem > 48 * 1024 &&                                                                                  \
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024) != cudaSuccess)  \
      return cudaGetLastError();                                                                             \
    kern<<<blocks, 256, smem, st>>>(I, B, a);                                                                \
    break;                                                                                                   \
  }
  switch (ncl) {
    CGB_SLAB_CASE(1) CGB_SLAB_CASE(2) CGB_SLAB_CASE(3) CGB_SLAB_CASE(4) CGB_SLAB_CASE(5) CGB_SLAB_CASE(6)
    CGB_SLAB_CASE(8)
    default: {
      auto kern = im2col_slab_kernel<V, 0>;
      if (smem > 48 * 1024 &&
          cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024) != cudaSuccess)
        return cudaGetLastError();
      kern<<<blocks, 256, smem, st>>>(I, B, a);
    }
  }
#undef CGB_SLAB_CASE
  return cudaGetLastError();
}

static bool launch_im2col_slab(const float* I, float* B, int64_t ldb, const ConvGeom& g, cudaStream_t st,
                               cudaError_t* err) {
  SlabArgs a;
  a.k_h = (int32_t)g.k_h; a.k_w = (int32_t)g.k_w; a.c_i = (int32_t)g.c_i; a.h_i = (int32_t)g.h_i;
  a.w_i = (int32_t)g.w_i; a.s = (int32_t)g.s; a.p = (int32_t)g.p; a.h_o = (int32_t)g.h_o; a.w_o = (int32_t)g.w_o;
  a.K = (int32_t)g.k; a.ldb = ldb; a.plane = g.h_i * g.w_i;
  const int V = (g.h_i % 2 == 0 && reinterpret_cast<uintptr_t>(I) % 8 == 0) ? 2 : 1;
  a.HT = (int32_t)std::min<int64_t>(g.h_o, 64);
  a.WT = (int32_t)std::min<int64_t>(g.w_o, std::max(1, 64 / a.HT));  // ~56-64 pixels per CTA
  // Short columns (low-channel layers: K = 27 or 147 rows): a CTA of 64 pixels would write
  // 7-37 KB and spend its time on the fixed costs (table, fill, barrier). Take whole output
  // columns, as many as fit 40 KB of slab, so the CTA's piece of B is one long contiguous
  // run for the flat write phase.
  if (g.k <= 160) {
    const int64_t hp_full = (g.h_o - 1) * g.s + g.k_h + 2;
    int64_t wt = 0;
    while (wt < g.w_o && wt < 16 && g.c_i * ((wt * g.s) + g.k_w) * (hp_full + 32) * 4 <= 40 * 1024 &&
           (wt + 1) * g.h_o <= 4096)
      ++wt;
    if (wt >= 1) {
      a.HT = (int32_t)g.h_o;
      a.WT = (int32_t)wt;
    }
  }
  a.NHT = (a.h_o + a.HT - 1) / a.HT;
  a.NWT = (a.w_o + a.WT - 1) / a.WT;
  a.HP = (a.HT - 1) * a.s + a.k_h;
  a.WS = (a.WT - 1) * a.s + a.k_w;
  a.HPpad = best_slab_stride(a, a.HP + V - 1, V, (int)std::min<int64_t>(g.k, 4096));
  const int64_t per_c = (int64_t)a.WS * a.HPpad * 4;
  const int64_t khw = g.k_h * g.k_w;
  // channel block: at most 48 KB of slab and ~640 lowered rows (5 chunks per lane in
  // registers); whole c_i when that fits, else a multiple of 4 channels (every block's
  // first lowered row then stays 16-byte aligned)
  int64_t cb = std::min<int64_t>({g.c_i, (48 * 1024) / per_c, std::max<int64_t>(640 / khw, 4)});
  if (cb < g.c_i) cb = cb / 4 * 4;
  if (cb < 1) return false;
  a.CB = (int32_t)cb;
  a.NCB = (int32_t)((g.c_i + cb - 1) / cb);
  a.RB = (int32_t)(cb * khw);
  const int64_t rows_last = ldb - (int64_t)(a.NCB - 1) * a.RB;
  const int64_t table_rows = std::max<int64_t>(a.RB, rows_last);
  const size_t smem = (size_t)((cb * per_c + 15) / 16 * 16) + (size_t)((table_rows + 3) / 4 * 4) * 4;
  const int64_t blocks = g.b * a.NHT * a.NWT * a.NCB;
  if (smem > 200 * 1024 || blocks > 0x7fffffffLL) return false;
  int ncl = (int)((table_rows / 4 + 31) / 32);  // chunks per lane
  {
    const int64_t nch = ldb / 4;
    // < 75% of the lanes busy in the chunk-per-lane loop, and a contiguous pixel run
    a.flat = a.NCB == 1 && (a.WT == 1 || a.HT == a.h_o) && nch * 4 < (int64_t)ncl * 32 * 3 ? 1 : 0;
    uint32_t lh = 0;
    while ((1ull << lh) < (uint64_t)a.h_o) ++lh;
    a.ho_p = 31 + lh;
    a.ho_m = (uint32_t)(((1ull << a.ho_p) + a.h_o - 1) / a.h_o);
    uint32_t l = 0;
    while ((1ull << l) < (uint64_t)nch) ++l;
    a.nch_p = 31 + l;
    a.nch_m = (uint32_t)(((1ull << a.nch_p) + nch - 1) / nch);
  }
  if (ncl == 7) ncl = 8;
  if (ncl > 8) ncl = 0;
  *err = V == 2 ? launch_slab_v<2>(ncl, (unsigned)blocks, smem, I, B, a, st)
                : launch_slab_v<1>(ncl, (unsigned)blocks, smem, I, B, a, st);
  count_launch();
  return true;
}

cudaError_t launch_im2col(const float* I, float* B, int64_t ldb, const ConvGeom& g, cudaStream_t st) {
  const bool vec = (ldb % 4 == 0) && (reinterpret_cast<uintptr_t>(B) % 16 == 0);
  cudaError_t err = cudaSuccess;
  if (vec && launch_im2col_slab(I, B, ldb, g, st, &err)) return err;
  Im2colArgs a;
  a.k_h = (int32_t)g.k_h; a.k_w = (int32_t)g.k_w; a.c_i = (int32_t)g.c_i; a.h_i = (int32_t)g.h_i;
  a.w_i = (int32_t)g.w_i; a.s = (int32_t)g.s; a.p = (int32_t)g.p; a.h_o = (int32_t)g.h_o; a.w_o = (int32_t)g.w_o;
  a.K = (int32_t)g.k; a.n = g.n; a.ldb = ldb; a.plane = g.h_i * g.w_i;
  const int64_t total = ((ldb + 3) / 4) * g.n;
  const int64_t blocks = std::min<int64_t>((total + 255) / 256, 148 * 16);
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
