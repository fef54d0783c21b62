// shifted_conv.cu -- V2: "shifted window" tcgen05 implicit GEMM for stride-1 convolutions.
//
// The reference materialises (explicit path, im2col.hpp:77-120) or packs on the fly
// (fused path, pack_b_im2col im2col.hpp:177-262) k_h*k_w shifted copies of every
// input element. On B200 the copies are unnecessary: index output pixels in the
// *padded* plane, m' = i_h + H_q*(i_w + W_q*i_b) with H_q = h_i + p, W_q = w_i + p at
// stride 1 -- neighbouring columns and images share their zero padding (plane_period) --
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
#include <map>
#include <mutex>
#include <cstdlib>
#include <cstdio>

#include "internal.h"

// Profiling stage switches (CGB_DEBUG_SW, tools/ only): compiled out of the product.
#ifdef CGB_PROFILING
#define CGB_DBG(bit) ((a.dbg & (bit)) != 0)
#else
#define CGB_DBG(bit) (false)
#endif

namespace cgb {
namespace sw {

constexpr int BK = 32;
#ifndef CGB_SW_PWARPS
#define CGB_SW_PWARPS 12
#endif
constexpr int PRODUCER_WARPS = CGB_SW_PWARPS;

// Warp roles: producers, the window forwarder (CTA pairs: one thread turns the local
// "window staged" barrier into one cluster-scope arrive on the leader's barrier per
// chunk), the filter TMA warp, the MMA issuer, 4 epilogue warps. The sub-partition
// (warp % 4) of the TMA/MMA/epilogue warps follows from this order; 12 producers plus
// the forwarder measured best on B200 (same-box A/B, tools/cmp_libs.sh).
constexpr int FWD_WARP = PRODUCER_WARPS;
constexpr int TMA_WARP = PRODUCER_WARPS + 1;
constexpr int MMA_WARP = TMA_WARP + 1;
constexpr int EPI_WARP0 = TMA_WARP + 2;  // 4 consecutive warps cover the 4 TMEM lane quadrants
constexpr int THREADS = (EPI_WARP0 + 4) * 32;

struct Args {
  int32_t k_n, k_h, k_w, c_i, h_i, w_i, p, h_o, w_o, b;
  int32_t s;          // stride: the window is split into s*s phase planes (polyphase)
  int32_t nph_h, nph_w, NPH;  // phases used: min(s, k_h) x min(s, k_w)
  int32_t R_pad;      // staged rows per phase rounded to 8 (phase stride in a slot = R_pad*128 B)
  int32_t Hq, Wq;     // padded plane
  int32_t dmax;       // (k_h-1) + Hq*(k_w-1)
  int32_t R;          // staged rows per chunk = MT*128 + dmax
  int32_t CC;         // channel chunks
  int32_t taps;
  int32_t m_tiles, n_tiles;
  int64_t Mp;         // padded output rows Hq*Wq*b
  int32_t Mp32;       // same, 32-bit (shifted_supported guarantees < 2^31 - tile)
  int64_t plane;      // h_i*w_i
  // Work split (see seg_get): the channel-chunk units of tiles [0, sk_units / CC) in one
  // contiguous, balanced range per group (stream-K), then dp_tiles whole tiles
  // round-robin over the `groups` CTAs (pairs: clusters).
  int32_t dp_tiles, sk_units, groups;
  // Tail tiles: m-tiles [m_full, m_tiles) have tail_mt (< MT) subtiles, so the last round
  // of a layer whose row count leaves it half empty is cut into smaller tiles that fill
  // all groups (0 = every m-tile has MT subtiles).
  int32_t m_full, tail_mt;
  int* counters;      // [sk tile][ranks*4 epilogue warps][2] pieces arrived / written; zero between launches
  float* sk_ws;       // partial tiles of split pieces: [sk tile][rank][sk_pieces][MT*128 x BN]
  int32_t sk_pieces;  // most pieces any split tile has
  // Split-K (layers with fewer tiles than half the groups, e.g. 7x7 512->512 at b=16):
  // the stream-K split of every tile into S equal pieces (S divides CC, groups = tiles*S,
  // one piece per group); each piece writes its partial tile to sk_ws slot (tile, rank,
  // piece) and splitk_reduce_kernel sums the S slots in order into O. No CTA waits for
  // another. 0/1 = off.
  int32_t splitk;
  int32_t vec;        // O rows take 32-byte vector stores (k_n % 8 == 0, O 32-byte aligned)
  int32_t ksteps;     // K=8 MMA steps per tap and chunk (4; fewer in the w-im2col mode)
  int32_t tps;        // taps per filter stage group (divides B_STAGES; see the filter TMA warp)
  int32_t urot;       // rotate the window unit -> staging warp assignment from chunk to chunk
  int32_t b_res;      // filters resident: CC*taps <= B_STAGES and one filter tile, so stage cc*taps+tap is
                      // loaded once per CTA and never recycled (no per-tile filter hand-overs)
  int32_t pstore;     // epilogue stores: 1 lane pairs 64 B (default), 0 per-lane 32 B (CGB_SW_PSTORE=0)
  int32_t tma_a;      // 1x1 layers: A (pixels x channels) TMA'd MN-major straight from I, no staging
  int32_t wim;        // w-im2col mode: a row holds the k_w*c_i values of one output row's w-taps
  int32_t wim_kw, wim_ci;  // the real k_w and c_i in that mode (k_w = 1 and c_i = 32 above)
  int32_t wim_off[32];     // w-im2col element j = c + c_i*kw: c*plane + kw*h_i (constant bank, uniform)
  int32_t wim_dw[32];      //   and its kw (a large negative value past k_w*c_i)
  // n / (Hq*Wq) and n / Hq as a multiply-shift (n < 2^31): the producers' per-row
  // padded-plane decomposition without integer-division sequences
  uint32_t fd_hwq_m, fd_hwq_p, fd_hq_m, fd_hq_p;
  // h-strips (wide stride-1 images): each image is cut into `strips` virtual images of strip_h
  // output rows with the unshared period Hq = strip_h + k_h - 1, so a tile's halo is two strip
  // columns instead of two image columns. strips = 1: off (strip_h = h_o).
  int32_t strips, strip_h;
  uint32_t fd_st_m, fd_st_p;
  unsigned long long* stats;  // per-CTA cycle counters when dbg & 64 (profiling only)
  int32_t dbg;        // profiling switches (CGB_DEBUG_SW): 1 = producers skip loads, 2 = skip MMAs,
                      //   4 = skip epilogue stores, 8 = skip filter TMA
};

// floor(n / d) for 0 <= n < 2^31 with m = ceil(2^p / d), p = 31 + ceil(log2 d): the
// error n*(m - 2^p/d)/2^p < 1/d never crosses an integer (m fits 32 bits for every d).
CGB_DEV int32_t fast_div(int32_t n, uint32_t m, uint32_t p) {
  return (int32_t)(((uint64_t)(uint32_t)n * m) >> p);
}
inline void fast_div_magic(uint32_t d, uint32_t& m, uint32_t& p) {
  uint32_t l = 0;
  while ((1ull << l) < d) ++l;
  p = 31 + l;
  m = (uint32_t)(((1ull << p) + d - 1) / d);
}

// Segment sequence of one group: first the pieces of its stream-K unit range
// [sk_begin(gid), sk_begin(gid+1)) over tiles [0, sk_tiles), cut at tile boundaries;
// then its whole (data-parallel) tiles sk_tiles + gid, + G, ... Split pieces come first
// so every group ends on plain whole-tile stores (a final split piece would leave the
// wait-for-the-other-piece and its red.adds exposed at the end of the kernel). Every
// role walks the same sequence; the state is just the segment index j (registers are
// the binding resource of this kernel).
CGB_DEV int64_t sk_begin(const Args& a, int g) { return (int64_t)g * a.sk_units / a.groups; }
// The per-group constants of the sequence, computed once per role (seg_init): the per-tile
// step (seg_at) is then free of integer divisions -- with one short chunk per tile (the
// w-im2col layers: ~1 us of UMMAs) the two 64-bit and four 32-bit divisions of a
// from-scratch lookup were ~1500 cycles per tile on the MMA issuing thread's critical path.
struct Seg {
  int ub, ue;      // this group's stream-K unit range
  int t0;          // first split tile (ub / CC)
  int npieces;     // pieces of split tiles
  int ndp;         // whole tiles
  int tbase;       // first whole tile of group 0 (sk_units / CC)
};
CGB_DEV Seg seg_init(const Args& a, int gid) {
  Seg s;
  s.ub = (int)sk_begin(a, gid);
  s.ue = (int)sk_begin(a, gid + 1);
  s.t0 = s.ub / a.CC;
  s.npieces = s.ue > s.ub ? (s.ue - 1) / a.CC - s.t0 + 1 : 0;
  s.ndp = gid < a.dp_tiles ? (a.dp_tiles - gid + a.groups - 1) / a.groups : 0;
  s.tbase = a.sk_units / a.CC;
  return s;
}
CGB_DEV bool seg_at(const Args& a, const Seg& s, int gid, int j, int& tile, int& cc0, int& cc1) {
  if (j < s.npieces) {
    const int t0 = s.t0 + j;
    const int us = j == 0 ? s.ub : t0 * a.CC;
    tile = t0;
    cc0 = us - t0 * a.CC;
    cc1 = min(a.CC, s.ue - t0 * a.CC);
    return true;
  }
  j -= s.npieces;
  if (j < s.ndp) {
    tile = s.tbase + gid + j * a.groups;
    cc0 = 0;
    cc1 = a.CC;
    return true;
  }
  return false;
}
CGB_DEV bool seg_get(const Args& a, int gid, int j, int& tile, int& cc0, int& cc1) {
  return seg_at(a, seg_init(a, gid), gid, j, tile, cc0, cc1);
}
// group whose stream-K range holds unit x
CGB_DEV int sk_group_of(const Args& a, int x) {
  int c = (int)((int64_t)x * a.groups / a.sk_units);
  while (c + 1 < a.groups && sk_begin(a, c + 1) <= x) ++c;
  return c;
}

// One w-im2col row for a compile-time (k_w, c_i): element j = c + CI*kw, the w bound
// checked once per kw and the offsets folded into immediates; zero past KW*CI.
template <int KW, int CI>
CGB_DEV void wim_row(const Args& a, const float* src, int32_t w0, float (&v)[32]) {
  const int32_t plane = (int32_t)a.plane;
#pragma unroll
  for (int kw = 0; kw < KW; ++kw) {
    const bool ok = (unsigned)(w0 + kw) < (unsigned)a.w_i;
    const float* p = src + kw * a.h_i;
#pragma unroll
    for (int c = 0; c < CI; ++c) v[c + CI * kw] = ok ? ldg_stream(p + c * plane) : 0.0f;
  }
#pragma unroll
  for (int j = KW * CI; j < 32; ++j) v[j] = 0.0f;
}

// First padded row of this CTA's part of a tile and its subtile count (MT, or tail_mt for
// the tail m-tiles); pair tiles stack rank 0's and rank 1's rows.
template <int MT, bool PAIR>
CGB_DEV void tile_rows(const Args& a, int tile, uint32_t rank, int32_t& m0, int& mtc) {
  constexpr int P = PAIR ? 2 : 1;
  const int32_t mi = a.n_tiles == 1 ? tile : tile % a.m_tiles;
  if (a.tail_mt && mi >= a.m_full) {
    mtc = a.tail_mt;
    m0 = a.m_full * (P * MT * 128) + (mi - a.m_full) * (P * a.tail_mt * 128) + (int32_t)rank * a.tail_mt * 128;
  } else {
    mtc = MT;
    m0 = mi * (P * MT * 128) + (int32_t)rank * (MT * 128);
  }
}

template <int MT, int BN, bool SPLIT, int A_SLOTS, int B_STAGES, bool PAIR = false>
struct Cfg {
  static constexpr int NS = SPLIT ? 2 : 1;
  static constexpr int NB = PAIR ? BN / 2 : BN;  // filters staged in this CTA (half per CTA for a pair)
  static constexpr int B_TILE = NB * BK * 4;
  static constexpr int ACC_COLS = MT * BN;  // per accumulator set
  static constexpr int TMEM_COLS = 2 * ACC_COLS <= 512 ? 2 * ACC_COLS : ACC_COLS;
  static constexpr int ACC_SETS = 2 * ACC_COLS <= 512 ? 2 : 1;
  static constexpr int UMMA_N = BN > 256 ? 256 : BN;
  static_assert(BN % 64 == 0, "epilogue works in 64-column blocks");
};

// The UMMAs of one tap: K = 4 k-steps of 8 x (BN / UMMA_N) N halves x MT M subtiles
// (3 per product for 3xTF32: lo*hi + hi*lo + hi*hi). Fully unrolled with compile-time
// descriptor offsets and no branches: the single issuing thread must keep up with N = 64
// UMMAs (~43 cycles each), so its per-UMMA instruction count matters (tools/pair_bench.cu).
// Descriptor units are 16 bytes: A m-subtile 128 rows = 1024, A k-step a_kstep (K-major
// window: 2; MN-major TMA-fed tile: 64), B k-step 8 rows of 128 B = 64, B 32-filter block
// 4096 B = 256.
template <int MT, int BN, bool SPLIT, bool PAIR, int KS>
CGB_DEV void issue_tap(uint32_t d_base, uint64_t at, uint64_t at_lo, uint64_t bt, uint64_t bt_lo, uint32_t idesc,
                       uint32_t a_kstep, uint32_t first) {
  constexpr int UN = BN > 256 ? 256 : BN;
#pragma unroll
  for (int kk = 0; kk < KS; ++kk)
#pragma unroll
    for (int hf = 0; hf < BN / UN; ++hf)
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) {
        const uint64_t ad = at + (uint64_t)(mt * 1024) + (uint64_t)kk * a_kstep;
        const uint64_t bd = bt + (uint64_t)(hf * ((PAIR ? UN / 2 : UN) / 32) * 256 + kk * 64);
        const uint32_t d = d_base + (uint32_t)(mt * BN + hf * UN);
        const uint32_t acc = kk == 0 ? first : 1u;
        if (SPLIT) {
          const uint64_t ad_lo = at_lo + (uint64_t)(mt * 1024) + (uint64_t)kk * a_kstep;
          const uint64_t bd_lo = bt_lo + (uint64_t)(hf * ((PAIR ? UN / 2 : UN) / 32) * 256 + kk * 64);
          if (PAIR) {
            mma_tf32_2cta(d, ad_lo, bd, idesc, acc);
            mma_tf32_2cta(d, ad, bd_lo, idesc, 1);
            mma_tf32_2cta(d, ad, bd, idesc, 1);
          } else {
            mma_tf32(d, ad_lo, bd, idesc, acc);
            mma_tf32(d, ad, bd_lo, idesc, 1);
            mma_tf32(d, ad, bd, idesc, 1);
          }
        } else {
          if (PAIR) mma_tf32_2cta(d, ad, bd, idesc, acc);
          else mma_tf32(d, ad, bd, idesc, acc);
        }
      }
}

// Tail tiles (mtc < MT subtiles) and w-im2col rows (ks < 4 k-steps): runtime bounds.
template <int MT, int BN, bool SPLIT, bool PAIR>
CGB_DEV void issue_tap_partial(uint32_t d_base, uint64_t at, uint64_t at_lo, uint64_t bt, uint64_t bt_lo,
                               uint32_t idesc, uint32_t a_kstep, uint32_t first, int mtc, int ks) {
  constexpr int UN = BN > 256 ? 256 : BN;
#pragma unroll 1
  for (int kk = 0; kk < ks; ++kk)
#pragma unroll
    for (int hf = 0; hf < BN / UN; ++hf)
#pragma unroll 1
      for (int mt = 0; mt < mtc; ++mt) {
        const uint64_t ad = at + (uint64_t)(mt * 1024) + (uint64_t)kk * a_kstep;
        const uint64_t bd = bt + (uint64_t)(hf * ((PAIR ? UN / 2 : UN) / 32) * 256 + kk * 64);
        const uint32_t d = d_base + (uint32_t)(mt * BN + hf * UN);
        const uint32_t acc = kk == 0 ? first : 1u;
        if (SPLIT) {
          const uint64_t ad_lo = at_lo + (uint64_t)(mt * 1024) + (uint64_t)kk * a_kstep;
          const uint64_t bd_lo = bt_lo + (uint64_t)(hf * ((PAIR ? UN / 2 : UN) / 32) * 256 + kk * 64);
          if (PAIR) {
            mma_tf32_2cta(d, ad_lo, bd, idesc, acc);
            mma_tf32_2cta(d, ad, bd_lo, idesc, 1);
            mma_tf32_2cta(d, ad, bd, idesc, 1);
          } else {
            mma_tf32(d, ad_lo, bd, idesc, acc);
            mma_tf32(d, ad, bd_lo, idesc, 1);
            mma_tf32(d, ad, bd, idesc, 1);
          }
        } else {
          if (PAIR) mma_tf32_2cta(d, ad, bd, idesc, acc);
          else mma_tf32(d, ad, bd, idesc, acc);
        }
      }
}

// Epilogue of one accumulator set: TMEM -> registers -> O for the units u = u0, u0 + du,
// ... of the tile's (M subtile, 32-column block) pairs, for the 32 rows of TMEM lane
// quadrant `sub` (the calling warp's warp % 4).
// MODE 0: store into O (add: red.add instead -- the second of two stream-K pieces);
// 1: write this piece's partial to its workspace slot (ws_own: [unit][sub][lane][32]
// floats, each lane one 128-byte run); 2: the last piece to arrive: O = p_0 + p_1 + ...
// in piece order (own registers at position prank, the others from the workspace slots
// ws_all + r * piece_stride), then store. Compile-time modes keep the common loop lean.
template <int BN, int MODE>
CGB_DEV void store_units(const Args& a, float* __restrict__ O, uint32_t trow0, int32_t m0, int n0, int mtc, int sub,
                         int lane, int u0, int du, bool add = false, float* ws_own = nullptr,
                         const float* ws_all = nullptr, size_t piece_stride = 0, int npieces = 1, int prank = 0) {
  constexpr int NCB = BN / 32;
  const int32_t hw_q = a.Hq * a.Wq;
#pragma unroll 1
  for (int u = u0; u < mtc * NCB && !CGB_DBG(16); u += du) {
    const int mt = u / NCB, cb = u - mt * NCB;
    const int32_t Q = m0 + mt * 128 + sub * 32 + lane;
    int64_t P = -1;
    if (Q < a.Mp32) {
      const int32_t bb = fast_div(Q, a.fd_hwq_m, a.fd_hwq_p);
      const int32_t rem = Q - bb * hw_q;
      const int32_t wq = fast_div(rem, a.fd_hq_m, a.fd_hq_p), hq = rem - wq * a.Hq;
      if (a.strips > 1) {
        const int32_t bi = fast_div(bb, a.fd_st_m, a.fd_st_p), h0 = (bb - bi * a.strips) * a.strip_h;
        if (hq < a.strip_h && h0 + hq < a.h_o && wq < a.w_o) P = (int64_t)(h0 + hq + a.h_o * (wq + a.w_o * bi));
      } else if (hq < a.h_o && wq < a.w_o) {
        P = (int64_t)(hq + a.h_o * (wq + a.w_o * bb));
      }
    }
    const uint32_t trow = trow0 + mt * BN;
    uint32_t r[32];
    tmem_ld_32x32b_x32(trow + cb * 32, r);
    tmem_ld_wait();
    const size_t run = ((size_t)(u * 4 + sub) * 32 + lane) * 32;  // this lane's 32 floats in a piece slot
    if (MODE == 1) {
#pragma unroll
      for (int j = 0; j < 32; j += 8) st_global_v8(ws_own + run + j, &r[j]);
      continue;
    }
    if (MODE == 2) {
      // four columns at a time (registers: the kernel runs at its launch bound)
#pragma unroll
      for (int j = 0; j < 32; j += 4) {
        float acc[4], v[4];
        const float own[4] = {__uint_as_float(r[j]), __uint_as_float(r[j + 1]), __uint_as_float(r[j + 2]),
                              __uint_as_float(r[j + 3])};
#pragma unroll 1
        for (int q = 0; q < npieces; ++q) {
          if (q == prank) {
#pragma unroll
            for (int i = 0; i < 4; ++i) v[i] = own[i];
          } else {
            ld_global_cg_v4(ws_all + (size_t)q * piece_stride + run + j, v);
          }
#pragma unroll
          for (int i = 0; i < 4; ++i) acc[i] = q == 0 ? v[i] : acc[i] + v[i];
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) r[j + i] = __float_as_uint(acc[i]);
      }
    }
    const int nb = n0 + cb * 32;
    if (a.pstore && a.vec && nb + 32 <= a.k_n && !CGB_DBG(4)) {
      // Lane pairs write whole 64-byte runs: in store A_k the pair writes segments
      // 2k, 2k+1 (8 floats each) of the even lane's pixel, in B_k those of the odd
      // lane's pixel, after one shfl.xor exchange. Each warp store then touches 16
      // lines with 64 bytes each instead of 32 lines with 32 bytes: half the L1->L2
      // write requests, which bound the epilogue (~1 request per clock per SM).
      // (Lane quads writing whole 128-byte lines after a 4x4 shuffle transpose
      // measured slower: the extra shuffles and selects cost more than they save.)
      const int par = lane & 1;
      const int64_t PA = __shfl_sync(0xffffffffu, P, lane & ~1), PB = __shfl_sync(0xffffffffu, P, lane | 1);
      float* dA = O + PA * a.k_n + nb + 8 * par;
      float* dB = O + PB * a.k_n + nb + 8 * par;
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        uint32_t x[8], v[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = __shfl_xor_sync(0xffffffffu, par ? r[16 * k + i] : r[16 * k + 8 + i], 1);
#pragma unroll
        for (int i = 0; i < 8; ++i) v[i] = par ? x[i] : r[16 * k + i];
        if (PA >= 0) {
          if (!add) st_global_v8(dA + 16 * k, v);
          else {  // second stream-K piece: the pair's 16-byte reds share 128-byte lines too
            red_add_v4(dA + 16 * k, v);
            red_add_v4(dA + 16 * k + 4, v + 4);
          }
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) v[i] = par ? r[16 * k + 8 + i] : x[i];
        if (PB >= 0) {
          if (!add) st_global_v8(dB + 16 * k, v);
          else {
            red_add_v4(dB + 16 * k, v);
            red_add_v4(dB + 16 * k + 4, v + 4);
          }
        }
      }
    } else if (P >= 0 && !CGB_DBG(4)) {
      float* dst = O + P * a.k_n + nb;
      if (a.vec && nb + 32 <= a.k_n) {
        if (!add) {
#pragma unroll
          for (int j = 0; j < 32; j += 8) st_global_v8(dst + j, &r[j]);
        } else {
#pragma unroll
          for (int j = 0; j < 32; j += 4) red_add_v4(dst + j, &r[j]);
        }
      } else {
#pragma unroll
        for (int j = 0; j < 32; ++j)
          if (nb + j < a.k_n) {
            if (!add) dst[j] = __uint_as_float(r[j]);
            else atomicAdd(dst + j, __uint_as_float(r[j]));
          }
      }
    }
  }
}

// Split-K: O = slot_0 + slot_1 + ... + slot_{S-1} for every output of every tile (the
// fixed order makes the result independent of which piece finished first). Slot layout
// per (tile, CTA rank): [unit = (subtile, 32-column block)][TMEM quadrant][lane][32],
// as store_units writes it; one thread per 4 consecutive columns of one row.
template <int MT, int BN, bool PAIR>
__global__ void __launch_bounds__(256) splitk_reduce_kernel(float* __restrict__ O, Args a) {
  griddep_wait();  // the partial tiles of the previous grid (launched with PDL)
  constexpr int NCB = BN / 32, P = PAIR ? 2 : 1;
  const int64_t piece = (int64_t)MT * 128 * BN;
  const int64_t per_tile = (int64_t)P * piece / 4;  // float4 items per tile (both ranks)
  const int64_t total = (int64_t)a.m_tiles * a.n_tiles * per_tile;
  const int32_t hw_q = a.Hq * a.Wq;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int tile = (int)(idx / per_tile);
    int64_t r = idx - (int64_t)tile * per_tile;
    const int rank = (int)(r / (piece / 4));
    r -= (int64_t)rank * (piece / 4);
    const int j4 = (int)(r & 7);  // float4 within the lane's 32-float run
    const int64_t run = r >> 3;   // (unit, sub, lane)
    const int lane = (int)(run & 31), sub = (int)((run >> 5) & 3), u = (int)(run >> 7);
    const int mt = u / NCB, cb = u - mt * NCB;
    int32_t m0;
    int mtc;
    tile_rows<MT, PAIR>(a, tile, (uint32_t)rank, m0, mtc);
    if (mt >= mtc) continue;
    const int32_t Q = m0 + mt * 128 + sub * 32 + lane;
    if (Q >= a.Mp32) continue;
    const int32_t bb = fast_div(Q, a.fd_hwq_m, a.fd_hwq_p);
    const int32_t rem = Q - bb * hw_q;
    const int32_t wq = fast_div(rem, a.fd_hq_m, a.fd_hq_p), hq = rem - wq * a.Hq;
    int64_t Pix;
    if (a.strips > 1) {
      const int32_t bi = fast_div(bb, a.fd_st_m, a.fd_st_p), h0 = (bb - bi * a.strips) * a.strip_h;
      if (hq >= a.strip_h || h0 + hq >= a.h_o || wq >= a.w_o) continue;
      Pix = (int64_t)(h0 + hq + a.h_o * (wq + a.w_o * bi));
    } else {
      if (hq >= a.h_o || wq >= a.w_o) continue;
      Pix = (int64_t)(hq + a.h_o * (wq + a.w_o * bb));
    }
    const int col = (tile / a.m_tiles) * BN + cb * 32 + 4 * j4;
    const float* src = a.sk_ws + ((int64_t)tile * P + rank) * a.splitk * piece + run * 32 + 4 * j4;
    float4 acc = *reinterpret_cast<const float4*>(src);
    for (int sp = 1; sp < a.splitk; ++sp) {
      const float4 v = *reinterpret_cast<const float4*>(src + sp * piece);
      acc.x += v.x;
      acc.y += v.y;
      acc.z += v.z;
      acc.w += v.w;
    }
    float* dst = O + Pix * a.k_n + col;
    if (a.vec && col + 4 <= a.k_n) {
      *reinterpret_cast<float4*>(dst) = acc;
    } else {
      const float v4[4] = {acc.x, acc.y, acc.z, acc.w};
      for (int e = 0; e < 4; ++e)
        if (col + e < a.k_n) dst[e] = v4[e];
    }
  }
}

// PAIR = true: launched as clusters of 2 CTAs (a TPC); the leader (rank 0) issues
// tcgen05.mma.cta_group::2 with M = 256 -- A rows 0-127 from the leader's window, 128-255
// from the peer's window at the same shared-memory offset, B split into two halves of
// BN/2 filters (one per CTA), accumulators in both CTAs' TMEM. Per SM this halves the
// filter-tile TMA traffic, the B operand reads and the B staging footprint.
// UPI: window units each producer warp keeps in flight (loads of UPI units issued before
// any of them is stored). 2 for the staging-bound configurations, else 1 (registers).
template <int MT, int BN, bool SPLIT, int A_SLOTS, int B_STAGES, bool PAIR, int UPI>
__global__ void __launch_bounds__(THREADS, 1)
    sw_conv_kernel(const __grid_constant__ CUtensorMap tmap_hi, const __grid_constant__ CUtensorMap tmap_lo,
                   const float* __restrict__ I, float* __restrict__ O, Args a, uint32_t a_slot_bytes) {
  using C = Cfg<MT, BN, SPLIT, A_SLOTS, B_STAGES, PAIR>;
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
  uint64_t* a_ready = t_empty + 2;  // [A_SLOTS] this CTA's producers done (CTA pairs)
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(a_ready + A_SLOTS);
  uint32_t* tap_shift = tmem_holder + 1;  // [taps], filled by the MMA warp

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  if (CGB_DBG(64) && threadIdx.x == 0) {
    a.stats[blockIdx.x * 16 + 8] = gtimer();
    a.stats[blockIdx.x * 16 + 14] = smid();
  }
  // Tiles: m_tiles x n_tiles units of (MT*128 rows [x2 for a pair], BN filters); a CTA
  // (or CTA pair) walks them round-robin. For a pair, this CTA owns rows
  // [m0 + rank*MT*128, +MT*128) of the pair tile and filters [n0 + rank*BN/2, +BN/2) of B.
  const uint32_t rank = PAIR ? cluster_ctarank() : 0;
  const int gid = PAIR ? (int)cluster_id_x() : (int)blockIdx.x;  // work group (CTA or CTA pair)

  if (warp == TMA_WARP) {
    if (lane == 0) {
      for (int s = 0; s < A_SLOTS; ++s) {
        // pairs: one forwarded arrive per CTA; TMA-fed A: the loader's expect_tx arrive
        mbar_init(&a_full[s], a.tma_a ? 1 : (PAIR ? 2 : PRODUCER_WARPS));
        mbar_init(&a_ready[s], PRODUCER_WARPS);
        mbar_init(&a_empty[s], 1);
      }
      for (int s = 0; s < B_STAGES; ++s) {
        // TMA-skipping profile mode: both ranks arrive, so neither runs phases ahead
        mbar_init(&b_full[s], (PAIR && CGB_DBG(8)) ? 2 : 1);
        mbar_init(&b_empty[s], 1);
      }
      for (int s = 0; s < 2; ++s) {
        mbar_init(&t_full[s], 1);
        mbar_init(&t_empty[s], 4 * (PAIR ? 2 : 1));
      }
      fence_mbar_init();
      tma_prefetch_desc(&tmap_hi);
      if (SPLIT) tma_prefetch_desc(&tmap_lo);
    }
    __syncwarp();
  }
  if (PAIR) cluster_sync();  // peer barriers initialised before any remote arrive
  if (warp == TMA_WARP) {
    if (PAIR) tmem_alloc2(tmem_holder, C::TMEM_COLS);
    else tmem_alloc(tmem_holder, C::TMEM_COLS);
  }
  tc_fence_before();
  if (PAIR) cluster_sync();
  else __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;
  // Everything above is private to this CTA (barriers, TMEM, the tensor-map parameter);
  // global memory is touched only after the previous grid in the stream has finished.
  griddep_wait();
  if (threadIdx.x == 0) griddep_launch_dependents();
  // cluster addresses of the leader's barriers (arrivals from both CTAs land there)
  const uint32_t lead_a_full = PAIR ? mapa_shared(a_full, 0) : smem_u32(a_full);
  const uint32_t lead_b_full = PAIR ? mapa_shared(b_full, 0) : smem_u32(b_full);
  const uint32_t lead_t_empty = PAIR ? mapa_shared(t_empty, 0) : smem_u32(t_empty);

  if (warp < PRODUCER_WARPS) {
    // ---------------------------------------------------------------- window producers
    // A unit = 32/nph_h consecutive padded rows of each of the nph_h h-phases of one
    // w-phase: lane l stages row j(l) = l%8 + 8*(l/(8*nph_h)) of h-phase a(l) = (l/8)%nph_h.
    // For stride 2 the 32 lanes of a warp then read 32 consecutive input rows h (both
    // parities) -> one 128-byte line per channel; every 8-lane group stores 8 consecutive
    // rows of one phase -> conflict-free 16-byte shared stores under the 128B swizzle.
    const int rows_per_unit = 32 / a.nph_h;
    int32_t Rt = a.R;  // staged rows of the current tile (fewer for tail tiles)
    int row_blocks = (Rt + rows_per_unit - 1) / rows_per_unit;
    int units = a.nph_w * row_blocks;
    auto set_tile_rows = [&](int mtc) {
      Rt = mtc * 128 + a.dmax;
      row_blocks = (Rt + rows_per_unit - 1) / rows_per_unit;
      units = a.nph_w * row_blocks;
    };
    const int32_t hw_q = a.Hq * a.Wq;
    const int32_t plane = (int32_t)a.plane;
    const int lane_row = (lane & 7) + 8 * (lane / (8 * a.nph_h));
    const int lane_pha = (lane >> 3) % a.nph_h;
    const uint32_t slot_stride = (uint32_t)a.R_pad * 128;
    int it = 0;  // chunk counter across tiles (slot ring position)
    auto row_src = [&](int32_t row, int32_t ph_a, int32_t ph_c, int32_t m0, int cc, bool& ok) -> const float* {
      const int32_t Q = m0 + row;
      ok = row < Rt && Q < a.Mp32;
      if (!ok) return I;
      const int32_t bb = fast_div(Q, a.fd_hwq_m, a.fd_hwq_p);
      const int32_t rem = Q - bb * hw_q;
      const int32_t wq = fast_div(rem, a.fd_hq_m, a.fd_hq_p), hq = rem - wq * a.Hq;
      int32_t bi = bb, h0 = 0;
      if (a.strips > 1) {  // virtual image bb = (image bi, strip): rows continue into the neighbouring strips
        bi = fast_div(bb, a.fd_st_m, a.fd_st_p);
        h0 = (bb - bi * a.strips) * a.strip_h;
      }
      const int32_t h = a.s * (h0 + hq) + ph_a - a.p, w = a.s * wq + ph_c - a.p;
      ok = (unsigned)h < (unsigned)a.h_i && (unsigned)w < (unsigned)a.w_i;
      return I + ((int64_t)bi * a.c_i + (int64_t)cc * BK) * a.plane + (w * a.h_i + h);
    };
    auto load_rows = [&](const float* src, bool ok, int cmax, float (&v)[BK]) {
      if (cmax >= BK) {
#pragma unroll
        for (int c = 0; c < BK; ++c) v[c] = ok ? ldg_stream(src + c * plane) : 0.0f;
      } else {
#pragma unroll
        for (int c = 0; c < BK; ++c) v[c] = (ok && c < cmax) ? ldg_stream(src + c * plane) : 0.0f;
      }
    };
    auto store_rows = [&](int32_t row, const float (&v)[BK], uint32_t dst_hi, uint32_t dst_lo) {
      if (row >= Rt) return;
#pragma unroll
      for (int ch = 0; ch < 8; ++ch) {
        const uint32_t off = row * 128 + ((ch ^ (row & 7)) << 4);
        if (SPLIT) {
          // 3xTF32 split with round-to-nearest on both halves (like the filters, K5):
          // hi = rna(x) leaves |lo| <= 2^-12 |x|, and rounding lo to TF32 here (the tensor
          // core would truncate it) bounds the split error at 2^-24 |x| instead of the
          // 2^-22 |x| of a truncated split (VGG/ResNet sweeps: max error vs conv_direct
          // under the reference's 1e-5 normalised bar, bench.cpp:57-66).
          const float h0 = to_tf32(v[4 * ch + 0]), h1 = to_tf32(v[4 * ch + 1]);
          const float h2 = to_tf32(v[4 * ch + 2]), h3 = to_tf32(v[4 * ch + 3]);
          st_shared_v4(dst_hi + off, h0, h1, h2, h3);
          st_shared_v4(dst_lo + off, to_tf32(v[4 * ch] - h0), to_tf32(v[4 * ch + 1] - h1), to_tf32(v[4 * ch + 2] - h2),
                       to_tf32(v[4 * ch + 3] - h3));
        } else {
          st_shared_v4(dst_hi + off, v[4 * ch], v[4 * ch + 1], v[4 * ch + 2], v[4 * ch + 3]);
        }
      }
    };
    int tile, cc0, cc1;
    if (a.tma_a) {
      // A arrives by TMA (filter warp): nothing to stage
    } else if (a.wim) {
      // ---- w-im2col rows (low-channel layers): row (h-phase pha, hq, wo, image) holds
      // I(s*hq + pha - p, s*wo + kw - p, c) at element j = c + c_i*kw (zero past k_w*c_i and
      // in the padding); only the k_h taps are row shifts. One chunk per tile.
      const Seg sg1 = seg_init(a, gid);
      for (int j = 0; seg_at(a, sg1, gid, j, tile, cc0, cc1); ++j) {
        int32_t m0;
        int mtc;
        tile_rows<MT, PAIR>(a, tile, rank, m0, mtc);
        set_tile_rows(mtc);
        for (int cc = cc0; cc < cc1; ++cc, ++it) {
          const int s = it % A_SLOTS;
          const uint32_t ph = (it / A_SLOTS) & 1;
          const uint32_t base_hi = smem_u32(a_slot(s, 0));
          const uint32_t base_lo = smem_u32(a_slot(s, SPLIT ? 1 : 0));
          // one chunk per tile here: the slot hand-over chain (commit -> producers ->
          // forwarder -> MMA) is on the critical path, so the waits spin (a suspended
          // try_wait wakes up late)
          if (lane == 0) mbar_wait_spin(&a_empty[s], ph ^ 1);
          __syncwarp();
          // One unit in flight per iteration: a second one (the regular loop's UPI = 2)
          // raised the register pressure of the two-unit kernels for every layer.
          constexpr int WU = 1;
          for (int u = warp; u < units && !CGB_DBG(1); u += WU * PRODUCER_WARPS) {
            float v[WU][BK];
            int32_t row[WU];
#pragma unroll
            for (int q = 0; q < WU; ++q) {
              row[q] = (u + q * PRODUCER_WARPS) * rows_per_unit + lane_row;
              const int32_t Q = m0 + row[q];
              const float* src = I;
              int32_t w0 = -(1 << 20);
              if (u + q * PRODUCER_WARPS < units && row[q] < Rt && Q < a.Mp32) {
                const int32_t bb = fast_div(Q, a.fd_hwq_m, a.fd_hwq_p);
                const int32_t rem = Q - bb * hw_q;
                const int32_t wo = fast_div(rem, a.fd_hq_m, a.fd_hq_p), hq = rem - wo * a.Hq;
                const int32_t h = a.s * hq + lane_pha - a.p;
                if ((unsigned)h < (unsigned)a.h_i) {
                  w0 = a.s * wo - a.p;
                  src = I + (int64_t)bb * a.wim_ci * a.plane + (int64_t)w0 * a.h_i + h;
                }
              }
              if (BN == 64 && a.wim_kw == 7 && a.wim_ci == 3) {
                wim_row<7, 3>(a, src, w0, v[q]);  // the 7x7 stem: bound checks once per kw
              } else if (BN == 64 && a.wim_kw == 3 && a.wim_ci == 3) {
                wim_row<3, 3>(a, src, w0, v[q]);  // VGG conv1
              } else {
#pragma unroll
                for (int e = 0; e < BK; ++e) {
                  // elements past ksteps*8 are never read by the MMAs: no loads for them
                  const int32_t w = w0 + a.wim_dw[e];
                  v[q][e] = (e < a.ksteps * 8 && (unsigned)w < (unsigned)a.w_i) ? ldg_stream(src + a.wim_off[e]) : 0.0f;
                }
              }
            }
#pragma unroll
            for (int q = 0; q < WU; ++q)
              if (u + q * PRODUCER_WARPS < units)
                store_rows(row[q], v[q], base_hi + (uint32_t)lane_pha * slot_stride,
                           base_lo + (uint32_t)lane_pha * slot_stride);
          }
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) mbar_arrive(PAIR ? &a_ready[s] : &a_full[s]);
        }
      }
    } else {
    // (from-scratch lookup here: these producers are the register-tightest path, and their
    // tiles carry whole chunks of staging work)
    int urot = 0;  // rotation of the unit -> warp assignment (units staged so far, mod the warps)
    for (int j = 0; seg_get(a, gid, j, tile, cc0, cc1); ++j) {
      int32_t m0;
      int mtc;
      tile_rows<MT, PAIR>(a, tile, rank, m0, mtc);
      set_tile_rows(mtc);
      for (int cc = cc0; cc < cc1; ++cc, ++it) {
        const int s = it % A_SLOTS;
        const uint32_t ph = (it / A_SLOTS) & 1;
        // WAR on this CTA's own window: completion of the reading UMMAs is all that is
        // needed, so a CTA-scope wait (a cluster-scope acquire compiles to an L1 flush).
        // The first unit's loads are issued before the wait, so their latency overlaps it.
        bool slot_free = false;
        const uint32_t base_hi = smem_u32(a_slot(s, 0));
        const uint32_t base_lo = smem_u32(a_slot(s, SPLIT ? 1 : 0));
        const int cmax = a.c_i - cc * BK;
        // UPI units in flight per iteration (UPI x 32 loads per thread). The unit -> warp
        // assignment rotates from chunk to chunk (unit u of this chunk goes to warp
        // (u + rot) % 12): with 18 or 20 units per chunk the same warps would otherwise
        // always carry the extra unit, and with fewer units than warps (1x1 layers: 4 or
        // 8 rows blocks per chunk) the same warps would always idle while the deep A ring
        // lets different warps fill different chunks at once.
        const int ufirst = a.urot ? (warp + PRODUCER_WARPS - urot) % PRODUCER_WARPS : warp;
        if (a.urot) urot = (urot + units) % PRODUCER_WARPS;
        for (int u = ufirst; u < units && !CGB_DBG(1); u += UPI * PRODUCER_WARPS) {
          float v[UPI][BK];
          int32_t row[UPI];
          uint32_t off[UPI];
          const float* src[UPI];
          bool ok[UPI];
#pragma unroll
          for (int q = 0; q < UPI; ++q) {
            const int uq = u + q * PRODUCER_WARPS;
            // phase column: nph_w <= 2 (stride <= 2), so a compare instead of a division
            const int pc = uq >= row_blocks ? 1 : 0, rb = uq - pc * row_blocks;
            row[q] = rb * rows_per_unit + lane_row;
            off[q] = (uint32_t)(lane_pha + a.nph_h * pc) * slot_stride;
            src[q] = row_src(row[q], lane_pha, pc, m0, cc, ok[q]);
            ok[q] = ok[q] && uq < units;
          }
#pragma unroll
          for (int q = 0; q < UPI; ++q) load_rows(src[q], ok[q], cmax, v[q]);
          if (!slot_free) {
            mbar_wait(&a_empty[s], ph ^ 1);
            slot_free = true;
          }
#pragma unroll
          for (int q = 0; q < UPI; ++q)
            if (q == 0 || u + q * PRODUCER_WARPS < units) store_rows(row[q], v[q], base_hi + off[q], base_lo + off[q]);
        }
        if (!slot_free) mbar_wait(&a_empty[s], ph ^ 1);  // no unit this chunk: still in phase order
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(PAIR ? &a_ready[s] : &a_full[s]);  // CTA scope: cheap (no GPU-wide fence)
        }
      }
    }
    }
    if (CGB_DBG(64) && warp == 0 && lane == 0) a.stats[blockIdx.x * 16 + 13] = gtimer();
  } else if (warp == FWD_WARP) {
    // ---------------------------------------------------------------- window forwarder
    // A cluster-scope release arrive costs a GPU-wide memory barrier; paying it once per
    // chunk here keeps it off the producer warps (the bottleneck of staging-bound layers).
    if (PAIR && lane == 0 && !a.tma_a) {
      int it = 0, tile, cc0, cc1;
      const Seg sg3 = seg_init(a, gid);
      for (int j = 0; seg_at(a, sg3, gid, j, tile, cc0, cc1); ++j)
        for (int cc = cc0; cc < cc1; ++cc, ++it) {
          const int s = it % A_SLOTS;
          if (a.wim) mbar_wait_spin(&a_ready[s], (it / A_SLOTS) & 1);
          else mbar_wait(&a_ready[s], (it / A_SLOTS) & 1);
          mbar_arrive_cluster(lead_a_full + s * 8);
        }
    }
  } else if (warp == TMA_WARP) {
    // ---------------------------------------------------------------- filter TMA
    if (elect_one()) {
      constexpr uint32_t bytes = C::NS * C::B_TILE * (PAIR ? 2 : 1);  // both halves signal the leader
      const int G = a.tps, NG = B_STAGES / a.tps;  // taps per filter stage group, groups in the ring
      int bs = 0, gq = 0, gb = 0;                    // ring slot, position in its group, group
      uint32_t gph = 0;
      // group complete: the leader's arrive (G > 1: after the group's expect_tx; TMA-less
      // profiling mode: both CTAs arrive)
      auto close_group = [&](int g) {
        if (CGB_DBG(8)) {
          if (PAIR) mbar_arrive_cluster(lead_b_full + g * 8);
          else mbar_arrive(&b_full[g]);
        } else if (G > 1 && rank == 0) {
          mbar_arrive(&b_full[g]);
        }
      };
      const uint32_t b0_hi = smem_u32(b_slot(0, 0)), b0_lo = smem_u32(b_slot(0, SPLIT ? 1 : 0));
      // Filter column of this CTA's j-th 32-filter block. A pair UMMA of N = UMMA_N takes
      // UMMA_N / 2 filters from each CTA, so for BN > 256 (two UMMAs per k-step) the CTA's
      // blocks interleave the two N halves: accumulator column c stays filter n0 + c.
      constexpr int HB = (PAIR ? C::UMMA_N / 2 : C::UMMA_N) / 32;  // blocks per UMMA half in this CTA
      auto fcol = [&](int nt0, int j) {
        return nt0 + (j / HB) * C::UMMA_N + (PAIR ? (int)rank * (C::UMMA_N / 2) : 0) + 32 * (j % HB);
      };
      int tile, cc0, cc1;
      if (a.b_res) {
        // resident filters: every (chunk, tap) stage once, each on its own barrier (phase 0)
        const int n0 = 0;
        for (int cc = 0; cc < a.CC; ++cc)
          for (int tap = 0; tap < a.taps; ++tap) {
            const int st_i = cc * a.taps + tap;
            if (rank == 0) mbar_arrive_expect_tx(&b_full[st_i], bytes);
            const uint32_t stage_off = (uint32_t)st_i * C::NS * C::B_TILE;
#pragma unroll
            for (int j = 0; j < C::NB / 32; ++j) {
              if (PAIR) {
                tma_load_3d_2sm(b0_hi + stage_off + j * 4096, &tmap_hi, lead_b_full + st_i * 8, fcol(n0, j), tap, cc * BK);
                if (SPLIT)
                  tma_load_3d_2sm(b0_lo + stage_off + j * 4096, &tmap_lo, lead_b_full + st_i * 8, fcol(n0, j), tap,
                                  cc * BK);
              } else {
                tma_load_3d(b0_hi + stage_off + j * 4096, &tmap_hi, &b_full[st_i], fcol(n0, j), tap, cc * BK);
                if (SPLIT) tma_load_3d(b0_lo + stage_off + j * 4096, &tmap_lo, &b_full[st_i], fcol(n0, j), tap, cc * BK);
              }
            }
          }
      }
      int ait = 0;  // TMA-fed A: chunk counter (window slot ring)
      const Seg sg4 = seg_init(a, gid);
      for (int j = 0; seg_at(a, sg4, gid, j, tile, cc0, cc1); ++j) {
        const int n0 = (tile / a.m_tiles) * BN;
        int32_t am0 = 0;
        int amtc = 0;
        if (a.tma_a) tile_rows<MT, PAIR>(a, tile, rank, am0, amtc);
        for (int cc = cc0; cc < cc1; ++cc) {
          if (a.tma_a) {
            // 1x1 layers: the A tile is MT x 4 boxes of 32 pixels x 32 channels, MN-major
            // SW128 (32-byte atoms) like the filter tiles; rows past an image's hw (padded
            // to 32) and past the batch are zero-filled by the TMA unit.
            const int s = ait % A_SLOTS;
            mbar_wait(&a_empty[s], ((ait / A_SLOTS) & 1) ^ 1);
            if (rank == 0) mbar_arrive_expect_tx(&a_full[s], (uint32_t)amtc * 16384u * (PAIR ? 2u : 1u));
            const uint32_t dst0 = smem_u32(a_slot(s, 0));
            for (int q = 0; q < amtc * 4; ++q) {
              const int32_t Q = am0 + q * 32;
              const int32_t bb = fast_div(Q, a.fd_hwq_m, a.fd_hwq_p);
              const int32_t px = Q - bb * a.Hq;
              if (PAIR) tma_load_3d_2sm(dst0 + q * 4096, &tmap_lo, lead_a_full + s * 8, px, cc * BK, bb);
              else tma_load_3d(dst0 + q * 4096, &tmap_lo, &a_full[s], px, cc * BK, bb);
            }
            ++ait;
          }
          for (int tap = 0; tap < a.taps && !a.b_res; ++tap) {
            // WAR on own smem: CTA scope suffices. A suspending try_wait, not a spin: the
            // ring is deep enough to hide the wake-up, and the spinning thread took issue
            // slots from the producer warps of its sub-partition (BN = 256 layers 0.5-1%).
            // Filter stages are handed over in groups of G taps (one wait, one arrive, one
            // commit per group): a hand-over costs the pair ~270-340 cycles
            // (tools/pair_bench.cu), more than one tap of UMMAs for MT = 1, BN <= 128.
            if (gq == 0) mbar_wait(&b_empty[gb], gph ^ 1);
            if (!CGB_DBG(8)) {
              if (rank == 0) {
                if (G == 1) mbar_arrive_expect_tx(&b_full[gb], bytes);
                else mbar_expect_tx(&b_full[gb], bytes);
              }
              const uint32_t stage_off = (uint32_t)bs * C::NS * C::B_TILE;
#pragma unroll
              for (int j = 0; j < C::NB / 32; ++j) {
                if (PAIR) {
                  tma_load_3d_2sm(b0_hi + stage_off + j * 4096, &tmap_hi, lead_b_full + gb * 8, fcol(n0, j), tap,
                                  cc * BK);
                  if (SPLIT)
                    tma_load_3d_2sm(b0_lo + stage_off + j * 4096, &tmap_lo, lead_b_full + gb * 8, fcol(n0, j), tap,
                                    cc * BK);
                } else {
                  tma_load_3d(b0_hi + stage_off + j * 4096, &tmap_hi, &b_full[gb], fcol(n0, j), tap, cc * BK);
                  if (SPLIT) tma_load_3d(b0_lo + stage_off + j * 4096, &tmap_lo, &b_full[gb], fcol(n0, j), tap, cc * BK);
                }
              }
            }
            if (gq == G - 1) close_group(gb);
            if (++bs == B_STAGES) bs = 0;
            if (++gq == G) {
              gq = 0;
              if (++gb == NG) { gb = 0; gph ^= 1; }
            }
          }
        }
      }
      if (gq != 0 && !a.b_res) close_group(gb);  // a last, partial group
    }
  } else if (warp == MMA_WARP) {
    // ---------------------------------------------------------------- MMA issue
    // Per-tap A-descriptor offsets (phase plane + row shift, in 16-byte units) are
    // tabulated once so the single issuing thread does no integer division: its
    // scalar work between UMMA batches is exposed as tensor-pipe idle time.
    for (int t = lane; t < a.taps; t += 32) {
      const int kh = t % a.k_h, kw = t / a.k_h;
      const int phase = (kh % a.s) + a.nph_h * (kw % a.s);
      tap_shift[t] = (uint32_t)((phase * a.R_pad + kh / a.s + a.Hq * (kw / a.s)) * 8);
    }
    __syncwarp();
    constexpr uint32_t idesc_k = idesc_tf32(C::UMMA_N, false, true, PAIR ? 256 : 128);
    constexpr uint32_t idesc_mn = idesc_tf32(C::UMMA_N, true, true, PAIR ? 256 : 128);
    const uint32_t idesc = a.tma_a ? idesc_mn : idesc_k;  // TMA-fed A is MN-major
    if (rank == 0 && elect_one()) {
      // Descriptors are built once per operand slot; per UMMA only the 14-bit start
      // address field moves (row shift d*128 B = d*8 units, k-step 32 B = 2 units,
      // m-subtile 128 rows = 1024 units, B k-step 1024 B = 64 units, 32-filter block
      // 4096 B = 256 units), so each issue is an add on a uniform register.
      int as = 0, bs = 0, t = 0;
      uint32_t aph = 0;
      const int G = a.tps, NG = B_STAGES / a.tps;  // filter stage groups (see the TMA warp)
      int gq = 0, gb = 0;
      uint32_t gph = 0;
      unsigned long long w_t = 0, w_a = 0, w_b = 0, t_start = clock64();
      if (CGB_DBG(64)) a.stats[blockIdx.x * 16 + 9] = gtimer();
      const bool st = CGB_DBG(64);
      // K-major window (128-byte rows, k-step 32 B = 2 units) or, TMA-fed, MN-major 32-pixel
      // blocks like the filter tiles (k-step = 8 channel rows of 128 B = 64 units)
      const uint64_t a_desc0 = a.tma_a ? smem_desc(smem_u32(a_slot(0, 0)), 4096, 512, 0, kLayoutSW128_32B)
                                       : smem_desc(smem_u32(a_slot(0, 0)), 16, 1024);
      const uint32_t a_kstep = a.tma_a ? 64u : 2u;
      const uint64_t a_lo_off = SPLIT ? (uint64_t)(a_slot_bytes >> 4) : 0;  // lo window follows hi
      const uint64_t a_slot_units = (uint64_t)(C::NS * a_slot_bytes) >> 4;
      const uint64_t b_desc0 = smem_desc(smem_u32(b_slot(0, 0)), 4096, 512, 0, kLayoutSW128_32B);
      constexpr uint64_t b_lo_off = SPLIT ? (uint64_t)(C::B_TILE >> 4) : 0;
      constexpr uint64_t b_stage_units = (uint64_t)(C::NS * C::B_TILE) >> 4;
      const bool full_steps = a.ksteps == BK / 8;  // every k-step issued (all but w-im2col rows)
      int tile, cc0, cc1;
      if (a.b_res) {  // resident filters: all stages land once (phase 0), then no filter waits at all
        for (int i = 0; i < a.CC * a.taps; ++i) mbar_wait_spin(&b_full[i], 0);
        tc_fence_after();
      }
      const Seg sg5 = seg_init(a, gid);
      for (; seg_at(a, sg5, gid, t, tile, cc0, cc1); ++t) {
        const int acc_set = C::ACC_SETS == 2 ? (t & 1) : 0;
        const uint32_t acc_ph = C::ACC_SETS == 2 ? ((t >> 1) & 1) : (t & 1);
        int32_t m0u;
        int mtc;
        tile_rows<MT, PAIR>(a, tile, 0, m0u, mtc);
        unsigned long long c0 = st ? clock64() : 0;
        if (PAIR) mbar_wait_spin_cl(&t_empty[acc_set], acc_ph ^ 1);
        else mbar_wait_spin(&t_empty[acc_set], acc_ph ^ 1);
        if (st) w_t += clock64() - c0;
        tc_fence_after();
        const uint32_t d_base = tmem_base + acc_set * C::ACC_COLS;
        for (int cc = cc0; cc < cc1; ++cc) {
          unsigned long long c1 = st ? clock64() : 0;
          if (PAIR) mbar_wait_spin_cl(&a_full[as], aph);
          else mbar_wait_spin(&a_full[as], aph);
          if (st) w_a += clock64() - c1;
          tc_fence_after();
          const uint64_t a_hi0 = a_desc0 + (uint64_t)as * a_slot_units;
          uint32_t shift_next = tap_shift[0];
          for (int tap = 0; tap < a.taps; ++tap) {
            const uint64_t shift = shift_next;
            if (tap + 1 < a.taps) shift_next = tap_shift[tap + 1];
            unsigned long long c2 = st ? clock64() : 0;
            // TMA completion bytes of both halves land on this (leader's) barrier; the
            // UMMA reads the data through the async proxy, so a CTA-scope wait suffices.
            if (a.b_res) {
              bs = cc * a.taps + tap;  // loaded once, waited for before the first tile
            } else if (gq == 0) {
              mbar_wait_spin(&b_full[gb], gph);
              tc_fence_after();
            }
            if (st) w_b += clock64() - c2;
            const uint64_t at = a_hi0 + shift, at_lo = at + a_lo_off;
            const uint64_t bt = b_desc0 + (uint64_t)bs * b_stage_units, bt_lo = bt + b_lo_off;
            const uint32_t first = (cc == cc0 && tap == 0) ? 0u : 1u;
            if (!CGB_DBG(2)) {
              // tail tiles have MT/2 or MT/4 subtiles: unrolled batches for those too
              constexpr int MT2 = MT >= 2 ? MT / 2 : 1, MT4 = MT >= 4 ? MT / 4 : 1;
              if (full_steps && mtc == MT)
                issue_tap<MT, BN, SPLIT, PAIR, BK / 8>(d_base, at, at_lo, bt, bt_lo, idesc, a_kstep, first);
              else if (full_steps && mtc == MT2)
                issue_tap<MT2, BN, SPLIT, PAIR, BK / 8>(d_base, at, at_lo, bt, bt_lo, idesc, a_kstep, first);
              else if (full_steps && mtc == MT4)
                issue_tap<MT4, BN, SPLIT, PAIR, BK / 8>(d_base, at, at_lo, bt, bt_lo, idesc, a_kstep, first);
              // w-im2col rows (stem: 3 k-steps per tap, VGG conv1: 2): unrolled batches too --
              // with one chunk of 7 or 3 taps per tile the issuing thread is the critical path
              else if (BN == 64 && a.ksteps == 3 && mtc == MT)
                issue_tap<MT, BN, SPLIT, PAIR, 3>(d_base, at, at_lo, bt, bt_lo, idesc, a_kstep, first);
              else if (BN == 64 && a.ksteps == 2 && mtc == MT)
                issue_tap<MT, BN, SPLIT, PAIR, 2>(d_base, at, at_lo, bt, bt_lo, idesc, a_kstep, first);
              else
                issue_tap_partial<MT, BN, SPLIT, PAIR>(d_base, at, at_lo, bt, bt_lo, idesc, a_kstep, first, mtc,
                                                       a.ksteps);
            }
            if (a.b_res) continue;
            if (gq == G - 1) {
              if (PAIR) mma_commit_mc2(&b_empty[gb], 3);
              else mma_commit(&b_empty[gb]);
            }
            if (++bs == B_STAGES) bs = 0;
            if (++gq == G) {
              gq = 0;
              if (++gb == NG) { gb = 0; gph ^= 1; }
            }
          }
          if (PAIR) mma_commit_mc2(&a_empty[as], 3);
          else mma_commit(&a_empty[as]);
          if (++as == A_SLOTS) { as = 0; aph ^= 1; }
        }
        if (PAIR) mma_commit_mc2(&t_full[acc_set], 3);
        else mma_commit(&t_full[acc_set]);
      }
      if (st) {
        unsigned long long* o = a.stats + blockIdx.x * 16;
        o[0] = clock64() - t_start; o[1] = w_t; o[2] = w_a; o[3] = w_b; o[4] = t;
        o[10] = gtimer();
      }
    }
  } else if (warp >= EPI_WARP0) {
    // ---------------------------------------------------------------- epilogue
    const int sub = warp % 4;  // TMEM lane quadrant this warp may access
    unsigned long long epi_wait = 0, epi_busy = 0;
    int t = 0;
    int tile, cc0, cc1;
    const Seg sg6 = seg_init(a, gid);
    for (; seg_at(a, sg6, gid, t, tile, cc0, cc1); ++t) {
      const int acc_set = C::ACC_SETS == 2 ? (t & 1) : 0;
      const uint32_t acc_ph = C::ACC_SETS == 2 ? ((t >> 1) & 1) : (t & 1);
      int32_t m0;
      int mtc;
      tile_rows<MT, PAIR>(a, tile, rank, m0, mtc);
      const int n0 = (tile / a.m_tiles) * BN;
      unsigned long long e0 = CGB_DBG(64) ? clock64() : 0;
      if (PAIR) {
        if (lane == 0) {
          if (a.wim) mbar_wait_spin(&t_full[acc_set], acc_ph);
          else mbar_wait(&t_full[acc_set], acc_ph);
        }
        __syncwarp();
      } else if (a.wim) {  // ~1 us of UMMAs per tile: a suspended try_wait wakes up too late
        if (lane == 0) mbar_wait_spin(&t_full[acc_set], acc_ph);
        __syncwarp();
      } else {
        mbar_wait_warp(&t_full[acc_set], acc_ph);
      }
      unsigned long long e1 = CGB_DBG(64) ? clock64() : 0;
      if (CGB_DBG(64)) epi_wait += e1 - e0;
      tc_fence_after();
      // ---- stream-K piece of a split tile. Groups' unit ranges are contiguous, so every
      // group whose range meets the tile holds exactly one piece of it; pieces are ranked
      // by channel chunk (prank 0 = the highest chunks). No piece ever waits for a piece
      // that has not started: each first arrives on the tile's counters (per CTA rank and
      // epilogue warp) and only ever waits for pieces that arrived before it -- those are
      // resident and running -- so there is no co-residency assumption (concurrent grids,
      // MPS, SM-limited contexts cannot deadlock it), and the sum is bitwise independent
      // of the arrival order:
      // * two pieces (every automatic split: each group holds >= one tile of units): the
      //   first to arrive stores its rows, the second waits for that store and red.adds
      //   its rows (p_0 + p_1 == p_1 + p_0 in fp32);
      // * more pieces (forced splits): all but the last to arrive write their partial
      //   rows to a workspace slot; the last waits for those writes and stores
      //   O = ((p_0 + p_1) + p_2) + ... in piece order.
      // The last piece resets the counters for the next launch.
      const bool whole = cc0 == 0 && cc1 == a.CC;
      const uint32_t trow0 = tmem_base + ((uint32_t)(sub * 32) << 16) + acc_set * C::ACC_COLS;
      // one call site per store mode plus a dedicated one for whole tiles (constant
      // folding keeps the common loop free of the red.add branch); an out-of-line call
      // measured far slower: the call ABI reshapes the whole kernel's register allocation
      bool add = false;  // plain stores, or red.adds for the second of two stream-K pieces
      int mode = 0;
      float* ws_own = nullptr;
      const float* ws_all = nullptr;
      int* cnt = nullptr;
      int npieces = 1, prank = 0;
      bool last = true;
      const size_t piece = (size_t)MT * 128 * BN;
      if (whole) {
        mode = 0;
      } else {
        const int u0 = tile * a.CC;  // stream-K tiles are tiles [0, sk_tiles)
        const int g_hi = sk_group_of(a, u0 + a.CC - 1);
        prank = g_hi - gid;
        npieces = g_hi - sk_group_of(a, u0) + 1;
      }
      if (!whole && a.splitk > 1) {  // split-K partial -> its workspace slot (splitk_reduce_kernel)
        ws_own = a.sk_ws + (((size_t)tile * (PAIR ? 2 : 1) + rank) * a.splitk + prank) * piece;
        mode = 1;
      } else if (!whole) {
        cnt = a.counters + 2 * ((size_t)tile * (PAIR ? 8 : 4) + rank * 4 + sub);
        int order = 0;
        if (lane == 0) order = atomicAdd(cnt, 1);
        order = __shfl_sync(0xffffffffu, order, 0);
        last = order + 1 == npieces;
        if (last && lane == 0) {
          while (ld_acquire_gpu(cnt + 1) < npieces - 1) {  // pieces that arrived earlier
          }
          cnt[0] = 0;  // every other piece has arrived and written: reset for the next launch
          cnt[1] = 0;
        }
        if (last) {
          __syncwarp();
          __threadfence();
        }
        if (npieces == 2) {
          add = last;
        } else {
          float* slots = a.sk_ws + ((size_t)tile * (PAIR ? 2 : 1) + rank) * a.sk_pieces * piece;
          ws_own = slots + prank * piece;
          ws_all = slots;
          mode = last ? 2 : 1;
        }
      }
      if (whole) store_units<BN, 0>(a, O, trow0, m0, n0, mtc, sub, lane, 0, 1, false);  // the common path
      else if (mode == 0) store_units<BN, 0>(a, O, trow0, m0, n0, mtc, sub, lane, 0, 1, add);
      else if (mode == 1) store_units<BN, 1>(a, O, trow0, m0, n0, mtc, sub, lane, 0, 1, false, ws_own);
      else store_units<BN, 2>(a, O, trow0, m0, n0, mtc, sub, lane, 0, 1, false, nullptr, ws_all, piece, npieces, prank);
      if (!whole && a.splitk <= 1 && !last) {
        __threadfence();  // the rows (O or workspace) before the "written" count
        __syncwarp();
        if (lane == 0) atomicAdd(cnt + 1, 1);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        // relaxed: the barrier only hands the drained accumulator set (tcgen05.wait::ld done,
        // tcgen05.fence above) back to the MMA issuer; a release here would first wait for
        // this tile's output stores to become visible GPU-wide
        if (PAIR && CGB_DBG(128)) mbar_arrive_cluster(lead_t_empty + acc_set * 8);  // A/B: the old release arrive
        else if (PAIR) mbar_arrive_cluster_relaxed(lead_t_empty + acc_set * 8);
        else mbar_arrive(&t_empty[acc_set]);
      }
      if (CGB_DBG(64)) epi_busy += clock64() - e1;
    }
    if (CGB_DBG(64) && warp == EPI_WARP0 && lane == 0) {
      a.stats[blockIdx.x * 16 + 5] = epi_wait;
      a.stats[blockIdx.x * 16 + 6] = epi_busy;
      a.stats[blockIdx.x * 16 + 11] = gtimer();
    }
  }
  tc_fence_before();
  if (PAIR) cluster_sync();  // the leader's MMAs write the peer's TMEM: both must be done
  else __syncthreads();
  if (CGB_DBG(64) && threadIdx.x == 0) a.stats[blockIdx.x * 16 + 12] = gtimer();
  if (warp == TMA_WARP) {
    __syncwarp();
    tc_fence_after();
    if (PAIR) tmem_dealloc2(tmem_base, C::TMEM_COLS);
    else tmem_dealloc(tmem_base, C::TMEM_COLS);
  }
}

// ------------------------------------------------------------------ stream-K counters
// Arrival counters of split tiles, one array per (device, stream) so launches that may
// run concurrently never share one. Zeroed once at allocation; every launch leaves them
// zero again (the second piece resets its pair).
constexpr double kSkFill = 0.9;  // split when the last round of whole tiles is < 90% full
struct SkState {
  int* counters = nullptr;  // zero between launches (the last piece of each tile resets its pair)
  size_t n = 0;
  float* ws = nullptr;      // partial tiles
  size_t ws_bytes = 0;
  bool captured = false;    // used while the stream was being captured: never freed implicitly
};
static std::mutex g_sk_mu;
static std::map<std::pair<int, cudaStream_t>, SkState> g_sk;
static std::vector<void*> g_sk_retired;

// Counters (n ints) and partial-tile workspace (ws_bytes) for a stream-K launch on st,
// one set per (device, stream) so launches that may run concurrently never share one.
bool sk_buffers(cudaStream_t st, size_t n, size_t ws_bytes, int** counters, float** ws) {
  std::lock_guard<std::mutex> lk(g_sk_mu);
  int dev = 0;
  cudaGetDevice(&dev);
  SkState& c = g_sk[{dev, st}];
  const bool capturing = !can_free_now(st);
  auto drop = [&](void* p) {
    if (!p) return;
    if (c.captured || capturing) g_sk_retired.push_back(p);  // a captured graph may use it
    else cudaFree(p);
  };
  if (c.n < n) {
    const size_t m = std::max<size_t>(n, 8192);
    drop(c.counters);
    c.counters = nullptr;
    c.n = 0;
    if (capture_safe_malloc(reinterpret_cast<void**>(&c.counters), m * sizeof(int), /*zero=*/true) != cudaSuccess)
      return false;  // no counters: whole tiles only
    c.n = m;
  }
  if (ws_bytes > 0 && c.ws_bytes < ws_bytes) {
    drop(c.ws);
    c.ws = nullptr;
    c.ws_bytes = 0;
    if (capture_safe_malloc(reinterpret_cast<void**>(&c.ws), ws_bytes) != cudaSuccess) return false;
    c.ws_bytes = ws_bytes;
  }
  c.captured = c.captured || capturing;
  *counters = c.counters;
  *ws = c.ws;
  return true;
}

template <int MT, int BN, bool SPLIT, int A_SLOTS, int B_STAGES, bool PAIR, int UPI>
cudaError_t launch_cfg(const CUtensorMap& th, const CUtensorMap& tl, const float* I, float* O, Args a,
                       cudaStream_t st, const Tuning& tu) {
  using C = Cfg<MT, BN, SPLIT, A_SLOTS, B_STAGES, PAIR>;
  a.R = MT * 128 + a.dmax;
  a.R_pad = (a.R + 7) / 8 * 8;
  // Filter stages per hand-over: enough taps that one group's UMMAs (~BN/2 cycles per
  // 128-row UMMA and k-step, x3 for 3xTF32) outlast a hand-over (~400 cycles measured),
  // keeping at least two groups in the ring.
  {
    const int tap_cycles = MT * a.ksteps * (BN / 2) * (SPLIT ? 3 : 1);
    // Long layers (>= 8 rounds of tiles per group, filter tiles >= 128, several taps) run in
    // steady state, where fewer, larger hand-overs win: groups of 3 taps measured 3-9% faster
    // on VGG's 112x112 and 56x56 layers (112x112 128->128 359 -> 336 us, 56x56 128->256
    // 171 -> 155, 256->256 312 -> 289; tools/ab_tune.py), while the ResNet-50 3x3 layers
    // (<= 6 rounds) and VGG's 28x28 / 14x14 layers measured 1-2% slower with them.
    int thr = 400;
    {
      int dev_ = 0, sms_ = 148;
      cudaGetDevice(&dev_);
      cudaDeviceGetAttribute(&sms_, cudaDevAttrMultiProcessorCount, dev_);
      const int64_t rows_ = (int64_t)MT * 128 * (PAIR ? 2 : 1);
      const int64_t tiles_ = (a.Mp + rows_ - 1) / rows_ * ((a.k_n + BN - 1) / BN);
      if (!SPLIT && BN >= 128 && a.taps > 1 && !a.wim && tiles_ >= (int64_t)8 * (PAIR ? sms_ / 2 : sms_)) thr = 1100;
    }
    int g = 1;
    if (tu.tps > 0) {
      g = tu.tps;
    } else {
      while (g * tap_cycles < thr && B_STAGES % (g + 1) == 0 && B_STAGES / (g + 1) >= 2) ++g;
      if (g * tap_cycles < thr)  // the next divisor of the ring (e.g. 3 of 6 after 2 failed)
        for (int h = g + 1; h <= B_STAGES / 2; ++h)
          if (B_STAGES % h == 0) { g = h; break; }
    }
    // TMA-fed A: the filter warp also loads A, one chunk (one tap) at a time, before each
    // chunk's filter tap; closing a group of G chunks needs A slots for all of them while
    // the MMAs still wait for that group: G <= A_SLOTS, or the two rings deadlock.
    if (a.tma_a && g > A_SLOTS) g = A_SLOTS;
    if (g < 1 || B_STAGES % g != 0 || (g > 1 && B_STAGES / g < 2)) g = 1;
    a.tps = g;
  }
  fast_div_magic((uint32_t)(a.Hq * a.Wq), a.fd_hwq_m, a.fd_hwq_p);
  fast_div_magic((uint32_t)a.Hq, a.fd_hq_m, a.fd_hq_p);
  const uint32_t a_slot_bytes = (uint32_t)(a.NPH * a.R_pad * 128);
  const size_t base_smem = (size_t)A_SLOTS * C::NS * a_slot_bytes + (size_t)B_STAGES * C::NS * C::B_TILE + 1024 + 1024;
  if (base_smem > 227 * 1024) return cudaErrorNotSupported;
  constexpr int pair_rows = (PAIR ? 2 : 1) * MT * 128;
  a.m_tiles = (int32_t)((a.Mp + pair_rows - 1) / pair_rows);
  a.n_tiles = (a.k_n + BN - 1) / BN;
  // Filters resident in the ring (no recycling, no per-tile hand-overs): when every
  // (chunk, tap) stage of the one filter tile fits -- the w-im2col layers (stem: 7 taps,
  // VGG conv1: 3), short 1x1 layers.
  {
    // rotation only where a chunk has fewer units than staging warps and one tap (the staged 1x1 layers:
    // 7x7 2048->512 97 -> 80 us, 512->2048 82 -> 73 us); with 18-20 units per chunk (3x3
    // windows) it measured neutral to slightly worse (s2 56->28: 94.7 vs 93.1 us)
    const int rpu = 32 / a.nph_h;
    const int units = a.nph_w * ((a.R + rpu - 1) / rpu);
    a.urot = tu.urot != 0 && units < PRODUCER_WARPS && a.taps == 1;  // (3x3 MT = 1 tiles, 5 units: 1.5% slower)
  }
  a.b_res = tu.b_res != 0 && a.CC * a.taps <= B_STAGES && a.n_tiles == 1 && !(tu.debug & 8);
  size_t smem = base_smem;
  if (tu.smem_pad_kb > 0)  // profiling: shrink the L1 carve-out
    smem = std::max<size_t>(smem, (size_t)tu.smem_pad_kb * 1024);
  auto kern = sw_conv_kernel<MT, BN, SPLIT, A_SLOTS, B_STAGES, PAIR, UPI>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int gmax = PAIR ? sms / 2 : sms;
  // Tail tiles (one filter tile, MT >= 2): when the whole-tile rounds leave a last round
  // that smaller tiles of tail_mt subtiles fill in ONE round, cut it that way (56x56
  // 64->64: 5 rounds of 1024-row pair tiles + 1 round of 512-row tiles instead of 6
  // rounds, the last half empty). Relative tile times as in the dispatcher's cost model.
  a.m_full = 0;
  a.tail_mt = 0;
  const int tail_mode = tu.tail;  // 0 = never, 2 = whenever it fits (tests), default: by cost
  if (a.n_tiles == 1 && MT >= 2 && tail_mode != 0) {
    auto tt = [](int mt) { return mt >= 4 ? 1.8 * mt / 4 : (mt == 2 ? 1.0 : 0.62); };
    const int64_t full_fit = a.Mp / pair_rows;
    const int rounds_full = (int)(full_fit / gmax);
    const int64_t rem = a.Mp - (int64_t)rounds_full * gmax * pair_rows;
    const double t_plain = (double)((a.m_tiles + gmax - 1) / gmax) * tt(MT);
    if (rounds_full >= 1 && rem > 0) {
      for (int tmt = MT / 2; tmt >= 1; tmt /= 2) {
        const int64_t tail_rows = (int64_t)(PAIR ? 2 : 1) * tmt * 128;
        const int64_t n_tail = (rem + tail_rows - 1) / tail_rows;
        if (n_tail > gmax) break;
        // only where stream-K would not take the last round (fill >= kSkFill)
        const double fill0 = (double)a.m_tiles / ((double)((a.m_tiles + gmax - 1) / gmax) * gmax);
        if (tail_mode == 2 || (fill0 >= kSkFill && rounds_full * tt(MT) + tt(tmt) < 0.97 * t_plain)) {
          a.m_full = rounds_full * gmax;
          a.tail_mt = tmt;
          a.m_tiles = (int32_t)(a.m_full + n_tail);
        }
        break;
      }
    }
  }
  const int tiles = a.m_tiles * a.n_tiles;
  // Work split: whole tiles round-robin while the last round is well filled; otherwise
  // the last one-to-two rounds of tiles are split by channel chunk over all groups
  // (stream-K), which needs the arrival counters.
  a.groups = std::min(tiles, gmax);
  a.dp_tiles = tiles;
  a.sk_units = 0;
  a.counters = nullptr;
  a.sk_ws = nullptr;
  a.sk_pieces = 1;
  a.splitk = 0;
  // Split-K when the tiles fill less than half the groups (small batches, e.g. the 7x7
  // and 14x14 layers of a b=16 shard): S pieces of >= 1 channel chunk per tile, partials
  // summed in order by splitk_reduce_kernel (tuning splitk: -1 off, 0 auto, S forced).
  {
    int S = 0;
    if (tu.splitk > 0) S = std::min(tu.splitk, a.CC);
    else if (tu.splitk == 0 && 2 * tiles <= gmax) S = std::min(a.CC, gmax / std::max(tiles, 1));
    while (S >= 2 && a.CC % S != 0) --S;  // equal pieces: one segment per group
    if (S >= 2 && !a.tail_mt && tiles * S <= gmax) {
      const size_t ws_bytes = (size_t)S * tiles * (PAIR ? 2 : 1) * MT * 128 * BN * sizeof(float);
      int* cnt = nullptr;
      float* ws = nullptr;
      if (sk_buffers(st, 0, ws_bytes, &cnt, &ws)) {
        a.splitk = S;
        a.sk_ws = ws;
        a.groups = tiles * S;
        a.dp_tiles = 0;
        a.sk_units = tiles * a.CC;  // the stream-K range split, one piece per group
      }
    }
  }
  const int rounds = (tiles + gmax - 1) / gmax;
  const double fill = (double)tiles / ((double)rounds * gmax);
  const int sk_mode = tu.sk;
  // Stream-K only for the last one-to-two rounds of at least one tile per group: every
  // split piece adds a pass over its rows through the workspace, which measured slower
  // than the idle SMs it saves when ALL tiles would be split (1-round layers: 7x7,
  // 14x14). The fixup itself handles any number of pieces per tile (sk_mode 2 forces it).
  // 1x1 layers (one tap) never gain: a split tile's second piece re-walks output rows the
  // layer is already bound by (14x14 1024->256 b=256: 74.7 us split, 64.6 us as two whole-tile
  // rounds; 256x1x1x64 on 27x56: 58 vs 48 us), so in TF32 mode only sk_mode 2 or 3 splits them
  // (3xTF32 1x1 layers are MMA-bound and keep the split: C3 3xTF32 650 us with, 725 us without).
  const bool sk_ok = !a.tail_mt && (sk_mode == 2 ? (int64_t)tiles * a.CC >= 2 * gmax : tiles >= gmax && (a.taps > 1 || SPLIT || sk_mode == 3));
  if (!a.splitk && sk_mode != 0 && a.CC >= 2 && sk_ok && (fill < kSkFill || sk_mode == 2)) {
    const int dp = std::max(0, tiles / gmax - 1) * gmax;
    const int sk_tiles = tiles - dp;
    const int units = sk_tiles * a.CC;
    auto begin = [&](int g) { return (int)((int64_t)g * units / gmax); };
    auto group_of = [&](int x) {
      int c = (int)((int64_t)x * gmax / units);
      while (c + 1 < gmax && begin(c + 1) <= x) ++c;
      return c;
    };
    int pieces = 1;
    for (int t = 0; t < sk_tiles; ++t)
      pieces = std::max(pieces, group_of(t * a.CC + a.CC - 1) - group_of(t * a.CC) + 1);
    // partial-tile workspace: only splits into more than two pieces use it
    const size_t ws_bytes = pieces > 2 ? (size_t)sk_tiles * (PAIR ? 2 : 1) * pieces * MT * 128 * BN * sizeof(float) : 0;
    int* cnt = nullptr;
    float* ws = nullptr;
    if (sk_buffers(st, (size_t)sk_tiles * (PAIR ? 8 : 4) * 2, ws_bytes, &cnt, &ws)) {
      a.counters = cnt;
      a.sk_ws = ws;
      a.sk_pieces = pieces;
      a.groups = gmax;
      a.dp_tiles = dp;
      a.sk_units = units;
    }
  }
  if (tu.verbose)
    fprintf(stderr,
            "[cgb] launch MT=%d BN=%d split=%d A=%d B=%d pair=%d upi=%d tps=%d smem=%.1fKB tiles=%d (tail %d of mt "
            "%d) sk_units=%d splitk=%d\n",
            MT, BN, (int)SPLIT, A_SLOTS, B_STAGES, (int)PAIR, UPI, a.tps, smem / 1024.0, tiles,
            a.tail_mt ? a.m_tiles - a.m_full : 0, a.tail_mt, a.sk_units, a.splitk);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)((PAIR ? 2 : 1) * a.groups));
  cfg.blockDim = dim3(THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  int na = 0;
  if (PAIR) {
    attr[na].id = cudaLaunchAttributeClusterDimension;
    attr[na].val.clusterDim.x = 2;
    attr[na].val.clusterDim.y = 1;
    attr[na].val.clusterDim.z = 1;
    ++na;
  }
  if (tu.pdl) {  // overlap this launch's setup with the tail of the previous grid
    attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  e = cudaLaunchKernelEx(&cfg, kern, th, tl, I, O, a, a_slot_bytes);
  if (e != cudaSuccess) return e;
  count_launch();
  if (a.splitk > 1) {  // the ordered sum of the partial tiles (PDL: waits for the grid above)
    const int64_t items = (int64_t)tiles * (PAIR ? 2 : 1) * MT * 128 * BN / 4;
    cudaLaunchConfig_t rc = {};
    rc.gridDim = dim3((unsigned)std::max<int64_t>(1, std::min<int64_t>((items + 255) / 256, (int64_t)sms * 8)));
    rc.blockDim = dim3(256);
    rc.stream = st;
    cudaLaunchAttribute ra[1];
    ra[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    ra[0].val.programmaticStreamSerializationAllowed = 1;
    rc.attrs = ra;
    rc.numAttrs = tu.pdl ? 1 : 0;
    if ((e = cudaLaunchKernelEx(&rc, splitk_reduce_kernel<MT, BN, PAIR>, O, a)) != cudaSuccess) return e;
    count_launch();
  }
  return cudaGetLastError();
}

static unsigned long long* g_stats = nullptr;

// Period of the padded plane along one spatial dimension (rows per column / columns per
// image). Phase a of a stride-s dimension holds input n = s*q + a - p at position q;
// output o reads phase a at q = o + kh/s for the taps kh = a (mod s). Consecutive
// columns (images) may SHARE their zero padding: a read past the period wraps into the
// next column's leading zero rows, which is exact as long as (i) every wrapped read lands
// in those zeros (q_max(a) - period < z_lead(a)), (ii) no row that a valid output reads
// holds data beyond the period (period > min(q_last(a), q_max(a))), and (iii) the valid
// outputs fit. For stride 1, k=3, p=1 this is n_i + 1 instead of n_i + 2 (7x7: 64 padded
// rows per image instead of 81); for stride 2 it equals the unshared n_o + 1.
static int32_t plane_period(int64_t n_i, int64_t n_o, int64_t k, int64_t s, int64_t p) {
  int64_t per = n_o;
  for (int64_t a = 0; a < std::min(s, k); ++a) {
    const int64_t z_lead = p > a ? (p - a + s - 1) / s : 0;
    const int64_t q_last = (n_i - 1 + p - a) / s;  // last data row of phase a
    const int64_t q_max = n_o - 1 + (k - 1 - a) / s;  // last row a valid output reads
    per = std::max(per, std::min(q_last, q_max) + 1);
    per = std::max(per, q_max - z_lead + 1);
  }
  return (int32_t)std::min(per, n_o + (k - 1) / s);
}

static Args make_args(const ConvGeom& g) {
  Args a;
  a.k_n = (int32_t)g.k_n; a.k_h = (int32_t)g.k_h; a.k_w = (int32_t)g.k_w; a.c_i = (int32_t)g.c_i;
  a.h_i = (int32_t)g.h_i; a.w_i = (int32_t)g.w_i; a.p = (int32_t)g.p; a.h_o = (int32_t)g.h_o;
  a.w_o = (int32_t)g.w_o; a.b = (int32_t)g.b;
  a.s = (int32_t)g.s;
  a.nph_h = (int32_t)std::min(g.s, g.k_h);
  a.nph_w = (int32_t)std::min(g.s, g.k_w);
  a.NPH = a.nph_h * a.nph_w;
  a.Hq = plane_period(g.h_i, g.h_o, g.k_h, g.s, g.p);
  a.Wq = plane_period(g.w_i, g.w_o, g.k_w, g.s, g.p);
  a.strips = 1;
  a.strip_h = a.h_o;
  {
    // h-strips for wide stride-1 images: 56 output rows per strip above 112 rows, 28 above 56
    // (VGG 224x224 64->64 at b=64: 648 -> 431 us; 150x150: 269 -> 222; 5x5 on 131x131: 378 -> 259;
    // 112x112 64->128 183 -> 175, 128->128 320 -> 314; tools/strip_ab.py). Same UMMAs per output in
    // the same order: bitwise-equal results. tuning strip_h: 0 = this rule, -1 = off, > 0 forced.
    const int knob = tuning().strip_h;
    const int sh = knob > 0 ? knob : (knob < 0 ? 0 : (g.h_o > 112 ? 56 : (g.h_o > 56 ? 28 : 0)));
    if (sh > 0 && g.s == 1 && g.c_i >= 16 && !(g.k_h == 1 && g.k_w == 1) && g.h_o > 2 * sh) {
      const int64_t st = (g.h_o + sh - 1) / sh;
      const int64_t hq = sh + g.k_h - 1;
      if (hq * a.Wq * g.b * st < (int64_t(1) << 30)) {
        a.strips = (int32_t)st;
        a.strip_h = sh;
        a.Hq = (int32_t)hq;
      }
    }
  }
  fast_div_magic((uint32_t)a.strips, a.fd_st_m, a.fd_st_p);
  a.dmax = (a.k_h - 1) / a.s + a.Hq * ((a.k_w - 1) / a.s);
  a.CC = (a.c_i + BK - 1) / BK;
  a.taps = a.k_h * a.k_w;
  a.Mp = (int64_t)a.Hq * a.Wq * g.b * a.strips;
  a.Mp32 = (int32_t)a.Mp;
  a.plane = g.h_i * g.w_i;
  a.R = 0; a.m_tiles = 0; a.n_tiles = 0;
  a.m_full = 0; a.tail_mt = 0;
  a.ksteps = BK / 8;
  a.tps = 1;
  a.pstore = tuning().pstore;
  a.wim = 0; a.wim_kw = 1; a.wim_ci = a.c_i;
  a.tma_a = 0;
  a.dbg = 0;
  a.stats = nullptr;
#ifdef CGB_PROFILING
  a.dbg = tuning().debug;
  if (CGB_DBG(64)) {  // 8 launch slots of 1024 CTAs x 16 counters (slot = launch index % 8)
    if (!g_stats)
      capture_safe_malloc(reinterpret_cast<void**>(&g_stats), 8 * 1024 * 16 * sizeof(unsigned long long), true);
    static int slot = 0;
    a.stats = g_stats + (size_t)(slot++ % 8) * 1024 * 16;
  }
#endif
  return a;
}

}  // namespace sw

// Domain: filters through the tap-major TMA map (k_n % 4 == 0), at least half a channel
// chunk, stride <= 2 (<= 4 phase planes). The padded plane may hold many more rows than
// outputs (unpadded large filters on small images: 5x5 on 7x7 computes 49 rows for 9
// outputs); a cap on that waste (1.7x until round 2) sent such layers to the tap-major
// gather kernel, which measured 2.9-6.8x slower on every one of them, up to a 49x waste
// (tools/waste_ab.py: 512x7x7x64 on 7x7, one output per image, 68 vs 302 us) -- so there
// is no cap by default (tuning waste_pct restores one for A/B).
static double padded_waste(const ConvGeom& g) {
  const double hq = sw::plane_period(g.h_i, g.h_o, g.k_h, g.s, g.p);
  const double wq = sw::plane_period(g.w_i, g.w_o, g.k_w, g.s, g.p);
  return hq * wq / (double)(g.h_o * g.w_o);
}

bool shifted_supported(const ConvGeom& g) {
  if (g.s > 2 || g.k_n % 4 != 0 || g.c_i < 16 || g.k_h * g.k_w > 64) return false;
  if (tuning().waste_pct > 0 && padded_waste(g) * 100.0 > (double)tuning().waste_pct) return false;
  const int64_t hq = sw::plane_period(g.h_i, g.h_o, g.k_h, g.s, g.p);
  const int64_t wq = sw::plane_period(g.w_i, g.w_o, g.k_w, g.s, g.p);
  const int64_t dmax = (g.k_h - 1) / g.s + hq * ((g.k_w - 1) / g.s);
  const int64_t mp = hq * wq * g.b;
  return dmax <= 2048 && mp < (int64_t(1) << 30) && g.c_i * g.h_i * g.w_i * g.b < (int64_t(1) << 31);
}

namespace sw {
// Candidate tile configurations (MT x 128 padded rows, BN filters, 3xTF32, A slots,
// B stages). A config is skipped when its shared memory does not fit
// (launch_cfg -> cudaErrorNotSupported).
struct Cand {
  int mt, bn, split, as, bs, pair, upi;
};
static const Cand kCands[] = {
    // CTA pairs (cta_group::2): B halves per CTA -> deeper filter pipelines
    {4, 64, 0, 2, 8, 1, 1},  {2, 64, 0, 2, 8, 1, 1},  {1, 64, 0, 2, 8, 1, 1},  {2, 64, 1, 1, 6, 1, 1},
    {1, 64, 1, 1, 6, 1, 1},  {2, 128, 0, 2, 6, 1, 1}, {1, 128, 0, 2, 4, 1, 1}, {1, 128, 0, 2, 3, 1, 1},
    {2, 128, 1, 1, 4, 1, 1}, {1, 128, 1, 1, 3, 1, 1}, {2, 256, 0, 2, 4, 1, 1}, {1, 256, 0, 2, 3, 1, 1},
    {1, 256, 0, 2, 2, 1, 1}, {1, 256, 1, 1, 2, 1, 1},
    // single CTA
    {4, 64, 0, 2, 6, 0, 1},  {2, 64, 0, 2, 6, 0, 1},  {1, 64, 0, 2, 6, 0, 1},  {2, 64, 1, 1, 4, 0, 1},
    {1, 64, 1, 1, 4, 0, 1},  {2, 128, 0, 2, 4, 0, 1}, {2, 128, 0, 1, 4, 0, 1}, {1, 128, 0, 2, 4, 0, 1},
    {1, 128, 0, 1, 4, 0, 1}, {2, 128, 1, 1, 3, 0, 1}, {1, 128, 1, 1, 3, 0, 1}, {2, 256, 0, 2, 3, 0, 1},
    {2, 256, 0, 1, 3, 0, 1}, {1, 256, 0, 2, 3, 0, 1}, {1, 256, 0, 2, 2, 0, 1}, {1, 256, 0, 1, 3, 0, 1},
    {1, 256, 1, 1, 2, 0, 1},
    // CTA pairs with one window slot
    {2, 64, 0, 1, 8, 1, 1},  {1, 64, 0, 1, 8, 1, 1},  {2, 128, 0, 1, 4, 1, 1}, {1, 128, 0, 1, 4, 1, 1},
    {1, 256, 0, 1, 3, 1, 1},
    // deep filter rings: only for filter-stream-heavy layers (BN = 256 and >= 2 filter
    // tiles or a stride-1 window, e.g. 7x7/14x14 512->512, 14x14 256->256: 3-9% faster);
    // elsewhere the extra shared memory costs L1 and measured slower (dispatch)
    {1, 256, 0, 2, 9, 1, 1}, {1, 256, 0, 2, 4, 1, 1},
    // two window units in flight per producer warp: staging-bound layers only (BN = 64,
    // or stride 2 with BN <= 128: 56x56 64->64 3% and 56->28 128 8% faster; slower where
    // the MMA or the filter stream binds)
    {4, 64, 0, 2, 8, 1, 2}, {2, 64, 0, 2, 8, 1, 2}, {1, 128, 0, 2, 4, 1, 2}, {2, 128, 0, 2, 6, 1, 2},
    {2, 256, 0, 2, 4, 1, 2},  // 1x1 layers (14x14 1024->256 143 -> 121 us, 7x7 512->2048 124 -> 113 us)
    // 3xTF32 with a double-buffered (hi + lo) window: fits the stride-1 windows
    {2, 64, 1, 2, 4, 1, 1}, {1, 64, 1, 2, 6, 1, 1}, {2, 128, 1, 2, 3, 1, 1}, {1, 128, 1, 2, 4, 1, 1},
    {1, 256, 1, 2, 2, 1, 1},
    // 1x1 layers (TMA-fed A, or staged windows without halo): A rings four chunks deep
    // cover the DRAM latency of the A tiles
    {2, 256, 0, 4, 4, 1, 1}, {2, 128, 0, 4, 6, 1, 1},
    // probes (tuning cfg only)
    {1, 128, 0, 2, 6, 1, 2}, {1, 256, 0, 2, 3, 1, 2}, {1, 256, 0, 2, 4, 1, 2},
    {2, 64, 0, 2, 8, 0, 1},  // single CTA with a ring that holds the stem's 7 taps resident
    // BN = 512 (two N = 256 UMMAs per k-step, all of TMEM for one 128-row subtile per CTA):
    // staging-bound 1x1 layers with k_n >= 512 stage each window once instead of twice
    {1, 512, 0, 4, 4, 1, 1}, {1, 512, 0, 2, 4, 1, 1},
};
constexpr int kNumCands = sizeof(kCands) / sizeof(kCands[0]);
constexpr int kFirstDeepCand = 36;
constexpr int kFirstUpi2Cand = 38;
constexpr int kFirstSplit2Cand = 43;  // 3xTF32 with two window slots
constexpr int kFirstTmaACand = 48;   // deep A rings, tried first for 1x1 layers
constexpr int kFirstProbeCand = 50;  // candidates from here on are CGB_SW_CFG probes only
constexpr int kWimCand = 53;         // the w-im2col layers' single-CTA kernel (dispatch)
constexpr int kBn512Cand = 54;       // staged 1x1 layers with k_n in (256, 512]: one 512-filter tile (dispatch)

static cudaError_t launch_cand(int i, const CUtensorMap& th, const CUtensorMap& tl, const float* I, float* O,
                               const Args& a, cudaStream_t st, const Tuning& tu) {
#define CGB_SW_CASE(IDX, MT, BN, SP, AS, BS, PR, U) \
  case IDX: return launch_cfg<MT, BN, SP, AS, BS, PR, U>(th, tl, I, O, a, st, tu);
  switch (i) {
    CGB_SW_CASE(0, 4, 64, false, 2, 8, true, 1)
    CGB_SW_CASE(1, 2, 64, false, 2, 8, true, 1)
    CGB_SW_CASE(2, 1, 64, false, 2, 8, true, 1)
    CGB_SW_CASE(3, 2, 64, true, 1, 6, true, 1)
    CGB_SW_CASE(4, 1, 64, true, 1, 6, true, 1)
    CGB_SW_CASE(5, 2, 128, false, 2, 6, true, 1)
    CGB_SW_CASE(6, 1, 128, false, 2, 4, true, 1)
    CGB_SW_CASE(7, 1, 128, false, 2, 3, true, 1)
    CGB_SW_CASE(8, 2, 128, true, 1, 4, true, 1)
    CGB_SW_CASE(9, 1, 128, true, 1, 3, true, 1)
    CGB_SW_CASE(10, 2, 256, false, 2, 4, true, 1)
    CGB_SW_CASE(11, 1, 256, false, 2, 3, true, 1)
    CGB_SW_CASE(12, 1, 256, false, 2, 2, true, 1)
    CGB_SW_CASE(13, 1, 256, true, 1, 2, true, 1)
    CGB_SW_CASE(14, 4, 64, false, 2, 6, false, 1)
    CGB_SW_CASE(15, 2, 64, false, 2, 6, false, 1)
    CGB_SW_CASE(16, 1, 64, false, 2, 6, false, 1)
    CGB_SW_CASE(17, 2, 64, true, 1, 4, false, 1)
    CGB_SW_CASE(18, 1, 64, true, 1, 4, false, 1)
    CGB_SW_CASE(19, 2, 128, false, 2, 4, false, 1)
    CGB_SW_CASE(20, 2, 128, false, 1, 4, false, 1)
    CGB_SW_CASE(21, 1, 128, false, 2, 4, false, 1)
    CGB_SW_CASE(22, 1, 128, false, 1, 4, false, 1)
    CGB_SW_CASE(23, 2, 128, true, 1, 3, false, 1)
    CGB_SW_CASE(24, 1, 128, true, 1, 3, false, 1)
    CGB_SW_CASE(25, 2, 256, false, 2, 3, false, 1)
    CGB_SW_CASE(26, 2, 256, false, 1, 3, false, 1)
    CGB_SW_CASE(27, 1, 256, false, 2, 3, false, 1)
    CGB_SW_CASE(28, 1, 256, false, 2, 2, false, 1)
    CGB_SW_CASE(29, 1, 256, false, 1, 3, false, 1)
    CGB_SW_CASE(30, 1, 256, true, 1, 2, false, 1)
    CGB_SW_CASE(31, 2, 64, false, 1, 8, true, 1)
    CGB_SW_CASE(32, 1, 64, false, 1, 8, true, 1)
    CGB_SW_CASE(33, 2, 128, false, 1, 4, true, 1)
    CGB_SW_CASE(34, 1, 128, false, 1, 4, true, 1)
    CGB_SW_CASE(35, 1, 256, false, 1, 3, true, 1)
    CGB_SW_CASE(36, 1, 256, false, 2, 9, true, 1)
    CGB_SW_CASE(37, 1, 256, false, 2, 4, true, 1)
    CGB_SW_CASE(38, 4, 64, false, 2, 8, true, 2)
    CGB_SW_CASE(39, 2, 64, false, 2, 8, true, 2)
    CGB_SW_CASE(40, 1, 128, false, 2, 4, true, 2)
    CGB_SW_CASE(41, 2, 128, false, 2, 6, true, 2)
    CGB_SW_CASE(42, 2, 256, false, 2, 4, true, 2)
    CGB_SW_CASE(43, 2, 64, true, 2, 4, true, 1)
    CGB_SW_CASE(44, 1, 64, true, 2, 6, true, 1)
    CGB_SW_CASE(45, 2, 128, true, 2, 3, true, 1)
    CGB_SW_CASE(46, 1, 128, true, 2, 4, true, 1)
    CGB_SW_CASE(47, 1, 256, true, 2, 2, true, 1)
    CGB_SW_CASE(48, 2, 256, false, 4, 4, true, 1)
    CGB_SW_CASE(49, 2, 128, false, 4, 6, true, 1)
    CGB_SW_CASE(50, 1, 128, false, 2, 6, true, 2)
    CGB_SW_CASE(51, 1, 256, false, 2, 3, true, 2)
    CGB_SW_CASE(52, 1, 256, false, 2, 4, true, 2)
    CGB_SW_CASE(53, 2, 64, false, 2, 8, false, 1)
    CGB_SW_CASE(54, 1, 512, false, 4, 4, true, 1)
    CGB_SW_CASE(55, 1, 512, false, 2, 4, true, 1)
    default: return cudaErrorNotSupported;
  }
#undef CGB_SW_CASE
}

static int bn_for(int k_n) { return k_n <= 64 ? 64 : (k_n <= 128 ? 128 : 256); }

static cudaError_t dispatch(const CUtensorMap& th, const CUtensorMap& tl, const float* I, float* O, const Args& a,
                            bool split, int sms, cudaStream_t st) {
  const Tuning tu = tuning();
  int bn = bn_for(a.k_n);
  if (tu.bn == 64 || tu.bn == 128 || tu.bn == 256 || tu.bn == 512) bn = tu.bn;  // forced filter tile
  const int n_tiles = (a.k_n + bn - 1) / bn;
  if (tu.cfg >= 0) {  // forced candidate (when it matches the filter tile and precision)
    const int i = tu.cfg;
    if (i < kNumCands && kCands[i].bn == bn && kCands[i].split == (int)split)
      return launch_cand(i, th, tl, I, O, a, st, tu);
  }
  // Staged 1x1 layers with 256 < k_n <= 512 and a long contraction (7x7 2048->512): one
  // 512-filter tile stages every window once instead of twice (79.4 -> 71.2 us; not for
  // k_n = 2048, where four 512-tiles per pixel tile measured slower: 81 vs 73 us).
  // Only with at least half a round of 256-row pair tiles: fewer tiles go to split-K, whose
  // piece counts (and rounding) would then depend on the filter tile.
  if (a.taps == 1 && !a.tma_a && !a.wim && !split && a.k_n > 256 && a.k_n <= 512 && a.CC >= 16 && tu.bn == 0 &&
      (a.Mp + 255) / 256 >= sms / 4) {
    cudaError_t e = launch_cand(kBn512Cand, th, tl, I, O, a, st, tu);
    if (e != cudaErrorNotSupported) {
      if (tu.verbose) fprintf(stderr, "[cgb] shifted cand %d (1x1, BN = 512)\n", kBn512Cand);
      return e;
    }
  }
  // w-im2col layers (one chunk of k_h taps per tile: ~1 us of UMMAs between hand-overs):
  // single CTAs -- CTA-scope barriers instead of the pair's cluster-scope hand-overs --
  // with the filters resident in the ring (b_res). Stem: 356 (pair) -> 345 (single CTA,
  // 6 stages) -> 310 us (8 stages, all 7 taps resident); VGG conv1 214 -> 201 us.
  if (a.wim && !split && tu.pair != 2) {
    if (a.taps > 6 && bn == 64) {
      cudaError_t e = launch_cand(kWimCand, th, tl, I, O, a, st, tu);
      if (e != cudaErrorNotSupported) {
        if (tu.verbose) fprintf(stderr, "[cgb] shifted cand %d (w-im2col, single CTA, resident filters)\n", kWimCand);
        return e;
      }
    }
  }
  // Preference (measured, tools/sweep_cfg.sh): CTA pairs first (CGB_SW_PAIR=0 disables),
  // then a double-buffered window (A slots = 2), then the M tile the cost model picks.
  const bool allow_pair = tu.pair != 0 && !(a.wim && !split && tu.pair != 2);
  // passes: pairs with a double-buffered window, pairs with any, single CTAs likewise
  for (int pass = 0; pass < 4; ++pass) {
    const int want_pair = pass < 2 ? 1 : 0;
    if (want_pair && !allow_pair) continue;
    // M tile by a cost model: (rounds of work per group) x (relative time of one tile).
    // Whole tiles cost ceil(tiles / groups) rounds; with stream-K (tiles >= groups, a
    // last round < 90% full, >= 2 channel chunks) the work spreads evenly: tiles / groups.
    // Tile times relative to MT = 2 measured on B200 (bigger M tiles reuse each filter
    // tile over more rows): MT 1 -> 0.62, 2 -> 1, 4 -> 1.8.
    const int units = want_pair ? 2 : 1;
    const int gmax = want_pair ? sms / 2 : sms;
    int mt_max = 1;
    double best = 1e30;
    for (int mt = 4; mt >= 1; mt /= 2) {
      const double tt = mt == 4 ? 1.8 : (mt == 2 ? 1.0 : 0.62);
      const int tiles = (int)((a.Mp + units * mt * 128 - 1) / (units * mt * 128)) * n_tiles;
      const int rounds = (tiles + gmax - 1) / gmax;
      const bool sk = tu.sk != 0 && a.CC >= 2 && tiles >= gmax && (double)tiles / (rounds * gmax) < kSkFill &&
                      (a.taps > 1 || split || tu.sk >= 2);
      // A split that reaches every tile (fewer than two rounds: no whole-tile round ahead of the
      // split ones) costs more than its share of a round -- every group pays a fixup and the
      // filter tile is re-streamed per small tile. With filter tiles <= 128 one round of larger
      // whole tiles measured 10-15% faster (64x3x3x192 on 56x56 b=16: MT 4 whole 39.9 us vs MT 2
      // split 46.1; 32x5x5x192 on 28x14 b=128: 77.9 vs 86.9; tools/fuzz_dispatch.py); with
      // BN = 256 (14x14 256->256) the two measured equal, so the factor applies to BN <= 128 only.
      const double sk_pen = (sk && tiles < 2 * gmax && bn <= 128) ? tu.sk_pen_pct / 100.0 : 1.0;
      const double cost = (sk ? (double)tiles / gmax * 1.03 * sk_pen : (double)rounds) * tt;
      if (cost < best * 0.98) {
        best = cost;
        mt_max = mt;
      }
    }
    if (tu.mt > 0) mt_max = tu.mt;  // forced M tile
    // deep filter rings for the filter-stream-heavy layers: BN = 256 with several filter
    // tiles, or with a stride-1 (small) window that leaves the shared memory for them
    // (14x14 256->256: 62 -> 57 us); stride-2 windows keep the L1 instead
    const bool deep_first = bn == 256 && (n_tiles >= 2 || a.s == 1);
    // staging-bound layers (stride-2 windows with BN <= 128) first try the candidates with
    // two units in flight per producer warp (and the 1x1 layers: one tap per staged row,
    // the most staging-bound of all): s2 56->28 128 87 vs 97 us. Stride-1 BN = 64 layers
    // no longer gain (56x56 64->64: 74.8 vs 73.3 us with one unit, same box, alternated).
    // The w-im2col producer stages one unit per iteration in either kernel; VGG conv1
    // runs equally fast in both (266-270 us), so its old rule (short rows) stays.
    const bool upi2 = a.wim ? a.ksteps <= 2 : ((a.s == 2 && bn <= 128) || (a.taps == 1 && !a.tma_a));
    // try order: 3xTF32 double-buffered windows (split), two-unit producers (upi2), deep
    // filter rings (deep_first), then the regular table; probes never
    int order[kFirstProbeCand];
    int no = 0;
    if (split)
      for (int i = kFirstSplit2Cand; i < kFirstTmaACand; ++i) order[no++] = i;
    // (staged 1x1 windows are as small -- no halo -- and gain too: 7x7 2048->512
    // 121 -> 100 us, 512->2048 96 -> 87 us)
    if ((a.tma_a || (a.taps == 1 && !a.wim)) && !split && tu.tma_deep)
      for (int i = kFirstTmaACand; i < kFirstProbeCand; ++i) order[no++] = i;
    if (upi2)
      for (int i = kFirstUpi2Cand; i < kFirstSplit2Cand; ++i) order[no++] = i;
    if (deep_first)
      for (int i = kFirstDeepCand; i < kFirstUpi2Cand; ++i) order[no++] = i;
    for (int i = 0; i < kFirstDeepCand; ++i) order[no++] = i;
    for (int k = 0; k < no; ++k) {
      const int i = order[k];
      const Cand& c = kCands[i];
      // The deep-A-ring 1x1 candidates (MT = 2) beat the cost model's MT = 1 choice while
      // their tiles fill at least half a round (7x7 2048->512: 100 vs 121 us).
      const bool deep_a = i >= kFirstTmaACand && i < kFirstProbeCand &&
                          (a.Mp + 511) / 512 * n_tiles >= (want_pair ? sms / 2 : sms) / 2;
      if (c.bn != bn || c.split != (int)split || (c.mt > mt_max && !deep_a) || c.pair != want_pair) continue;
      if (pass % 2 == 0 && c.as < 2) continue;
      cudaError_t e = launch_cand(i, th, tl, I, O, a, st, tu);
      if (e != cudaErrorNotSupported) {
        if (tu.verbose)
          fprintf(stderr, "[cgb] shifted cand %d: MT=%d BN=%d split=%d A=%d B=%d pair=%d upi=%d\n", i, c.mt, c.bn,
                  c.split, c.as, c.bs, c.pair, c.upi);
        return e;
      }
    }
  }
  return cudaErrorNotSupported;
}
}  // namespace sw

cudaError_t launch_tc_conv_shifted(const float* f_hi, const float* f_lo, int64_t ldf, const float* I, float* O,
                                   const ConvGeom& g, bool split, cudaStream_t st) {
  (void)ldf;
  sw::Args a = sw::make_args(g);
  a.vec = (g.k_n % 8) == 0 && reinterpret_cast<uintptr_t>(O) % 32 == 0;
  CUtensorMap th, tl;
  cudaError_t e = make_filter_tmap_tapmajor(&th, f_hi, g);
  if (e != cudaSuccess) return e;
  if (split) {
    if ((e = make_filter_tmap_tapmajor(&tl, f_lo, g)) != cudaSuccess) return e;
  } else {
    tl = th;
  }
  // 1x1 stride-1 layers in TF32: A straight from I by TMA (pixels are contiguous per
  // channel plane, i.e. MN-major), no producer staging. Needs 16-byte channel-plane
  // strides (h*w % 4 == 0) and a 16-byte aligned I; rows are the pixels of each image
  // padded to a multiple of 32 (the TMA box), so the plane is (hw32 x 1) per image.
  const int64_t hw = g.h_i * g.w_i;
  if (!split && g.k_h == 1 && g.k_w == 1 && g.s == 1 && g.p == 0 && hw % 4 == 0 &&
      reinterpret_cast<uintptr_t>(I) % 16 == 0 && tuning().tma_a) {
    const int64_t hwp = (hw + 31) / 32 * 32;
    if ((hwp * g.b) < (int64_t(1) << 30) && make_input_tmap_1x1(&tl, I, g) == cudaSuccess) {
      a.tma_a = 1;
      a.Hq = (int32_t)hwp;
      a.Wq = 1;
      a.h_o = (int32_t)hw;
      a.w_o = 1;
      a.dmax = 0;
      a.Mp = hwp * g.b;
      a.Mp32 = (int32_t)a.Mp;
    }
  }
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  return sw::dispatch(th, tl, I, O, a, split, sms, st);
}

bool wim_supported(const ConvGeom& g) {
  if (g.s > 2 || g.k_n % 4 != 0 || g.k_w * g.c_i > 32 || g.k_h > 64) return false;
  const int64_t hq = sw::plane_period(g.h_i, g.h_o, g.k_h, g.s, g.p);
  if ((double)hq / (double)g.h_o > 1.7) return false;
  return hq * g.w_o * g.b < (int64_t(1) << 30) && g.c_i * g.h_i * g.w_i * g.b < (int64_t(1) << 31);
}

// w-im2col mode: the kernel sees a (k_h x 1) convolution over 32 "channels" (one chunk)
// whose window rows the producers build from the k_w*c_i real (kw, c) values; filters
// come from launch_wim_filter_prep as a (k_n, k_h, 32) tap-major array.
cudaError_t launch_tc_conv_wim(const float* f_hi, const float* f_lo, const float* I, float* O, const ConvGeom& g,
                               bool split, cudaStream_t st) {
  sw::Args a = sw::make_args(g);
  a.wim = 1;
  a.wim_kw = (int32_t)g.k_w;
  a.wim_ci = (int32_t)g.c_i;
  a.k_w = 1;
  a.c_i = sw::BK;
  a.CC = 1;
  a.taps = a.k_h;
  a.nph_w = 1;
  a.NPH = a.nph_h;
  a.Wq = a.w_o;
  a.dmax = (a.k_h - 1) / a.s;
  a.Mp = (int64_t)a.Hq * a.Wq * g.b;
  a.Mp32 = (int32_t)a.Mp;
  a.ksteps = (int32_t)((g.k_w * g.c_i + 7) / 8);
  for (int j = 0; j < sw::BK; ++j) {
    const int kw = j / (int)g.c_i, c = j - kw * (int)g.c_i;
    a.wim_off[j] = (int32_t)(c * g.h_i * g.w_i + kw * g.h_i);
    a.wim_dw[j] = kw < g.k_w ? kw : -(1 << 20);
  }
  a.vec = (g.k_n % 8) == 0 && reinterpret_cast<uintptr_t>(O) % 32 == 0;
  ConvGeom gf = g;  // the prepared filters: k_h taps of 32 channels
  gf.k_w = 1;
  gf.c_i = sw::BK;
  CUtensorMap th, tl;
  cudaError_t e = make_filter_tmap_tapmajor(&th, f_hi, gf);
  if (e != cudaSuccess) return e;
  if (split) {
    if ((e = make_filter_tmap_tapmajor(&tl, f_lo, gf)) != cudaSuccess) return e;
  } else {
    tl = th;
  }
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return sw::dispatch(th, tl, I, O, a, split, sms, st);
}

}  // namespace cgb

// Profiling hook (CGB_DEBUG_SW & 64): copies 16 counters per CTA of the last
// shifted-window launch: MMA-thread cycles (total, wait t_empty, wait a_full, wait
// b_full), segments, epilogue wait/busy cycles, then %globaltimer stamps (ns): entry,
// MMA loop start, MMA loop end, epilogue end, exit, producers end; and the SM id.
extern "C" int cgb_debug_sw_stats(unsigned long long* host, int n_cta) {
  // n_cta > 1024: all 8 launch slots (8 x 1024 x 16 counters); host == NULL: zero them
#ifndef CGB_PROFILING
  (void)host;
  (void)n_cta;
  return -1;
#endif
  if (!cgb::sw::g_stats) return -1;
  const size_t n = n_cta > 1024 ? (size_t)8 * 1024 * 16 : (size_t)n_cta * 16;
  if (!host) return cudaMemset(cgb::sw::g_stats, 0, n * sizeof(unsigned long long)) == cudaSuccess ? 0 : -1;
  return cudaMemcpy(host, cgb::sw::g_stats, n * sizeof(unsigned long long), cudaMemcpyDeviceToHost) == cudaSuccess
             ? 0
             : -1;
}
