// K4: 1-D convolution (16 taps, stride 1|2, "same" padding) as an implicit GEMM
// on tcgen05 tensor cores, with the folded-BN bias / shortcut add / ReLU and the
// optional mean-pool+FC head fused into the TMEM epilogue.
//
//   GEMM view (one tile = 128 output positions of one patient x bn channels):
//     D[m, n] = sum_{t, c} X[s*(l0+m) + t - pad, c] * W[n, c, t]
//   A (positions x K) is never materialised.  Per 8-channel group the producer
//   TMA-loads the contiguous run of input rows the tile touches as 128-byte
//   lines (8 rows x 8 channels): rows [l0+row0, l0+row0+152) for s=1; for s=2
//   the even- and odd-position planes of the parity-split (S) layout, 144 rows
//   each.  That smem image is the canonical K-major no-swizzle UMMA layout
//   (rows 16 B apart, SBO = 128 B), so tap t is the same region shifted by
//   whole rows: descriptor start + 16 B * row offset.  "Same" padding rows
//   outside [0, L) are zero-filled by TMA (negative / past-the-end lines) or
//   are the zero rows every producer writes past L.
//   B (weights) is pre-packed on the host into the exact smem image and moved
//   with plain bulk copies; it stays resident in smem across tiles when the
//   whole layer's weights fit.
//
// Roles (384 threads, 1 CTA/SM, persistent over tiles):
//   warp 0  : TMA producer (one lane)
//   warp 1  : MMA issuer (warp-uniform loop, one elected lane issues),
//             double-buffered TMEM accumulators (tile i of the CTA -> buffer i%2)
//   warp 2  : TMEM allocator
//   warps 4-7 / 8-11: two epilogue warpgroups, warpgroup e drains buffer e
//             (every other tile); thread r <-> TMEM lane r <-> position l0+r
#include "hb_kernels.cuh"
#include "hb_ptx.cuh"

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

namespace hb {

constexpr int kRowsS1 = 152;  // A rows per group for stride 1 (19 TMA lines)
constexpr int kRowsS2 = 144;  // A rows per (parity, group) for stride 2 (18 lines)

__host__ __device__ __forceinline__ int floordiv(int a, int b) { return (a >= 0) ? a / b : -((-a + b - 1) / b); }

__device__ __forceinline__ size_t out_offset(const ConvArgs& a, int p, int g, int l) {
  return q_off(static_cast<size_t>(p) * (a.cout / 8) + g, a.out_qs, a.out_lq, l);
}

// Shortcut source row for output position l: identity x[l], or maxpool(2)
// max(x[2l], x[2l+1]); x in its own Q-phase layout.
__device__ __forceinline__ uint4 res_row(const ConvArgs& a, size_t plane, int l) {
  if (a.res_mode == 1) return __ldg(reinterpret_cast<const uint4*>(a.res + q_off(plane, a.res_qs, a.res_lq, l)));
  const uint4 r0 = __ldg(reinterpret_cast<const uint4*>(a.res + q_off(plane, a.res_qs, a.res_lq, 2 * l)));
  const uint4 r1 = __ldg(reinterpret_cast<const uint4*>(a.res + q_off(plane, a.res_qs, a.res_lq, 2 * l + 1)));
  uint4 o;
  const __half2* h0 = reinterpret_cast<const __half2*>(&r0);
  const __half2* h1 = reinterpret_cast<const __half2*>(&r1);
  __half2* o2 = reinterpret_cast<__half2*>(&o);
#pragma unroll
  for (int k = 0; k < 4; ++k) o2[k] = __hmax2_nan(h0[k], h1[k]);
  return o;
}

// Tile order: member g of the group (slowest), N tile, patient, M tile.
struct TileIdx {
  int g, nt, p, mt;  // p = global row of the [G*Pm] activation tensors
};
// Pair mode: `tile` counts PAIRS of M tiles that share a weight image (member
// g, N tile nt): the flattened (patient, M tile) index f = 2*pair + rank, so a
// pair may span two beds (a layer with one M tile per bed still fills both
// CTAs).  An odd count leaves the last pair's second tile a phantom: M tile
// mt_per_p of the member's last bed, whose rows are all past the layer.
template <bool kPair = false>
__device__ __forceinline__ TileIdx decode_tile(const ConvArgs& a, int tile, int rank = 0) {
  const int per_nt = kPair ? a.mtp_per_p : a.Pm * a.mt_per_p;
  const int per_g = a.n_ntiles * per_nt;
  TileIdx t;
  t.g = tile / per_g;
  int rem = tile - t.g * per_g;
  t.nt = rem / per_nt;
  rem -= t.nt * per_nt;
  if (kPair) {
    const int f = 2 * rem + rank;
    if (f < a.Pm * a.mt_per_p) {
      const int pl = f / a.mt_per_p;
      t.mt = f - pl * a.mt_per_p;
      t.p = t.g * a.Pm + pl;
    } else {
      t.mt = a.mt_per_p;
      t.p = t.g * a.Pm + a.Pm - 1;
    }
    return t;
  }
  const int pl = rem / a.mt_per_p;
  t.mt = rem - pl * a.mt_per_p;
  t.p = t.g * a.Pm + pl;
  return t;
}

// Folded epilogue read: D'[r, (j, c)] holds folded tap j of output row r - j,
// so out[r, c] = D'[r, (0, c)] + D'[r + 1, (1, c)] for F = 2.  Row r + 1 of the
// same warp comes by shuffle; lane 31 takes row 32(w+1) from the next warp's
// lane 0 through a small shared-memory exchange (one named barrier per round).
#ifndef HB_K4_RES_PREFETCH
#define HB_K4_RES_PREFETCH 8
#endif
// Shortcut groups fetched before the accumulator wait.  16 lifts the 128-channel
// shortcut layers 15 % alone (zero data) but spills and leaves the power-capped
// c3 tick unchanged (47.4 vs 47.4 ms, profiles/r02_k4_wide_slots.txt): 8 stays.
constexpr int kResPrefetch = HB_K4_RES_PREFETCH;
constexpr int kXchRound = 3 * 32;            // [warp 0..2][32 channels]
constexpr int kXchPerWg = 2 * kXchRound;     // double-buffered by round parity
// Release of the accumulator after the last TMEM load: a local arrive, or in
// pair mode an arrive on the leader CTA's barrier (`release_cl`, shared::cluster).
template <bool kPair>
__device__ __forceinline__ void acc_release(uint64_t* release, uint32_t release_cl) {
  tc_fence_before();
  if constexpr (kPair) {
    mbar_arrive_cluster(release_cl);
  } else {
    mbar_arrive(release);
  }
}

template <int F, bool kPair>
__device__ __forceinline__ void fetch_round(uint32_t taddr, int bn, bool two, int wq, uint32_t lane, float* xch,
                                            int eg, float* v, uint64_t* release, uint32_t release_cl) {
  uint32_t r0[16], r1[16];
  tmem_ld16_nw(taddr, r0);
  if (two) tmem_ld16_nw(taddr + 16, r1);
  if constexpr (F == 1) {
    tmem_wait_ld();
    if (release) acc_release<kPair>(release, release_cl);
#pragma unroll
    for (int k = 0; k < 16; ++k) v[k] = __uint_as_float(r0[k]);
    if (two) {
#pragma unroll
      for (int k = 0; k < 16; ++k) v[16 + k] = __uint_as_float(r1[k]);
    }
  } else {
    uint32_t s0[16], s1[16];
    tmem_ld16_nw(taddr + static_cast<uint32_t>(bn), s0);
    if (two) tmem_ld16_nw(taddr + static_cast<uint32_t>(bn) + 16, s1);
    tmem_wait_ld();
    if (release) acc_release<kPair>(release, release_cl);
    if (wq > 0 && lane == 0) {  // my row 0, folded block 1 -> the warp above
      float* d = xch + (wq - 1) * 32;
#pragma unroll
      for (int k = 0; k < 16; ++k) d[k] = __uint_as_float(s0[k]);
      if (two) {
#pragma unroll
        for (int k = 0; k < 16; ++k) d[16 + k] = __uint_as_float(s1[k]);
      }
    }
    named_bar_sync(1 + eg, 128);
    const float* b = xch + (wq < 3 ? wq : 0) * 32;
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      float t = __shfl_down_sync(0xffffffffu, __uint_as_float(s0[k]), 1);
      if (lane == 31) t = (wq < 3) ? b[k] : 0.f;
      v[k] = __uint_as_float(r0[k]) + t;
    }
    if (two) {
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        float t = __shfl_down_sync(0xffffffffu, __uint_as_float(s1[k]), 1);
        if (lane == 31) t = (wq < 3) ? b[16 + k] : 0.f;
        v[16 + k] = __uint_as_float(r1[k]) + t;
      }
    }
  }
}

// MMA issue for one k-chunk with `F` taps folded into N, by the calling
// (elected) lane: two descriptor adds per MMA, no per-MMA election (the issue
// loop is on the tensor pipe's critical path, as in K4b).
template <bool kPair>
__device__ __forceinline__ void mma_any(uint32_t d, uint64_t ad, uint64_t bd, uint32_t idesc, uint32_t acc) {
  if constexpr (kPair) {
    mma_f16_ss_pair(d, ad, bd, idesc, acc);
  } else {
    mma_f16_ss(d, ad, bd, idesc, acc);
  }
}
template <bool kPair>
__device__ __forceinline__ void commit_any(uint64_t* bar) {
  if constexpr (kPair) {
    mma_commit_pair(bar);
  } else {
    mma_commit(bar);
  }
}

template <int F, bool kPair, typename ToffS2>
__device__ __forceinline__ void issue_groups(const ConvArgs& a, uint32_t d_tmem, uint64_t adesc, uint64_t bdesc,
                                             uint32_t idesc, uint32_t& accum, int per_tap, uint32_t rows16,
                                             uint32_t bstep16, uint32_t btap, ToffS2 toff_s2) {
  for (int j = 0; j < per_tap; ++j) {
    uint64_t bd = bdesc + static_cast<uint32_t>(j) * bstep16;
    if (a.stride == 1) {
      uint64_t ad = adesc + static_cast<uint32_t>(2 * j) * rows16 + static_cast<uint32_t>(-a.pad - a.row0);
#pragma unroll
      for (int q = 0; q < kTaps / F; ++q) {
        mma_any<kPair>(d_tmem, ad, bd, idesc, accum);
        accum = 1u;
        ad += F;
        bd += btap;
      }
    } else {
      const uint64_t ag = adesc + static_cast<uint32_t>(2 * j) * rows16;
      uint64_t a0 = ag + toff_s2(0), a1 = ag + toff_s2(1);
#pragma unroll
      for (int q = 0; q < kTaps / (2 * F); ++q) {
        mma_any<kPair>(d_tmem, a0, bd, idesc, accum);
        accum = 1u;
        bd += btap;
        mma_any<kPair>(d_tmem, a1, bd, idesc, 1u);
        bd += btap;
        a0 += F;
        a1 += F;
      }
    }
  }
}

// kHalf (pair mode only): M = 128 over the pair, 64 output positions per CTA, for
// layers whose whole output fits 64 rows per bed (the 1024-channel L = 59 / 30
// layers: two beds per pair instead of one bed per 128-row tile).  The UMMA
// 2-SM M=128 accumulator is laid out 64 rows x N in two halves: TMEM lanes
// 0-63 hold columns [0, N/2), lanes 64-127 columns [N/2, N) of the same rows.
template <int F, bool kPair, bool kHalf = false>
__global__ void __launch_bounds__(kConvThreads, 1)
    conv_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   const __grid_constant__ ConvArgs a) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sB = smem;
  uint8_t* sA = smem + a.nb_slots * a.b_slot_bytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sA + a.na_stages * a.a_stage_bytes);
  uint64_t* a_full = bars;
  uint64_t* a_empty = a_full + a.na_stages;
  uint64_t* b_full = a_empty + a.na_stages;
  uint64_t* b_empty = b_full + a.nb_slots;
  uint64_t* acc_full = b_empty + a.nb_slots;
  uint64_t* acc_empty = acc_full + 2;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(acc_empty + 2);
  float* s_head = reinterpret_cast<float*>(tmem_holder + 4);  // [2][4] per-warp head partials
  float* s_bias = s_head + 8;                                  // [G][bn] when every N tile is whole
  float* s_fc = s_bias + a.sb_len;                             // [G][bn]
  float* s_xch = s_fc + a.sb_len;                              // [2 wg][kXchPerWg] folded-row exchange

  const uint32_t warp = warp_id();
  const uint32_t lane = lane_id();
  // Pair mode: cluster of two CTAs; rank 0 (the leader) issues every MMA and
  // owns the full / acc_empty barriers both CTAs' TMA bytes and epilogues count on.
  const int rank = kPair ? static_cast<int>(cluster_rank()) : 0;
  const bool leader = rank == 0;
  const int t_first = kPair ? static_cast<int>(cluster_id_x()) : static_cast<int>(blockIdx.x);
  const int t_step = kPair ? static_cast<int>(n_clusters_x()) : static_cast<int>(gridDim.x);

  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tmA);
    if (kPair) prefetch_tmap(&tmB);
    for (int i = 0; i < a.na_stages; ++i) {
      mbar_init(&a_full[i], 1);
      mbar_init(&a_empty[i], 1);
    }
    for (int i = 0; i < a.nb_slots; ++i) {
      mbar_init(&b_full[i], 1);
      mbar_init(&b_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&acc_full[i], 1);
      mbar_init(&acc_empty[i], kPair ? 256 : 128);  // one epilogue warpgroup per buffer (per CTA of the pair)
    }
    fence_barrier_init();
    // Weights are immutable: the first tile's resident B goes out right behind
    // the barrier init (before the dependency wait), hiding the prologue.
    if (!kPair && a.b_resident && static_cast<int>(blockIdx.x) < a.num_tiles) {
      const TileIdx t0 = decode_tile(a, blockIdx.x);
      for (int kc = 0; kc < a.n_kchunks; ++kc) {
        mbar_arrive_expect_tx(&b_full[kc], a.b_chunk_bytes);
        bulk_load(sB + static_cast<size_t>(kc) * a.b_chunk_bytes,
                  a.wpack + static_cast<size_t>(t0.g) * a.wpack_stride +
                      (static_cast<size_t>(t0.nt) * a.n_kchunks + kc) * a.b_chunk_bytes,
                  a.b_chunk_bytes, &b_full[kc]);
      }
    }
  }
  if (warp == 2) {
    if (kPair) {
      tmem_alloc_pair(tmem_holder, a.tmem_cols);
    } else {
      tmem_alloc(tmem_holder, a.tmem_cols);
    }
  }
  const bool smem_bias = a.sb_len > 0;  // every member's bias / fc cached in smem (filled by the epilogue warps)
  tc_fence_before();
  __syncthreads();
  if (kPair) cluster_sync_all();  // the peer's TMA / arrives target the leader's barriers: both initialised first
  tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;
  // Programmatic dependent launch: let the next layer's CTAs start their
  // prologue as SMs free up; everything that reads the previous layer's
  // output or writes ours happens after griddepcontrol.wait.
  pdl_trigger();

  const int groups = a.ck / 8;
  const uint32_t region_bytes = static_cast<uint32_t>(groups * a.rows * 16);

  if (warp == 0) {
    if (lane == 0) {
      // ------------------------------------------------------------ producer
      int as = 0;
      uint32_t aph = 0;
      int bs = 0;
      uint32_t bph = 0;
      int loaded_key = -1;
      auto b_src = [&](const TileIdx& t, int kc) {
        return a.wpack + static_cast<size_t>(t.g) * a.wpack_stride +
               (static_cast<size_t>(t.nt) * a.n_kchunks + kc) * a.b_chunk_bytes;
      };
      if (!kPair && a.b_resident && static_cast<int>(blockIdx.x) < a.num_tiles) {  // loaded in the prologue
        const TileIdx t0 = decode_tile(a, blockIdx.x);
        loaded_key = t0.g * a.n_ntiles + t0.nt;
      }
      // pair mode: the leader's full barriers (shared::cluster addresses) and the B box shape
      const int b_rows = static_cast<int>(a.b_slot_bytes >> 7);
      const int b_box = b_rows < 256 ? b_rows : 256;
      pdl_wait();
      int li = 0;       // local tile count
      int reloads = 0;  // resident-B reloads so far
      for (int tile = t_first; tile < a.num_tiles; tile += t_step, ++li) {
        const TileIdx t = decode_tile<kPair>(a, tile, rank);
        const int p = t.p;
        const int blk = (t.mt * a.stride_m + a.row0) / 8;  // first 128-B line (8 rows)
        const int key = t.g * a.n_ntiles + t.nt;
        const bool load_b = !a.b_resident || key != loaded_key;
        // Reloading resident weights (next member of the group): the MMA warp
        // signals b_empty[0] once per reload, after the last MMA that reads
        // the old weights has completed (one completion per reload, so the
        // phase parity is unambiguous).
        if (a.b_resident && load_b && li > 0) mbar_wait(&b_empty[0], static_cast<uint32_t>(reloads++) & 1u, 1);
        loaded_key = key;
        for (int kc = 0; kc < a.n_kchunks; ++kc) {
          if (load_b) {
            const int slot = a.b_resident ? kc : bs;
            if (!a.b_resident) mbar_wait(&b_empty[bs], bph ^ 1, 2);
            if constexpr (kPair) {
              // this CTA's half of the k-chunk's image (N rows [rank*bn/2, (rank+1)*bn/2)),
              // counted on the leader's b_full
              if (leader) mbar_arrive_expect_tx(&b_full[slot], 2 * a.b_slot_bytes);
              const uint32_t bar = map_to_rank(&b_full[slot], 0);
              const size_t off = static_cast<size_t>(t.g) * a.wpack_stride +
                                 (static_cast<size_t>(t.nt) * a.n_kchunks + kc) * a.b_chunk_bytes +
                                 static_cast<size_t>(rank) * a.b_slot_bytes;
              const int row = static_cast<int>(off >> 7);
              for (int r0 = 0; r0 < b_rows; r0 += b_box)
                tma_load_2d_pair(sB + static_cast<size_t>(slot) * a.b_slot_bytes + static_cast<size_t>(r0) * 128,
                                 &tmB, bar, 0, row + r0);
            } else {
              mbar_arrive_expect_tx(&b_full[slot], a.b_chunk_bytes);
              bulk_load(sB + static_cast<size_t>(slot) * a.b_chunk_bytes, b_src(t, kc), a.b_chunk_bytes,
                        &b_full[slot]);
            }
            if (!a.b_resident && ++bs == a.nb_slots) {
              bs = 0;
              bph ^= 1;
            }
          }
          mbar_wait(&a_empty[as], aph ^ 1, 3);
          uint8_t* dst = sA + static_cast<size_t>(as) * a.a_stage_bytes;
          if constexpr (kPair) {
            if (leader) mbar_arrive_expect_tx(&a_full[as], 2 * a.a_stage_bytes);
            const uint32_t bar = map_to_rank(&a_full[as], 0);
            if (a.stride == 1) {
              tma_load_4d_pair(dst, &tmA, bar, 0, blk, kc * groups, p);
            } else {
              tma_load_5d_pair(dst, &tmA, bar, 0, blk, 0, kc * groups, p);
              tma_load_5d_pair(dst + region_bytes, &tmA, bar, 0, blk, 1, kc * groups, p);
            }
          } else {
            mbar_arrive_expect_tx(&a_full[as], a.a_stage_bytes);
            if (a.stride == 1) {
              tma_load_4d(dst, &tmA, &a_full[as], 0, blk, kc * groups, p);
            } else {
              tma_load_5d(dst, &tmA, &a_full[as], 0, blk, 0, kc * groups, p);
              tma_load_5d(dst + region_bytes, &tmA, &a_full[as], 0, blk, 1, kc * groups, p);
            }
          }
          if (++as == a.na_stages) {
            as = 0;
            aph ^= 1;
          }
        }
      }
      if constexpr (kPair) {
        // The leader's commits arrive on BOTH CTAs' empty barriers: wait until every
        // stage / slot this CTA filled has been released before the CTA may exit.
        if (li > 0) {
          for (int i = 0; i < a.na_stages; ++i) {
            mbar_wait(&a_empty[as], aph ^ 1, 4);
            if (++as == a.na_stages) {
              as = 0;
              aph ^= 1;
            }
          }
          for (int i = 0; i < a.nb_slots; ++i) {
            mbar_wait(&b_empty[bs], bph ^ 1, 5);
            if (++bs == a.nb_slots) {
              bs = 0;
              bph ^= 1;
            }
          }
        }
      }
    }
  } else if (warp == 1 && leader) {
    // -------------------------------------------------------------- MMA issuer
    // The whole warp walks the loop with warp-uniform values (kept in uniform
    // registers); one elected lane issues each tcgen05.mma / commit.
    const uint32_t idesc = make_idesc_f16(kPair ? (kHalf ? kBM : 2 * kBM) : kBM, a.bnp);
    const int acc_cols = kHalf ? a.bnp / 2 : a.bnp;  // TMEM columns per accumulator
    const uint32_t a_lbo = (a.ck >= 16) ? static_cast<uint32_t>(a.rows * 16) : 16u;
    const int b_n = kPair ? a.bnp / 2 : a.bnp;  // B rows held by this CTA
    const uint32_t b_lbo = static_cast<uint32_t>(b_n * 16);
    const uint32_t rows16 = static_cast<uint32_t>(a.rows);  // one group column, 16 B units
    const uint32_t region16 = region_bytes >> 4;           // one parity region
    const uint32_t bstep16 = static_cast<uint32_t>(2 * b_n);
    const int per_tap = a.ck >> 4;  // 0 for 8-channel chunks
    // stride-2 A offset (16 B units) of tap t in {0, 1}: parity region + pair row
    auto toff_s2 = [&](int t) -> uint32_t {
      const int u = t - a.pad;
      return static_cast<uint32_t>(u & 1) * region16 + static_cast<uint32_t>((u >> 1) - a.row0);
    };
    int as = 0;
    uint32_t aph = 0;
    int bs = 0;
    uint32_t bph = 0;
    int acc = 0;
    uint32_t accph = 0;
    uint32_t bres_ph = 0;  // phase of the resident B slots (flips on every reload)
    // weight key of a tile = tile / per_key (member g, N tile nt); tracked with
    // a compare per tile, a division only when the key changes
    const bool multi_key = a.b_resident && (a.G > 1 || a.n_ntiles > 1);
    const int per_key = a.Pm * a.mt_per_p;
    int mkey = static_cast<int>(blockIdx.x) / per_key;
    int kbound = (mkey + 1) * per_key;
    unsigned long long t_acc = 0, t_a = 0, t_issue = 0, t0 = 0;
    const bool prof = (a.dbg & 8) && a.prof;
    for (int tile = t_first; tile < a.num_tiles; tile += t_step) {
      if (multi_key && tile >= kbound) {
        bres_ph ^= 1;
        mkey = tile / per_key;
        kbound = (mkey + 1) * per_key;
      }
      if (prof) t0 = clock64();
      mbar_wait(&acc_empty[acc], accph ^ 1, 10 + 1000 * static_cast<int>(bres_ph));
      if (prof) t_acc += clock64() - t0;
      tc_fence_after();
      const uint32_t d_tmem = tmem_base + static_cast<uint32_t>(acc * acc_cols);
      for (int kc = 0; kc < a.n_kchunks; ++kc) {
        const int slot = a.b_resident ? kc : bs;
        if (prof) t0 = clock64();
        mbar_wait(&b_full[slot], a.b_resident ? bres_ph : bph, 11 + 1000 * slot);
        mbar_wait(&a_full[as], aph, 12 + 1000 * as);
        if (prof) {
          const unsigned long long t1 = clock64();
          t_a += t1 - t0;
          t0 = t1;
        }
        tc_fence_after();
        const uint64_t adesc = make_desc(smem_u32(sA + static_cast<size_t>(as) * a.a_stage_bytes), a_lbo, 128);
        const uint64_t bdesc = make_desc(smem_u32(sB + static_cast<size_t>(slot) * a.b_slot_bytes), b_lbo, 128);
        // Descriptor walk with two 64-bit adds per MMA.  B K-steps are ordered
        // (tap, 16-channel sub-chunk j); A for tap t is the region shifted by
        // toff(t) rows: s=1 -> t - pad - row0 (+1 per tap); s=2 -> even/odd
        // taps alternate parity regions, each advancing one row per tap pair.
        uint32_t accum = kc > 0 ? 1u : 0u;
        if (elect_one()) {
        if (per_tap > 0) {
          // K-steps are (tap group q, 16-channel sub-chunk j); a tap group is
          // `fold` taps sharing one A view (s=1: taps qF..qF+F-1; s=2: taps of
          // one parity, t0, t0+2, ..), their weights side by side in N.
          const uint32_t btap = static_cast<uint32_t>(per_tap) * bstep16;
          issue_groups<F, kPair>(a, d_tmem, adesc, bdesc, idesc, accum, per_tap, rows16, bstep16, btap, toff_s2);
        } else {
          // 8-channel chunk: one K-step pairs taps (t, t+1) [s=1] or (t, t+2) [s=2],
          // i.e. the same region one row apart (LBO = 16 B)
          uint64_t bd = bdesc;
          if (a.stride == 1) {
            uint64_t ad = adesc + static_cast<uint32_t>(-a.pad - a.row0);
#pragma unroll
            for (int ks = 0; ks < 8; ++ks) {
              mma_any<kPair>(d_tmem, ad, bd, idesc, accum);
              accum = 1u;
              ad += 2;
              bd += bstep16;
            }
          } else {
            uint64_t a0 = adesc + toff_s2(0), a1 = adesc + toff_s2(1);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              mma_any<kPair>(d_tmem, a0, bd, idesc, accum);
              accum = 1u;
              bd += bstep16;
              mma_any<kPair>(d_tmem, a1, bd, idesc, 1u);
              bd += bstep16;
              a0 += 2;
              a1 += 2;
            }
          }
        }
          commit_any<kPair>(&a_empty[as]);  // the same lane that issued the k-chunk's MMAs
          if (!a.b_resident) commit_any<kPair>(&b_empty[bs]);
        }
        __syncwarp();
        if (prof) t_issue += clock64() - t0;
        if (!a.b_resident && ++bs == a.nb_slots) {
          bs = 0;
          bph ^= 1;
        }
        if (++as == a.na_stages) {
          as = 0;
          aph ^= 1;
        }
      }
      if (elect_one()) commit_any<kPair>(&acc_full[acc]);
      __syncwarp();
      if (multi_key && tile + static_cast<int>(gridDim.x) >= kbound &&
          tile + static_cast<int>(gridDim.x) < a.num_tiles) {  // the next tile needs other weights
        if (elect_one()) mma_commit(&b_empty[0]);
        __syncwarp();
      }
      if (++acc == 2) {
        acc = 0;
        accph ^= 1;
      }
    }
    if (prof && lane == 0) {
      a.prof[blockIdx.x * 8 + 0] = t_acc;
      a.prof[blockIdx.x * 8 + 1] = t_a;
      a.prof[blockIdx.x * 8 + 2] = t_issue;
    }
  } else if (warp >= 4) {
    // -------------------------------------------------------------- epilogue
    const int eg = (static_cast<int>(warp) - 4) >> 2;  // epilogue warpgroup = accumulator buffer
    const int wq = static_cast<int>(warp) & 3;          // TMEM lane quadrant of this warp
    const int r_lane = wq * 32 + static_cast<int>(lane);
    const int r = kHalf ? (r_lane & 63) : r_lane;         // output row of this thread
    const int chalf = kHalf ? (r_lane >> 6) : 0;          // kHalf: which half of the N tile's channels
    const int acc = eg;
    uint32_t accph = 0;
    const int out_groups = a.cout / 8;
    const int res_groups = a.res_mode ? a.res_c / 8 : 0;
    const bool eprof = (a.dbg & 8) && a.prof && wq == 0 && lane == 0 && eg == 0;
    unsigned long long e_wait = 0, e_work = 0, et0 = 0, e_start = eprof ? clock64() : 0;
    uint32_t xround = 0;  // exchange buffer parity, alternates every round across tiles
    if (smem_bias) {
      for (int i = static_cast<int>(threadIdx.x) - 128; i < a.G * a.bn; i += static_cast<int>(blockDim.x) - 128) {
        const int g = i / a.bn, c = i - g * a.bn;
        s_bias[i] = a.bias[static_cast<size_t>(g) * a.bias_stride + c];
        s_fc[i] = a.fc_w ? a.fc_w[static_cast<size_t>(g) * a.cout + (c < a.cout ? c : 0)] : 0.f;
      }
      named_bar_sync(3, blockDim.x - 128);  // the epilogue warps alone (ids 1, 2: per-warpgroup exchange)
    }
    const uint32_t release_cl = kPair ? map_to_rank(&acc_empty[acc], 0) : 0u;
    pdl_wait();
    for (int tile = t_first + eg * t_step; tile < a.num_tiles; tile += 2 * t_step) {
      const TileIdx ti = decode_tile<kPair>(a, tile, rank);
      const int nt = ti.nt;
      const int p = ti.p;
      const int mt = ti.mt;
      const int l = mt * a.stride_m + r;
      const bool own = r < a.stride_m;  // rows past stride_m belong to the next tile (folded taps)
      const bool valid = own && l < a.lout;
      const bool in_buf = own && l < a.out_rows;
      const int g0 = nt * (a.bn / 8) + chalf * (a.bn / 16);
      const int ng = min(kHalf ? a.bn / 16 : a.bn / 8, out_groups - g0);
      // Shortcut rows are independent of the accumulator: fetch the first 8
      // groups while the MMAs of this tile are still running.
      // identity: block input in I layout; maxpool: block input in S layout,
      // max(x[2l], x[2l+1]) = max(even plane row l, odd plane row l).
      uint4 rres[kResPrefetch];
#pragma unroll
      for (int j = 0; j < kResPrefetch; ++j) {
        rres[j] = make_uint4(0u, 0u, 0u, 0u);
        const int g = g0 + j;
        if (j < ng && g < res_groups && valid) {
          rres[j] = res_row(a, static_cast<size_t>(p) * res_groups + g, l);
        }
      }
      const int coff = chalf * (a.bn / 2);  // kHalf: this thread's channels start half an N tile in
      const float* bias_t = smem_bias ? s_bias + ti.g * a.bn + coff
                                      : a.bias + static_cast<size_t>(ti.g) * a.bias_stride +
                                            static_cast<size_t>(nt) * a.bn + coff;
      const float* fc_t = smem_bias ? s_fc + ti.g * a.bn + coff
                                    : a.fc_w + static_cast<size_t>(ti.g) * a.cout + static_cast<size_t>(nt) * a.bn + coff;
      if (eprof) et0 = clock64();
      mbar_wait(&acc_full[acc], accph, 20 + 1000 * mt);
      if (eprof) {
        const unsigned long long t1 = clock64();
        e_wait += t1 - et0;
        et0 = t1;
      }
      tc_fence_after();
      const uint32_t taddr = tmem_base + (static_cast<uint32_t>(wq * 32) << 16) +
                             static_cast<uint32_t>(acc * (kHalf ? a.bnp / 2 : a.bnp));
      float head = 0.f;
      // Rounds of up to 32 output channels: all TMEM loads of a round are
      // issued before one wait; after the last round's loads the accumulator
      // is released, so the next tile's MMAs overlap this tile's math/stores.
      const int nrounds = (ng + 3) >> 2;
      if (nrounds <= 0) acc_release<kPair>(&acc_empty[acc], release_cl);  // (kHalf: no channels in this half)
#pragma unroll
      for (int q = 0; q < 8; ++q) {  // unrolled: the shortcut registers are indexed statically
        if (q >= nrounds) break;
        const bool two = ng > 4 * q + 2;  // second 16-channel chunk in this round
        float v[32];
        fetch_round<F, kPair>(taddr + static_cast<uint32_t>(q * 32), a.bn, two, wq, lane,
                              s_xch + eg * kXchPerWg + (xround++ & 1) * kXchRound, eg, v,
                              q == nrounds - 1 ? &acc_empty[acc] : nullptr, release_cl);
#pragma unroll
        for (int h = 0; h < 4; ++h) {
          const int j = 4 * q + h;
          if (j >= ng) break;
          const int g = g0 + j;
          float y[8];
#pragma unroll
          for (int k = 0; k < 8; ++k) y[k] = v[8 * h + k] + bias_t[8 * j + k];
          if (g < res_groups && valid) {
            uint4 rv;
            if (j < kResPrefetch) {
              rv = rres[j < kResPrefetch ? j : 0];
            } else {
              rv = res_row(a, static_cast<size_t>(p) * res_groups + g, l);
            }
            const __half2* h2 = reinterpret_cast<const __half2*>(&rv);
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const float2 f = __half22float2(h2[k]);
              y[2 * k] += f.x;
              y[2 * k + 1] += f.y;
            }
          }
          if (a.relu) {
#pragma unroll
            for (int k = 0; k < 8; ++k) y[k] = fmax_nan(y[k], 0.f);
          }
          if (a.fc_w != nullptr) {
            if (valid) {
#pragma unroll
              for (int k = 0; k < 8; ++k) head = fmaf(y[k], fc_t[8 * j + k], head);
            }
          } else if (in_buf) {
            uint4 pk;
            __half2* o2 = reinterpret_cast<__half2*>(&pk);
#pragma unroll
            for (int k = 0; k < 4; ++k)
              o2[k] = valid ? __floats2half2_rn(y[2 * k], y[2 * k + 1]) : __floats2half2_rn(0.f, 0.f);
            *reinterpret_cast<uint4*>(a.out + out_offset(a, p, g, l)) = pk;
          }
        }
      }
      if (eprof) e_work += clock64() - et0;
      accph ^= 1;
      if (a.fc_w != nullptr) {
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) head += __shfl_xor_sync(0xffffffffu, head, off);
        float* sh = s_head + 4 * eg;
        if (lane == 0) sh[wq] = head;
        named_bar_sync(1 + eg, 128);
        if (wq == 0 && lane == 0 && (!kPair || mt < a.mt_per_p)) {  // (pair mode: an odd last tile has no slot)
          const float sum = ((sh[0] + sh[1]) + sh[2]) + sh[3];
          a.head_out[static_cast<size_t>(ti.g) * a.head_g_stride +
                     (static_cast<size_t>(p - ti.g * a.Pm) * a.n_ntiles + nt) * a.mt_per_p + mt] = sum;
        }
        named_bar_sync(1 + eg, 128);
      }
    }
    if (eprof) {
      a.prof[blockIdx.x * 8 + 3] = e_wait;
      a.prof[blockIdx.x * 8 + 4] = e_work;
      a.prof[blockIdx.x * 8 + 5] = clock64() - e_start;
    }
  }

  tc_fence_before();
  __syncthreads();
  if (kPair) cluster_sync_all();  // the peer's last releases reached the leader; every MMA has completed
  tc_fence_after();
  if (warp == 2) {
    if (kPair) {
      tmem_dealloc_pair(tmem_base, a.tmem_cols);
    } else {
      tmem_dealloc(tmem_base, a.tmem_cols);
    }
  }
}

// ------------------------------------------------------------------ host side

int conv_bn(int cout) {
  const int c = round_up(cout < 16 ? 16 : cout, 16);
  if (c <= 256) return c;
  const int nt = (c + 255) / 256;  // split N into equal tiles of <= 256 (multiple of 16)
  return round_up((c + nt - 1) / nt, 16);
}

// barriers + holder/head scratch + per-member bias and fc (up to 1024 floats each)
constexpr int kSmemBiasMax = 1024;
constexpr uint32_t kXchBytes = 2 * kXchPerWg * 4;  // folded-row exchange, both epilogue warpgroups
// upper bound used for the k-chunk / residency decision (shared with the packer)
constexpr uint32_t kFixedSmem = 1024 + 256 + 2 * kSmemBiasMax * 4 + kXchBytes;

int conv_stride_m(int fold) { return fold > 1 ? 120 : kBM; }
static int pick_ck(int cin, int cout, int stride, int* resident);

// Taps folded into N: enough to lift a narrow layer off the shared-memory
// bound (A is read once per tap group instead of once per tap) while
// F*bn <= 256 (MMA N, and 2 TMEM accumulators <= 512 columns).  HB_FOLD
// caps it (1 disables).  8-channel k-chunks keep their tap-pair K layout.
int conv_fold(int cin, int cout, int stride) {
  static const int cap = getenv("HB_FOLD") ? atoi(getenv("HB_FOLD")) : 1;  // off by default (see below)
  int resident;
  const int ck = pick_ck(cin, cout, stride, &resident);
  const int bn = conv_bn(cout);
  if (ck < 16 || round_up(cout, 16) > bn) return 1;  // (several N tiles: no fold)
  // Measured (profiles/r01_fold_ab.txt): at bn = 32 the folded epilogue, not
  // the MMA, bounds the tile; 64 -> 64 layers gain 4-8 % alone, wider or
  // channel-doubling layers lose, and inside the two-branch tick graph even
  // the 64 -> 64-only setting loses (1.212 vs 1.177 ms), so HB_FOLD=2 is an
  // opt-in experiment.
  if (bn != 64 || cin < 64) return 1;
  int f = 1;
  while (f * 2 <= cap && f * 2 <= 2 && f * 2 * bn <= 256) f *= 2;
  return f;
}

static int a_rows(int stride) { return stride == 1 ? kRowsS1 : kRowsS2; }

// CTA pairs (cta_group::2) for the streamed-weight layers: two CTAs of a TPC
// share each MMA (M = 256 = two adjacent M tiles, B split along N), so each
// SM reads half the weight image per MMA from shared memory and fetches half
// of it from L2.  Read once per process: the weight packer and the planner
// must agree.  HB_K4_PAIR=0 keeps single-CTA tiles.
bool conv_pair(int cin, int cout, int stride) {
  static const int on = getenv("HB_K4_PAIR") ? atoi(getenv("HB_K4_PAIR")) : 1;
  if (!on) return false;
  int resident;
  const int ck = pick_ck(cin, cout, stride, &resident);
  if (ck == 0 || resident || conv_fold(cin, cout, stride) != 1) return false;
  const int bn = conv_bn(cout);
  if (bn < 128 || bn % 32) return false;
  const int ksteps = ck >= 16 ? ck : 8;
  const int half_rows = ksteps * bn / 8;  // 128-B rows of one CTA's half of a k-chunk image
  return half_rows <= 256 || half_rows % 256 == 0;
}

// Channels per k-chunk.  Prefer the largest chunk whose whole-layer weights
// stay resident in smem next to two A stages; otherwise the largest chunk that
// streams with two B slots + two A stages.  The host packer and the planner
// both call this, so the B image always matches the kernel's K-step order.
static int pick_ck(int cin, int cout, int stride, int* resident) {
  const int bn = conv_bn(cout);
  const int nnt = (round_up(cout, 16) + bn - 1) / bn;
  const uint32_t budget = kSmemLimit - kFixedSmem;
  const int cands[4] = {64, 32, 16, 8};
  if (nnt == 1) {
    for (int ck : cands) {
      if (cin % ck || cin / ck > 32) continue;
      const uint32_t b_all = 32u * cin * bn;  // 16 taps * cin * bn * 2 B
      const uint32_t a_stage = static_cast<uint32_t>(stride * a_rows(stride) * ck * 2);
      if (b_all + 2 * a_stage <= budget) {
        *resident = 1;
        return ck;
      }
    }
  }
  for (int ck : cands) {
    if (cin % ck) continue;
    const uint32_t b_chunk = 32u * ck * bn;
    const uint32_t a_stage = static_cast<uint32_t>(stride * a_rows(stride) * ck * 2);
    if (2 * b_chunk + 2 * a_stage <= budget) {
      *resident = 0;
      return ck;
    }
  }
  *resident = 0;
  return 0;
}

size_t wpack_bytes(int cin, int cout) {
  const int bn = conv_bn(cout);
  const int nnt = (round_up(cout, 16) + bn - 1) / bn;
  return static_cast<size_t>(nnt) * bn * cin * kTaps * 2;
}

// B image per (ntile, kchunk): [kstep][half][bn rows][8 fp16] in the MMA
// issuer's K-step order (tap-major, then 16-channel sub-chunks; 8-channel
// chunks pair taps (t, t+1) for s=1 or (t, t+2) for s=2).
void pack_weights(const float* w, int cin, int cout, int stride, uint16_t* dst) {
  const int bn = conv_bn(cout);
  const int nnt = (round_up(cout, 16) + bn - 1) / bn;
  int resident;
  const int ck = pick_ck(cin, cout, stride, &resident);
  if (ck == 0) return;
  const int nkc = cin / ck;
  const int F = conv_fold(cin, cout, stride);
  const int ksteps = (ck >= 16) ? ck / F : 8;  // K-steps per k-chunk
  // pair mode: each k-chunk image is two halves, one per CTA of the pair, each
  // holding N rows [r*bn/2, (r+1)*bn/2) in the same (kstep, half) order
  const int nr = conv_pair(cin, cout, stride) ? 2 : 1;
  const int rows = bn / nr;
  size_t o = 0;
  for (int nt = 0; nt < nnt; ++nt)
    for (int kc = 0; kc < nkc; ++kc)
      for (int rk = 0; rk < nr; ++rk)
      for (int ks = 0; ks < ksteps; ++ks)
        for (int half = 0; half < 2; ++half)
          for (int jj = 0; jj < F; ++jj) {  // N rows: folded tap jj, then output channel
            int t, c0;
            if (ck >= 16) {
              const int per_tap = ck / 16;
              const int gi = ks / per_tap;  // tap group
              const int base = (stride == 1) ? gi * F : (gi >> 1) * 2 * F + (gi & 1);
              t = base + jj * stride;
              c0 = kc * ck + 16 * (ks % per_tap) + 8 * half;
            } else {
              const int t0 = (stride == 1) ? 2 * ks : (ks / 2) * 4 + (ks % 2);
              t = t0 + half * stride;
              c0 = kc * ck;
            }
            for (int n = rk * rows; n < (rk + 1) * rows; ++n)
              for (int j = 0; j < 8; ++j) {
                const int co = nt * bn + n;
                const float v = (co < cout) ? w[(static_cast<size_t>(co) * cin + (c0 + j)) * kTaps + t] : 0.f;
                const __half hv = __float2half_rn(v);
                uint16_t bits;
                std::memcpy(&bits, &hv, 2);
                dst[o++] = bits;
              }
          }
}

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn get_encode() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

size_t bias_len(int cout) {
  const int bn = conv_bn(cout);
  return static_cast<size_t>(((round_up(cout, 16) + bn - 1) / bn) * bn);
}

bool pdl_enabled() {
  static const bool on = !(getenv("HB_NO_PDL") && atoi(getenv("HB_NO_PDL")));
  return on;
}

const char* plan_conv(ConvPlan* plan, int G, int Pm, int cin, int cout, int lin, int lout, int stride, int pad,
                      const __half* in, __half* out, int out_q, const uint8_t* wpack, const float* bias,
                      const __half* res, int res_mode, int res_c, int res_len, int res_q, const float* fc_w,
                      float* head_out, int num_sms, size_t head_g_stride) {
  std::memset(plan, 0, sizeof(*plan));
  if (G < 1 || G > kMaxGroup || Pm < 1) return "conv: bad group shape";
  const int P = G * Pm;
  if (cin % 8 || cout % 8) return "conv: channels must be multiples of 8";
  if (stride != 1 && stride != 2) return "conv: stride must be 1 or 2";
  if (lout != (lin + stride - 1) / stride) return "conv: lout must be ceil(lin/stride)";
  ConvArgs& a = plan->args;
  a.P = P;
  a.G = G;
  a.Pm = Pm;
  a.cin = cin;
  a.cout = cout;
  a.bn = conv_bn(cout);
  a.n_ntiles = (round_up(cout, 16) + a.bn - 1) / a.bn;
  a.lin = lin;
  a.lout = lout;
  if (out_q < 1 || out_q > 32 || (out_q & (out_q - 1))) return "conv: out_q must be a power of two <= 32";
  if (res && (res_q < 1 || res_q > 32 || (res_q & (res_q - 1)))) return "conv: res_q must be a power of two <= 32";
  a.out_qs = ilog2(out_q);
  a.out_lq = lq_Q(lout, out_q);
  a.out_rows = fc_w ? lout : act_rows_q(lout, out_q);
  a.stride = stride;
  a.pad = pad;
  a.rows = a_rows(stride);
  if (stride == 1) {
    a.row0 = -8 * ((pad + 7) / 8);
    if (kBM - 1 + (kTaps - 1 - pad - a.row0) >= a.rows) return "conv: padding too large for the A tile";
  } else {
    a.row0 = 8 * floordiv(floordiv(-pad, 2), 8);
    if (kBM - 1 + (floordiv(kTaps - 1 - pad, 2) - a.row0) >= a.rows) return "conv: padding too large for the A tile";
  }
  int resident = 0;
  a.ck = pick_ck(cin, cout, stride, &resident);
  if (a.ck == 0) return "conv: no k-chunk fits in shared memory";
  a.n_kchunks = cin / a.ck;
  a.fold = conv_fold(cin, cout, stride);
  a.bnp = a.fold * a.bn;
  a.stride_m = conv_stride_m(a.fold);
  a.pair = conv_pair(cin, cout, stride) ? 1 : 0;
  {  // half pairs: M = 128 over the pair (64 rows per CTA) when a bed's whole output fits 64 rows;
    // not on a member's last conv, whose fused head sums keep the single-CTA grouping
    static const int half_on = getenv("HB_K4_HALF") ? atoi(getenv("HB_K4_HALF")) : 1;
    a.half = (half_on && a.pair && fc_w == nullptr && a.out_rows <= kBM / 2) ? 1 : 0;
    if (a.half) a.stride_m = kBM / 2;
  }
  const int ksteps = (a.ck >= 16) ? a.ck / a.fold : 8;
  a.mt_per_p = (a.out_rows + a.stride_m - 1) / a.stride_m;
  a.num_tiles = a.n_ntiles * P * a.mt_per_p;
  a.a_stage_bytes = static_cast<uint32_t>(stride * (a.ck / 8) * a.rows * 16);
  a.b_chunk_bytes = static_cast<uint32_t>(ksteps * 2 * a.bnp * 16);
  a.sb_len = (a.n_ntiles == 1 && G * a.bn <= kSmemBiasMax) ? G * a.bn : 0;
  const uint32_t fixed = 1024 + 256 + 2 * static_cast<uint32_t>(a.sb_len) * 4 + (a.fold > 1 ? kXchBytes : 0);
  const uint32_t budget = kSmemLimit - fixed;
  const uint32_t b_all = a.b_chunk_bytes * a.n_kchunks;
  a.b_resident = resident;
  a.b_slot_bytes = a.pair ? a.b_chunk_bytes / 2 : a.b_chunk_bytes;
  a.mtp_per_p = (Pm * a.mt_per_p + 1) / 2;               // pairs per (member, N tile)
  if (a.pair) a.num_tiles = G * a.n_ntiles * a.mtp_per_p;  // M-tile pairs
  a.nb_slots = resident ? a.n_kchunks : 2;
  if (!resident) {
    // Streamed weights (the wide layers): a k-chunk's B image (up to 64 KB) is
    // consumed in ~1k MMA cycles, less than one image takes to arrive from L2,
    // so every extra slot that fits next to 3 A stages is another image in
    // flight (HB_K4_BSLOTS caps it; 2 = the old double buffer).
    const int cap = getenv("HB_K4_BSLOTS") ? atoi(getenv("HB_K4_BSLOTS")) : (a.pair ? 8 : 4);
    while (a.nb_slots < cap && (a.nb_slots + 1) * a.b_slot_bytes + 3 * a.a_stage_bytes <= budget) ++a.nb_slots;
  }
  const uint32_t b_smem = resident ? b_all : a.nb_slots * a.b_slot_bytes;
  a.na_stages = static_cast<int>((budget - b_smem) / a.a_stage_bytes);
  const int dbg = getenv("HB_DEBUG") ? atoi(getenv("HB_DEBUG")) : 0;
  const int max_stages = (dbg & 2) ? 8 : (dbg & 4) ? 12 : 4;
  if (a.na_stages > max_stages) a.na_stages = max_stages;
  if (a.na_stages < 2) return "conv: k-chunk does not fit in shared memory";
  uint32_t cols = 32;
  while (cols < static_cast<uint32_t>(a.half ? a.bnp : 2 * a.bnp)) cols <<= 1;
  a.tmem_cols = cols;
  a.wpack = wpack;
  a.wpack_stride = wpack_bytes(cin, cout);
  a.bias = bias;
  a.bias_stride = static_cast<int>(bias_len(cout));
  a.out = out;
  a.res = res;
  a.res_mode = res ? res_mode : 0;
  a.res_c = res_c;
  a.res_qs = res ? ilog2(res_q) : 0;
  a.res_lq = res ? lq_Q(res_len, res_q) : 0;
  if (a.res && a.res_mode == 2 && act_rows_q(res_len, res_q) < 2 * lout)
    return "conv: maxpool shortcut shorter than the output";
  a.relu = 1;
  a.fc_w = fc_w;
  a.head_out = head_out;
  a.head_g_stride = head_g_stride ? head_g_stride : static_cast<size_t>(Pm) * a.n_ntiles * a.mt_per_p;
  a.dbg = dbg;
  plan->smem_bytes = a.nb_slots * a.b_slot_bytes + a.na_stages * a.a_stage_bytes + fixed;
  plan->grid = a.num_tiles < num_sms ? a.num_tiles : num_sms;
  if (a.pair) plan->grid = 2 * std::max(1, std::min(a.num_tiles, num_sms / 2));  // clusters of two CTAs

  EncodeTiledFn enc = get_encode();
  if (!enc) return "conv: cuTensorMapEncodeTiled unavailable";
  const cuuint64_t CG = static_cast<cuuint64_t>(cin / 8);
  const cuuint32_t estr[5] = {1, 1, 1, 1, 1};
  CUresult rc;
  if (stride == 1) {  // I layout: [P][G][lp][8] as {64 elems = 8 rows, lp/8 lines, G, P}
    const cuuint64_t lp = static_cast<cuuint64_t>(lp_I(lin));
    const cuuint64_t dims[4] = {64, lp / 8, CG, static_cast<cuuint64_t>(P)};
    const cuuint64_t strides[3] = {128, lp * 16, CG * lp * 16};
    const cuuint32_t box[4] = {64, static_cast<cuuint32_t>(a.rows / 8), static_cast<cuuint32_t>(a.ck / 8), 1};
    rc = enc(&plan->tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 4, const_cast<__half*>(in), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  } else {  // S layout: [P][G][2][lh][8] as {64, lh/8 lines, 2 parities, G, P}
    const cuuint64_t lh = static_cast<cuuint64_t>(lh_S(lin));
    const cuuint64_t dims[5] = {64, lh / 8, 2, CG, static_cast<cuuint64_t>(P)};
    const cuuint64_t strides[4] = {128, lh * 16, 2 * lh * 16, CG * 2 * lh * 16};
    const cuuint32_t box[5] = {64, static_cast<cuuint32_t>(a.rows / 8), 1, static_cast<cuuint32_t>(a.ck / 8), 1};
    rc = enc(&plan->tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 5, const_cast<__half*>(in), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
  if (rc != CUDA_SUCCESS) return "conv: cuTensorMapEncodeTiled rejected the activation view";
  if (a.pair) {  // the group's packed weights as 128-B rows; one box = up to 256 rows of one CTA's half
    const cuuint64_t rows = static_cast<cuuint64_t>(G) * a.wpack_stride / 128;
    const int b_rows = static_cast<int>(a.b_slot_bytes / 128);
    const cuuint64_t dims[2] = {64, rows};
    const cuuint64_t strides[1] = {128};
    const cuuint32_t box[2] = {64, static_cast<cuuint32_t>(b_rows < 256 ? b_rows : 256)};
    rc = enc(&plan->tmapB, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<uint8_t*>(wpack), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (rc != CUDA_SUCCESS) return "conv: cuTensorMapEncodeTiled rejected the weight view";
  }
  return nullptr;
}

cudaError_t init_conv_kernel() {
  cudaError_t e =
      cudaFuncSetAttribute(conv_tc_kernel<1, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemLimit);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(conv_tc_kernel<2, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemLimit);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(conv_tc_kernel<1, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemLimit);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(conv_tc_kernel<1, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             kSmemLimit);
  return e;
}

cudaError_t launch_conv(const ConvPlan& plan, cudaStream_t st) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(plan.grid);
  cfg.blockDim = dim3(kConvThreads);
  cfg.dynamicSmemBytes = plan.smem_bytes;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  int na = 0;
  if (plan.args.pair) {
    attr[na].id = cudaLaunchAttributeClusterDimension;
    attr[na].val.clusterDim.x = 2;
    attr[na].val.clusterDim.y = 1;
    attr[na].val.clusterDim.z = 1;
    ++na;
  }
  if (pdl_enabled()) {
    attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  if (plan.args.pair && plan.args.half)
    return cudaLaunchKernelEx(&cfg, conv_tc_kernel<1, true, true>, plan.tmap, plan.tmapB, plan.args);
  if (plan.args.pair) return cudaLaunchKernelEx(&cfg, conv_tc_kernel<1, true>, plan.tmap, plan.tmapB, plan.args);
  if (plan.args.fold == 2) return cudaLaunchKernelEx(&cfg, conv_tc_kernel<2, false>, plan.tmap, plan.tmapB, plan.args);
  return cudaLaunchKernelEx(&cfg, conv_tc_kernel<1, false>, plan.tmap, plan.tmapB, plan.args);
}

}  // namespace hb
