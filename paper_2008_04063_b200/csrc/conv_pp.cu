// K4b: polyphase implicit-GEMM conv1d for narrow layers (C_out in {16, 32, 64},
// C_in in {16, 32, 64}; 16 taps, stride 1|2, "same" padding) on tcgen05, with
// bias / shortcut (identity or maxpool(2), zero-padded channels) / ReLU fused
// into the TMEM epilogue.
//
// Why a second conv kernel.  K4 (conv_tc.cu) puts 128 output positions on the
// UMMA M side and C_out on N.  For C_out = 32 every 128x32x16 MMA then reads a
// 4 KB A slice + 1 KB B slice from shared memory for 16 cycles of math: the
// layer runs at the shared-memory read rate (~45 cycles per MMA, 35-40 % of
// the tensor peak, profiles/r01_convbench.txt).  Here the roles swap and the
// M side is filled with output PHASES:
//
//   ph = 128 / C_out output phases, Q = stride * ph input phases,
//   Y[c, ph*n + p] = sum_{ci, t} W[c, ci, t] X[ci, Q*n + (stride*p + t) - pad]
//   D[(p', c), n]  = sum_{u, ci} A[(p', c), (u, ci)] B[n, (u, ci)]     (p' = ph-1-p)
//   A[(p', c), (u, ci)] = W[c, ci, u - stride*p]  (zero outside the 16 taps)
//   B[n, (u, ci)]       = X[ci, Q*n + u - pad],   u in [0, U), U = stride*(ph-1) + 16
//
// so one MMA is M=128 (all phases x all output channels) x N=nb (up to 256
// output columns) x K=16 (one shift u, 16 input channels): per 128x256x16 MMA
// the shared-memory traffic is 4 KB (A) + 8 KB (B) for 128 cycles of math.
// The zero taps cost U/16 - 1 of the MMA work (19/16 for C_out=32, s=1).
//
// Both operands are addressed without materialising anything:
//  * A: per (input-channel half, tap parity) the weights are stored as a
//    padded tap array [ph-1 zeros, taps, ph-1 zeros] of C_out x 16 B rows.
//    M row (p', c) of shift u is array entry (u - pi)/s + p' at row c, i.e.
//    the 128 rows of the A slice are 128 CONSECUTIVE 16-B rows starting at
//    entry (u - pi)/s: a canonical K-major no-swizzle tile (SBO = 128 B)
//    whose start address slides by one tap per shift.  Resident in smem.
//  * B: the input is stored in the Q-phase layout (hb_kernels.cuh), so
//    position Q*n + v lives in phase plane v mod Q at row n + floor(v/Q):
//    for a fixed shift the N rows are consecutive 16-B rows of one phase
//    plane.  One TMA box per (tile, 16-channel pair) brings every phase of
//    the tile's row range; shift u is a descriptor offset.
//
// Roles (640 threads, 1 CTA/SM, persistent over tiles): warp 0 TMA producer,
// warp 1 MMA issuer, warp 2 TMEM allocator, warps 4-19 four epilogue
// warpgroups (two per TMEM accumulator, one per half of its columns).
// Epilogue thread r holds M row r = (p', c) for nb columns; an 8x8 register
// transpose by warp shuffles inside each 8-lane group turns that into 8
// channels x one position per lane, so the shortcut read and the output store
// are 16-byte rows.
//
// Shortcuts: an identity shortcut whose x is in this conv's own Q-phase
// layout (ph >= 4) is added by the tensor core -- x's tile arrives as extra
// B stages (second tensor map) and ph MMAs per 16 channels with A = a window
// of a ones-array (appended to the weight image) add x[c, ph*n + p] to
// D[(p', c), n].  Other shortcuts (maxpool, wider phases) are read by the
// epilogue.  A member's last conv writes no output: the epilogue folds
// mean-pool . FC into one partial per (tile, column half, warp).
#include <algorithm>
#include <functional>
#include <vector>

#include "hb_kernels.cuh"
#include "hb_ptx.cuh"

#include <cstdio>
#include <cstdlib>
#include <cstring>

namespace hb {

constexpr int kPPThreads = 640;  // warp 0 TMA, 1 MMA, 2 TMEM, 4-19 four epilogue warpgroups

struct PPTile {
  int g, p, nt;  // member of the group, global patient row [G*Pm], column tile
};
__device__ __forceinline__ PPTile pp_tile(const PPArgs& a, int tile) {
  const int per_g = a.Pm * a.nt_per_p;
  PPTile t;
  t.g = tile / per_g;
  int rem = tile - t.g * per_g;
  const int pl = rem / a.nt_per_p;
  t.nt = rem - pl * a.nt_per_p;
  t.p = t.g * a.Pm + pl;
  return t;
}

// Shortcut row load (HB_PP_DBG & 64: L2-only ld.global.cg instead of the
// read-only L1 path).
__device__ __forceinline__ uint4 ldres_sel(const uint4* p, bool cg) { return cg ? __ldcg(p) : __ldg(p); }

// This CTA's tiles: first, first + stride, ... < end.  Default: round robin
// over every tile of the group.  member_split: the CTAs are partitioned
// between the group's members in contiguous blocks, so a CTA never changes
// weight image (the planner enables it when it costs no extra wave).
struct CtaRange {
  int first, stride, end;
};
__device__ __forceinline__ CtaRange cta_range(const PPArgs& a) {
  CtaRange r{static_cast<int>(blockIdx.x), static_cast<int>(gridDim.x), a.num_tiles};
  if (a.member_split) {
    const int grid = static_cast<int>(gridDim.x), c = static_cast<int>(blockIdx.x);
    int g = 0;
    while (g + 1 < a.G && ((g + 1) * grid) / a.G <= c) ++g;
    const int lo = (g * grid) / a.G, hi = ((g + 1) * grid) / a.G;
    const int per_g = a.Pm * a.nt_per_p;
    r.first = g * per_g + (c - lo);
    r.stride = hi - lo;
    r.end = (g + 1) * per_g;
  }
  return r;
}

// MMAs of one staged 16-channel pair (or one shortcut pair), issued by the
// calling (elected) lane, then one commit to the stage's empty barrier.
// Descriptors advance on their low words only (the 14-bit start-address
// field; shared addresses never carry out of it): A by one tap-array entry per
// shift (stride 2: alternating parity arrays, w_par16 apart), B by one phase
// plane per shift and by one row, back to phase 0, when the phase wraps.  The
// issue loop is on the MMA's critical path (measured: one extra uniform
// instruction per MMA cost 6 % of the c2 tick), hence no per-MMA election,
// division or modulo.
__device__ __forceinline__ void pp_issue_pair(const PPArgs& a, uint32_t d_tmem, uint64_t a0, uint64_t b0,
                                              uint32_t idesc, bool first, uint64_t* empty_bar) {
  const uint64_t a_hi = a0 & 0xFFFFFFFF00000000ull, b_hi = b0 & 0xFFFFFFFF00000000ull;
  const int Q = a.Q, R = a.R, pad = a.pad;
  int q = (-pad) & (Q - 1);
  uint32_t b_lo = static_cast<uint32_t>(b0) + static_cast<uint32_t>(q * R + 8 + ((-pad) >> a.qs));
  const uint32_t b_wrap = static_cast<uint32_t>(1 - (Q - 1) * R), b_step = static_cast<uint32_t>(R);
  uint32_t a_lo = static_cast<uint32_t>(a0);
  const uint32_t a_step = static_cast<uint32_t>(a.cout);
  uint32_t acc = first ? 0u : 1u;
  auto adv_b = [&]() {
    if (q == Q - 1) {
      q = 0;
      b_lo += b_wrap;
    } else {
      ++q;
      b_lo += b_step;
    }
  };
  if (a.stride == 1) {
    for (int u = 0; u < a.U; ++u) {
      mma_f16_ss(d_tmem, a_hi | a_lo, b_hi | b_lo, idesc, acc);
      acc = 1u;
      a_lo += a_step;
      adv_b();
    }
  } else {  // U even: shift u uses parity u & 1, entry u >> 1
    const uint32_t par = a.w_par16;
    for (int u = 0; u < a.U; u += 2) {
      mma_f16_ss(d_tmem, a_hi | a_lo, b_hi | b_lo, idesc, acc);
      acc = 1u;
      adv_b();
      mma_f16_ss(d_tmem, a_hi | (a_lo + par), b_hi | b_lo, idesc, 1u);
      adv_b();
      a_lo += a_step;
    }
  }
  mma_commit(empty_bar);
}

// One tile's epilogue for the calling warpgroup (one half of the tile's
// columns): TMEM -> + bias -> fp16 -> 8x8 register transpose -> + shortcut,
// ReLU -> 16-B row stores, or (a member's last conv) the fused mean-pool . FC
// partial.  After the transpose, lane (M row (p', c), column octet r8) covers
// positions l = l0 + h * step, h = 2 * chunk + b, step = 8 * ph; every Q-phase
// layout involved has Q | step (Q <= 32, checked by the planner), so each load
// and store address is a per-tile base + h * a constant and the bounds checks
// are h < h_valid (l < lout) / h < h_rows (l < out_rows).  The per-chunk work
// is then the TMEM load, bias, conversion, transpose and shortcut math only --
// the 64-bit Q-phase address arithmetic per access made the epilogue
// instruction-issue bound (~275 SASS per chunk, as many issue cycles as the
// MMAs of the tile at 32 channels).
// kLateRes: read the shortcut only after the accumulator wait (K4c: the rows
// are written inside the same launch); otherwise the first two chunks' rows
// are requested before it.  Returns after arriving on acc_empty.
template <bool kLateRes, int kParts>
__device__ __forceinline__ void pp_epi_tile(const PPArgs& a, const PPTile& t, int ew, int wq, int lane,
                                            uint32_t taddr, uint64_t* acc_full, uint32_t accph,
                                            uint64_t* acc_empty, float bias, bool cg, bool skip_math) {
  const int cout = a.cout, ph = a.ph;
  const int row = wq * 32 + lane;  // M row = (p', c)
  const int lc = __ffs(cout) - 1;
  const int c = row & (cout - 1);
  const int phase = ph - 1 - (row >> lc);
  const int g8 = c >> 3;
  const int r8 = lane & 7;
  // 16-column chunks; this warpgroup drains part `ew` of kParts (the first parts the larger).  The
  // fused head writes one partial per QUARTER of the columns whatever kParts is (a part of a half
  // split covers two quarters), so the fp32 grouping of a bed's head sum is the same in K4b
  // (quarters) and K4c (halves): both paths stay bit-identical.
  const int nch = a.nb >> 4;
  const int c_lo = (ew * nch + kParts - 1) / kParts, c_hi = ((ew + 1) * nch + kParts - 1) / kParts;
  constexpr int kQ = kHeadParts / kParts;  // head quarters per part
  const int q0 = ew * kQ;                  // first quarter of this part
  const int step = 8 * ph;
  const int l0 = ph * (t.nt * a.nb + r8) + phase;
  const int h_valid = l0 < a.lout ? (a.lout - l0 + step - 1) / step : 0;
  const int h_rows = l0 < a.out_rows ? (a.out_rows - l0 + step - 1) / step : 0;
  const int res_mode = a.res_mode;
  const bool has_res = res_mode != 0 && g8 * 8 < a.res_c;
  const __half* r0p = a.res;
  const __half* r1p = a.res;
  int r_inc = 0;
  if (has_res) {
    const size_t res_plane = static_cast<size_t>(t.p) * (a.res_c >> 3) + g8;
    if (res_mode == 2) {
      r0p = a.res + q_off(res_plane, a.res_qs, a.res_lq, 2 * l0);
      r1p = a.res + q_off(res_plane, a.res_qs, a.res_lq, 2 * l0 + 1);
      r_inc = ((2 * step) >> a.res_qs) * 8;
    } else {
      r0p = a.res + q_off(res_plane, a.res_qs, a.res_lq, l0);
      r_inc = (step >> a.res_qs) * 8;
    }
  }
  const float* fcw = a.fc_w;
  __half* outp = fcw ? nullptr : a.out + q_off(static_cast<size_t>(t.p) * (cout >> 3) + g8, a.out_qs, a.out_lq, l0);
  const int o_inc = (step >> a.out_qs) * 8;
  float head0 = 0.f, head1 = 0.f;  // quarter q0 (and q0 + 1 when a part spans two quarters)
  const int q_split = ((q0 + 1) * nch + kHeadParts - 1) / kHeadParts;  // first chunk of quarter q0 + 1
  float fc8[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) fc8[q] = fcw ? __ldg(fcw + static_cast<size_t>(t.g) * cout + g8 * 8 + q) : 0.f;
  // Shortcut rows (2 positions per lane and chunk; maxpool reads 2 rows each)
  // are loaded two chunks ahead through two register sets (the chunk loop is
  // unrolled by two so both stay in registers).
  uint4 rawA[4], rawB[4];
  auto ld = [&](const __half* p) {
    return cg ? __ldcg(reinterpret_cast<const uint4*>(p)) : __ldg(reinterpret_cast<const uint4*>(p));
  };
  auto load_res = [&](int ch, uint4 (&raw)[4]) {
#pragma unroll
    for (int b = 0; b < 2; ++b) {
      const int h = 2 * ch + b;
      const bool ok = has_res && h < h_valid;
      const uint4 z = make_uint4(0u, 0u, 0u, 0u);
      raw[2 * b] = ok ? ld(r0p + h * r_inc) : z;
      if (res_mode == 2) raw[2 * b + 1] = ok ? ld(r1p + h * r_inc) : z;
    }
  };
  if (!kLateRes && res_mode) {
    load_res(c_lo, rawA);
    if (c_lo + 1 < c_hi) load_res(c_lo + 1, rawB);
  }
  mbar_wait(acc_full, accph, 120);
  tc_fence_after();
  if (kLateRes && res_mode) {
    load_res(c_lo, rawA);
    if (c_lo + 1 < c_hi) load_res(c_lo + 1, rawB);
  }
  auto chunk = [&](int ch, uint4 (&raw)[4]) {
    uint32_t r[16];
    tmem_ld16_nw(taddr + static_cast<uint32_t>(ch * 16), r);
    uint4 rv[2];
#pragma unroll
    for (int b = 0; b < 2; ++b) {
      if (res_mode == 2) {
        const __half2* h0 = reinterpret_cast<const __half2*>(&raw[2 * b]);
        const __half2* h1 = reinterpret_cast<const __half2*>(&raw[2 * b + 1]);
        __half2* o2 = reinterpret_cast<__half2*>(&rv[b]);
#pragma unroll
        for (int q = 0; q < 4; ++q) o2[q] = __hmax2_nan(h0[q], h1[q]);
      } else {
        rv[b] = res_mode ? raw[2 * b] : make_uint4(0u, 0u, 0u, 0u);
      }
    }
    if (res_mode && ch + 2 < c_hi) load_res(ch + 2, raw);
    tmem_wait_ld();
    if (ch == c_hi - 1) {  // this warpgroup's columns drained (a part is never empty: nb >= 64)
      tc_fence_before();
      mbar_arrive(acc_empty);
    }
    if (skip_math) return;
    // (acc + bias) is rounded to fp16 before the transpose; the shortcut add
    // and ReLU run on half2 (two roundings instead of one: within one fp16 ulp
    // of the fp32 reference, tests/test_conv_pp_gpu.py).
#pragma unroll
    for (int b = 0; b < 2; ++b) {
      const int h = 2 * ch + b;
      uint32_t hv[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const __half2 v2 = __floats2half2_rn(__uint_as_float(r[8 * b + 2 * q]) + bias,
                                             __uint_as_float(r[8 * b + 2 * q + 1]) + bias);
        hv[q] = *reinterpret_cast<const uint32_t*>(&v2);
      }
      transpose8_h2(hv, r8);
      if (h < h_rows) {
        const __half2* rr = reinterpret_cast<const __half2*>(&rv[b]);
        const __half2 zero = __float2half2_rn(0.f);
        const bool valid = h < h_valid;
        uint4 pk;
        __half2* o2 = reinterpret_cast<__half2*>(&pk);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const __half2 y = __hmax2_nan(__hadd2(*reinterpret_cast<const __half2*>(&hv[q]), rr[q]), zero);
          o2[q] = valid ? y : zero;
        }
        if (outp != nullptr) {
          *reinterpret_cast<uint4*>(outp + h * o_inc) = pk;
        } else if (valid) {  // fused head: this position's 8 channels . fc
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const float2 f = __half22float2(o2[q]);
            if (kQ > 1 && ch >= q_split)
              head1 = fmaf(f.x, fc8[2 * q], fmaf(f.y, fc8[2 * q + 1], head1));
            else
              head0 = fmaf(f.x, fc8[2 * q], fmaf(f.y, fc8[2 * q + 1], head0));
          }
        }
      }
    }
  };
  for (int ch = c_lo; ch < c_hi; ch += 2) {
    chunk(ch, rawA);
    if (ch + 1 < c_hi) chunk(ch + 1, rawB);
  }
  if (fcw != nullptr) {  // one partial per (tile, epilogue warp), summed in fixed order by K5
#pragma unroll
#pragma unroll
    for (int i = 0; i < kQ; ++i) {
      float hv = i == 0 ? head0 : head1;
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) hv += __shfl_xor_sync(0xffffffffu, hv, off);
      if (lane == 0)
        a.head_out[static_cast<size_t>(t.g) * a.head_g_stride + static_cast<size_t>(t.p - t.g * a.Pm) * a.head_mt +
                   static_cast<size_t>(t.nt) * (4 * kHeadParts) + (q0 + i) * 4 + wq] = hv;  // (column quarter, warp)
    }
  }
}

__global__ void __launch_bounds__(kPPThreads, 1)
    conv_pp_kernel(const __grid_constant__ CUtensorMap tmB, const __grid_constant__ CUtensorMap tmX,
                   const __grid_constant__ PPArgs a) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sW = smem;
  uint8_t* sB = smem + a.w_bytes;
  uint64_t* st_full = reinterpret_cast<uint64_t*>(sB + static_cast<size_t>(a.n_stages) * a.stage_bytes);
  uint64_t* st_empty = st_full + a.n_stages;
  uint64_t* w_full = st_empty + a.n_stages;
  uint64_t* w_empty = w_full + 1;
  uint64_t* acc_full = w_empty + 1;
  uint64_t* acc_empty = acc_full + 2;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(acc_empty + 2);
  float* s_bias = reinterpret_cast<float*>(tmem_holder + 4);  // [G][cout]

  const uint32_t warp = warp_id();
  const uint32_t lane = lane_id();
  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tmB);
    if (a.n_res_pairs) prefetch_tmap(&tmX);
    for (int i = 0; i < a.n_stages; ++i) {
      mbar_init(&st_full[i], 1);
      mbar_init(&st_empty[i], 1);
    }
    mbar_init(w_full, 1);
    mbar_init(w_empty, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&acc_full[i], 1);
      mbar_init(&acc_empty[i], 128 * kEpiPartsPP);  // every epilogue warpgroup drains its part of every tile
    }
    fence_barrier_init();
    // the first weight image (immutable, so before the dependency wait) goes out
    // right behind the barrier init: its latency hides the rest of the prologue
    const CtaRange cr = cta_range(a);
    if (cr.first < cr.end) {
      const uint8_t* src = a.wimg + static_cast<size_t>(pp_tile(a, cr.first).g) * a.w_stride;
      mbar_arrive_expect_tx(w_full, a.w_bytes);
      for (uint32_t off = 0; off < a.w_bytes; off += 32768u)
        bulk_load(sW + off, src + off, (a.w_bytes - off) < 32768u ? (a.w_bytes - off) : 32768u, w_full);
    }
  }
  if (warp == 2) tmem_alloc(tmem_holder, a.tmem_cols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;
  pdl_trigger();

  if (warp == 0) {
    if (lane == 0) {
      // -------------------------------------------------------------- producer
      auto load_w = [&](int g) {
        const uint8_t* src = a.wimg + static_cast<size_t>(g) * a.w_stride;
        mbar_arrive_expect_tx(w_full, a.w_bytes);
        for (uint32_t off = 0; off < a.w_bytes; off += 32768u) {
          const uint32_t n = (a.w_bytes - off) < 32768u ? (a.w_bytes - off) : 32768u;
          bulk_load(sW + off, src + off, n, w_full);
        }
      };
      const CtaRange cr = cta_range(a);
      int loaded_g = cr.first < cr.end ? pp_tile(a, cr.first).g : -1, reloads = 0;
      pdl_wait();
      int st = 0;
      uint32_t sph = 0;
      const int planes_per_p = a.cin / 8;
      for (int tile = cr.first; tile < cr.end; tile += cr.stride) {
        const PPTile t = pp_tile(a, tile);
        if (t.g != loaded_g) {  // next member of the group: wait until the MMAs on the old weights retired
          mbar_wait(w_empty, static_cast<uint32_t>(reloads++) & 1u, 101);
          load_w(t.g);
          loaded_g = t.g;
        }
        const int line0 = t.nt * (a.nb / 8) - 1;  // rows from n0 - 8
        for (int j = 0; j < a.n_pairs + a.n_res_pairs; ++j) {
          mbar_wait(&st_empty[st], sph ^ 1u, 102);
          if (a.dbg & 4) {
            mbar_arrive(&st_full[st]);
          } else {
            mbar_arrive_expect_tx(&st_full[st], a.stage_bytes);
            if (j < a.n_pairs)
              tma_load_4d(sB + static_cast<size_t>(st) * a.stage_bytes, &tmB, &st_full[st], 0, line0, 0,
                          t.p * planes_per_p + 2 * j);
            else  // the identity shortcut's rows, same box geometry (x is in this conv's Q-phase layout)
              tma_load_4d(sB + static_cast<size_t>(st) * a.stage_bytes, &tmX, &st_full[st], 0, line0, 0,
                          t.p * (a.res_c / 8) + 2 * (j - a.n_pairs));
          }
          if (++st == a.n_stages) {
            st = 0;
            sph ^= 1u;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------------- MMA issuer
    const uint32_t idesc = make_idesc_f16(kBM, a.nb);
    const uint32_t b_lbo = static_cast<uint32_t>(a.Q * a.R * 16);
    int st = 0;
    uint32_t sph = 0;
    int acc = 0;
    uint32_t accph = 0;
    uint32_t wph = 0;
    const CtaRange cr = cta_range(a);
    int cur_g = cr.first < cr.end ? pp_tile(a, cr.first).g : 0;
    const bool prof = (a.dbg & 16) && a.prof && lane == 0;
    unsigned long long c_acc = 0, c_b = 0, c_start = prof ? clock64() : 0;
    for (int tile = cr.first; tile < cr.end; tile += cr.stride) {
      const PPTile t = pp_tile(a, tile);
      if (t.g != cur_g) {
        wph ^= 1u;
        cur_g = t.g;
      }
      mbar_wait(w_full, wph, 111);
      unsigned long long t0 = prof ? clock64() : 0;
      mbar_wait(&acc_empty[acc], accph ^ 1u, 112);
      if (prof) {
        const unsigned long long t1 = clock64();
        c_acc += t1 - t0;
      }
      tc_fence_after();
      const uint32_t d_tmem = tmem_base + static_cast<uint32_t>(acc * a.nb);
      for (int j = 0; j < a.n_pairs + a.n_res_pairs; ++j) {
        if (prof) t0 = clock64();
        mbar_wait(&st_full[st], sph, 113);
        if (prof) {
          const unsigned long long t1 = clock64();
          c_b += t1 - t0;
        }
        tc_fence_after();
        const uint64_t b0 = make_desc(smem_u32(sB + static_cast<size_t>(st) * a.stage_bytes), b_lbo, 128);
        if (elect_one()) {
          if (a.dbg & 2) {
            mma_commit(&st_empty[st]);
          } else if (j >= a.n_pairs) {
            // identity shortcut on the tensor core: D[(p', c), n] += x[c, ph*n + p] as one K=16 MMA per
            // phase p, A = the phase-p window of the selection array Z (ones at (p', c) -> channel c)
            const uint64_t z0 = make_desc(smem_u32(sW) + a.z_off + static_cast<uint32_t>(j - a.n_pairs) * a.z_pair_bytes,
                                          a.z_half_bytes, 128);
            for (int ps = 0; ps < a.ph; ++ps)
              mma_f16_ss(d_tmem, z0 + static_cast<uint32_t>(ps * a.cout), b0 + static_cast<uint32_t>(ps * a.R + 8),
                         idesc, 1u);
            mma_commit(&st_empty[st]);
          } else {
            const uint64_t a0 = make_desc(smem_u32(sW) + static_cast<uint32_t>(j) * a.w_pair_bytes, a.w_half_bytes, 128);
            pp_issue_pair(a, d_tmem, a0, b0, idesc, j == 0, &st_empty[st]);
          }
        }
        __syncwarp();
        if (++st == a.n_stages) {
          st = 0;
          sph ^= 1u;
        }
      }
      if (elect_one()) mma_commit(&acc_full[acc]);
      __syncwarp();
      const int nxt = tile + cr.stride;
      if (nxt < cr.end && pp_tile(a, nxt).g != t.g) {  // the weights change after this tile
        if (elect_one()) mma_commit(w_empty);
        __syncwarp();
      }
      if (++acc == 2) {
        acc = 0;
        accph ^= 1u;
      }
    }
    if (prof) {
      a.prof[blockIdx.x * 8 + 0] = c_acc;
      a.prof[blockIdx.x * 8 + 1] = c_b;
      a.prof[blockIdx.x * 8 + 2] = clock64() - c_start;
    }
  } else if (warp >= 4) {
    // ------------------------------------------------------------------ epilogue
    // Four warpgroups, each drains one quarter of every tile's columns (part
    // ew).  The accumulator is held while its columns are drained and the MMA
    // of tile k+2 waits for the epilogue of tile k: splitting each tile over
    // all four warpgroups (instead of two per buffer, alternate tiles) halves
    // that hold time; the total epilogue work is the same.
    const int ew = (static_cast<int>(warp) - 4) >> 2;
    const int wq = static_cast<int>(warp) & 3;
    const int c = (wq * 32 + static_cast<int>(lane)) & (a.cout - 1);
    for (int i = static_cast<int>(threadIdx.x) - 128; i < a.G * a.cout; i += kPPThreads - 128) {
      const int g = i / a.cout;
      s_bias[i] = a.bias[static_cast<size_t>(g) * a.bias_stride + (i - g * a.cout)];
    }
    named_bar_sync(1, kPPThreads - 128);  // the epilogue warps alone: off the producer's path
    pdl_wait();
    const CtaRange cr = cta_range(a);
    int k = 0;
    for (int tile = cr.first; tile < cr.end; tile += cr.stride, ++k) {
      const PPTile t = pp_tile(a, tile);
      const int eb = k & 1;  // the accumulator the MMA used for this tile
      const uint32_t taddr = tmem_base + (static_cast<uint32_t>(wq * 32) << 16) + static_cast<uint32_t>(eb * a.nb);
      pp_epi_tile<false, kEpiPartsPP>(a, t, ew, wq, static_cast<int>(lane), taddr, &acc_full[eb], static_cast<uint32_t>(k >> 1) & 1u,
                         &acc_empty[eb], s_bias[t.g * a.cout + c], (a.dbg & 64) != 0, (a.dbg & 1) != 0);
    }
  }

  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_dealloc(tmem_base, a.tmem_cols);
}

// ------------------------------------------------------------------ K4c: chain
// A whole member-group chain of K4b layers (and several chains side by side)
// in ONE persistent launch.  Every CTA walks its own list of (layer, tile)
// items, layer-major; a tile of layer j starts as soon as the tiles of its
// producer layers that cover its input rows (and shortcut rows) are written,
// tracked by per-tile counters in global memory, instead of at a grid-wide
// kernel boundary.  Per item the three roles are those of conv_pp_kernel;
// what changes:
//  * the layer descriptors live in the parameter block (ChainArgs::L, read
//    with uniform constant-bank loads) and the tensor maps in global memory;
//  * the weight image is reloaded when the (layer, member) of the next item
//    differs (MMA -> producer handshake w_empty / w_full, as a group change in
//    conv_pp_kernel); the stage ring restarts at slot 0 there because the
//    stage region begins right after the new image, and per-slot barrier
//    phases are tracked as bit masks so a layer with fewer or more stages
//    keeps both roles in step;
//  * accumulators sit at fixed TMEM offsets (0 / 256), bias and FC weights
//    are read from global (L1) per tile;
//  * after its stores, each column half of a tile publishes itself: named
//    barrier of its warpgroup, proxy fence, release add of 1 to the tile's
//    counter.  The producer thread acquires every counter its next TMA boxes
//    depend on (target 2 * (epoch + 1): counters only grow, `epoch` counts
//    finished launches of this chain, bumped by the last CTA to exit), then
//    issues a proxy fence and the loads.  The epilogue's shortcut rows are
//    read through L2 (ld.global.cg): they are written inside this launch;
//  * (ChainArgs::agg) the ensemble aggregation runs inside the launch: each
//    half of a member's last-conv tile counts itself on a per-bed counter
//    after its head partials are stored, and warp 3 (otherwise idle) of CTA
//    p mod grid waits for bed p's count and sums the bed's partials in K5's
//    order (bit-identical to the separate aggregate kernel).
// Deadlock freedom: each CTA's list is sorted by layer and a layer only waits
// on lower layers, so by induction on the layer index every item completes
// (the grid is at most one CTA per SM, all resident); the aggregation only
// waits on head tiles, which by the same induction all complete.
__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ uint32_t ld_acquire_u32(const unsigned* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_release_add_u32(unsigned* p, uint32_t v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

// K5's aggregation of one bed, by one warp, in K5's arithmetic order (per member: lane-strided
// partial sums, xor-shuffle reduction, fc bias; then the members left to right): the fused and the
// separate aggregation are bit-identical.  The partials were written by other CTAs in this launch
// (published through the bed counter's acquire): read through L2.
__device__ __forceinline__ void chain_aggregate_bed(const ChainArgs& ca, int bed /* global */, int lane) {
  const HeadMember* heads = static_cast<const HeadMember*>(ca.heads);
  const int M = ca.n_heads;
  float sp = 0.f, sl = 0.f;
  // members in batches of 8 whose partial loads are all in flight at once (a bed's partials sit in
  // L2: one round trip per batch instead of one per member); up to 64 partials per member a lane
  // holds its (at most two) terms of K5's strided sum, added in K5's order
  for (int m0 = 0; m0 < M; m0 += 8) {
    const int nm = M - m0 < 8 ? M - m0 : 8;
    HeadMember hm[8];
    float va[8], vb[8];
    bool small = true;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      if (k < nm) {
        hm[k] = heads[m0 + k];
        small = small && hm[k].mt <= 64;
      }
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      va[k] = vb[k] = 0.f;
      if (small && k < nm) {
        const float* src = hm[k].partial + static_cast<size_t>(bed) * hm[k].mt;
        if (lane < hm[k].mt) va[k] = __ldcg(src + lane);
        if (lane + 32 < hm[k].mt) vb[k] = __ldcg(src + lane + 32);
      }
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      if (k >= nm) break;
      float s = 0.f;
      if (small) {
        if (lane < hm[k].mt) s += va[k];
        if (lane + 32 < hm[k].mt) s += vb[k];
      } else {
        const float* src = hm[k].partial + static_cast<size_t>(bed) * hm[k].mt;
        for (int i = lane; i < hm[k].mt; i += 32) s += __ldcg(src + i);
      }
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
      const float lg = hm[k].fc_b + s * hm[k].inv_len;
      if (lane == 0) {
        ca.member_logits[static_cast<size_t>(bed) * M + m0 + k] = lg;
        sp += 1.f / (1.f + expf(-lg));
        sl += lg;
      }
    }
  }
  if (lane == 0) {
    ca.ens_prob[bed] = sp / static_cast<float>(M);
    ca.ens_logit[bed] = sl / static_cast<float>(M);
    ca.ens_sums[bed] = sp;
    ca.ens_sums[ca.P + bed] = sl;
  }
}

// Wait until the counters [a0, a1) and [b0, b1) (at most kMaxRange each) reached
// `target`: all read in one batch of independent acquire loads (one L2 round
// trip), registers only, re-polled with a short sleep while any is short.
constexpr int kMaxRange = 6;
__device__ __forceinline__ void chain_wait_ranges(const unsigned* flags, int a0, int a1, int b0, int b1,
                                                  uint32_t target) {
  uint32_t spins = 0;
  while (true) {
    uint32_t va[kMaxRange], vb[kMaxRange];
#pragma unroll
    for (int k = 0; k < kMaxRange; ++k) va[k] = a0 + k < a1 ? ld_acquire_u32(flags + a0 + k) : target;
#pragma unroll
    for (int k = 0; k < kMaxRange; ++k) vb[k] = b0 + k < b1 ? ld_acquire_u32(flags + b0 + k) : target;
    bool ok = true;
#pragma unroll
    for (int k = 0; k < kMaxRange; ++k) ok = ok && static_cast<int>(va[k] - target) >= 0 && static_cast<int>(vb[k] - target) >= 0;
    if (ok) return;
    __nanosleep(64);
    if (++spins == (1u << 26)) asm volatile("trap;");  // a dependency that never lands is a planning bug
  }
}

__global__ void __launch_bounds__(kPPThreads, 1) chain_pp_kernel(const __grid_constant__ ChainArgs ca) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* st_full = reinterpret_cast<uint64_t*>(smem);
  uint64_t* st_empty = st_full + kChainStages;
  uint64_t* w_full = st_empty + kChainStages;
  uint64_t* w_empty = w_full + 1;
  uint64_t* acc_full = w_empty + 1;
  uint64_t* acc_empty = acc_full + 2;
  uint64_t* it_full = acc_empty + 2;       // item ring: producer -> MMA + epilogue
  uint64_t* it_empty = it_full + kChainRing;
  uint64_t* it_ready = it_empty + kChainRing;  // the item's dependencies are met (its shortcut rows are readable)
  int* ring = reinterpret_cast<int*>(it_ready + kChainRing);
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(ring + kChainRing);
  uint8_t* const sW = smem + kChainFixed;  // weight image, then the stage ring

  const uint32_t warp = warp_id();
  const uint32_t lane = lane_id();
  // Queue item gi: idesc[gi] = {(layer << 22) | tile, bed row p, column tile nt, member g}
  // (decoded on the host: this role's thread shares its sub-partition with four busy
  // epilogue warps, so every instruction on its path is dear)
  auto item_key = [&](int gi) {  // (layer, member): the weight image the item needs
    const int4 d = __ldg(ca.idesc + gi);
    return (d.x >> 22) * kMaxGroup + d.w;
  };
  auto load_w = [&](int key) {
    const int li = key / kMaxGroup, g = key - li * kMaxGroup;
    const PPArgs& a = ca.L[li];
    const uint8_t* src = a.wimg + static_cast<size_t>(g) * a.w_stride;
    mbar_arrive_expect_tx(w_full, a.w_bytes);
    for (uint32_t off = 0; off < a.w_bytes; off += 32768u)
      bulk_load(sW + off, src + off, (a.w_bytes - off) < 32768u ? (a.w_bytes - off) : 32768u, w_full);
  };
  // Next item of this CTA: its home chain's queue first, then (work stealing
  // once that is drained) the other chains' queues in turn; -1 = all drained.
  // The queue-head atomic is issued one item ahead (pull_issue) and resolved
  // when the item is needed (pull_take), so its L2 round trip overlaps the
  // current item's work instead of sitting on the producer's path.
  int chain = ca.home[blockIdx.x], visited = 0;
  int q_lo = ca.queue_off[chain], q_n = ca.queue_off[chain + 1] - q_lo;  // the current queue's bounds
  unsigned pend = 0;
  auto pull_issue = [&]() { pend = atomicAdd(ca.ctr + chain, 1u); };
  // returns the item's global queue index (idesc[gi] describes it), -1 when drained
  auto pull_take = [&]() -> int {
    while (visited < ca.n_chains) {
      if (static_cast<int>(pend) < q_n) return q_lo + static_cast<int>(pend);
      chain = chain + 1 == ca.n_chains ? 0 : chain + 1;
      q_lo = ca.queue_off[chain];
      q_n = ca.queue_off[chain + 1] - q_lo;
      if (++visited < ca.n_chains) pull_issue();
    }
    return -1;
  };
  auto pull = [&]() -> int {
    pull_issue();
    return pull_take();
  };
  int first = -1;
  if (warp == 0 && lane == 0) {
    for (int i = 0; i < kChainStages; ++i) {
      mbar_init(&st_full[i], 1);
      mbar_init(&st_empty[i], 1);
    }
    mbar_init(w_full, 1);
    mbar_init(w_empty, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&acc_full[i], 1);
      mbar_init(&acc_empty[i], 128 * kEpiPartsChain);  // the two warpgroups of that accumulator
    }
    for (int i = 0; i < kChainRing; ++i) {
      mbar_init(&it_full[i], 1);
      mbar_init(&it_empty[i], 1 + 128 * kEpiPartsChain);  // the MMA warp + the two epilogue warpgroups of that parity
      mbar_init(&it_ready[i], 1);
    }
    fence_barrier_init();
    first = pull();
    if (first >= 0) load_w(item_key(first));  // immutable: before the dependency wait
  }
  if (warp == 2) tmem_alloc(tmem_holder, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;

  if (warp == 0) {
    if (lane == 0) {
      // -------------------------------------------------------------- producer
      // with flagged stems every input of the launch is guarded by a tile counter: no
      // whole-grid wait on the stem launch (its CTAs are all resident: PDL launched us)
      if (!ca.stems_flagged) pdl_wait();
      const bool prof = ca.prof != nullptr;
      unsigned long long p_dep = 0, p_w = 0, p_st = 0, p_start = prof ? clock64() : 0;
      // counters grow by kEpiPartsChain per launch for a chain layer's tile (one per epilogue part), by 2
      // for a stem tile (two column halves)
      const uint32_t epoch1 = *reinterpret_cast<volatile unsigned*>(ca.sync) + 1u;
      const uint32_t target = static_cast<uint32_t>(kEpiPartsChain) * epoch1, target_stem = 2u * epoch1;
      int cur_key = first >= 0 ? item_key(first) : -1, reloads = 0;
      int st = 0;
      uint32_t empty_ph = 0;  // per stage slot: parity of its uses so far
      int gi = first, seq = 0;
      unsigned long long* trace = ca.trace;
      auto publish = [&](int value, int sq) {
        const int slot = sq & (kChainRing - 1);
        mbar_wait(&it_empty[slot], ((sq / kChainRing) & 1) ^ 1u, 200);
        ring[slot] = value;
        mbar_arrive(&it_full[slot]);
      };
      for (;; ++seq) {
        if (seq > 0) gi = pull_take();
        if (gi >= 0) pull_issue();  // the following item's queue head, resolved next iteration
        publish(gi, seq);
        if (gi < 0) {  // a second end mark for the other epilogue parity
          publish(-1, seq + 1);
          break;
        }
        if (trace) trace[5 * gi + 0] = globaltimer();
        const int4 dsc = __ldg(ca.idesc + gi);
        const int li = dsc.x >> 22;
        const PPArgs& a = ca.L[li];
        PPTile t;
        t.p = dsc.y;
        t.nt = dsc.z;
        t.g = dsc.w;
        const int key = li * kMaxGroup + t.g;
        unsigned long long q0 = prof ? clock64() : 0;
        if (key != cur_key) {  // next (layer, member): wait until the MMAs on the old image retired
          // (w_empty is committed by the MMA warp once per image change, so its
          // phases cannot alias however far ahead this thread runs)
          mbar_wait(w_empty, static_cast<uint32_t>(reloads++) & 1u, 201);
          if (prof) {
            const unsigned long long q1 = clock64();
            p_w += q1 - q0;
            q0 = q1;
          }
          load_w(key);
          cur_key = key;
          st = 0;
        }
        if (trace) trace[5 * gi + 1] = globaltimer();
        const int line0 = t.nt * (a.nb / 8) - 1;  // rows from n0 - 8
        {  // counters of the producer tiles this item's TMA boxes read (ranges decoded on the host)
          const int4 dr = __ldg(ca.ideps + gi);
          const uint32_t t_in = ca.dep_in[li] == kChainDepStem ? target_stem : target;
          const uint32_t t_res = ca.dep_res[li] == kChainDepStem ? target_stem : target;
          if (t_in == t_res) {
            chain_wait_ranges(ca.flags, dr.x, dr.y, dr.z, dr.w, t_in);
          } else {
            chain_wait_ranges(ca.flags, dr.x, dr.y, 0, 0, t_in);
            chain_wait_ranges(ca.flags, dr.z, dr.w, 0, 0, t_res);
          }
        }
        if (trace) trace[5 * gi + 2] = globaltimer();
        if (!(ca.opts & 1)) fence_proxy_async_global();
        mbar_arrive(&it_ready[seq & (kChainRing - 1)]);  // the epilogue may now read this item's shortcut rows
        if (prof) {
          const unsigned long long q1 = clock64();
          p_dep += q1 - q0;
          q0 = q1;
        }
        const CUtensorMap* tmB = ca.tmaps + 2 * li;
        uint8_t* sB = sW + a.w_bytes;
        const int planes_per_p = a.cin / 8;
        for (int j = 0; j < a.n_pairs + a.n_res_pairs; ++j) {
          mbar_wait(&st_empty[st], ((empty_ph >> st) & 1u) ^ 1u, 202);
          if (prof) {
            const unsigned long long q1 = clock64();
            p_st += q1 - q0;
            q0 = q1;
          }
          empty_ph ^= 1u << st;
          mbar_arrive_expect_tx(&st_full[st], a.stage_bytes);
          if (j < a.n_pairs)
            tma_load_4d(sB + static_cast<size_t>(st) * a.stage_bytes, tmB, &st_full[st], 0, line0, 0,
                        t.p * planes_per_p + 2 * j);
          else
            tma_load_4d(sB + static_cast<size_t>(st) * a.stage_bytes, tmB + 1, &st_full[st], 0, line0, 0,
                        t.p * (a.res_c / 8) + 2 * (j - a.n_pairs));
          if (++st == a.n_stages) st = 0;
        }
      }
      if (prof) {
        unsigned long long* pr = ca.prof + blockIdx.x * 16;
        pr[0] = p_dep;
        pr[1] = p_w;
        pr[2] = p_st;
        pr[3] = clock64() - p_start;
        pr[4] = static_cast<unsigned long long>(seq);
      }
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------------- MMA issuer
    int st = 0;
    uint32_t full_ph = 0;
    int acc = 0;
    uint32_t accph = 0;
    uint32_t wph = 0;
    int cur_key = -1;
    const bool prof = ca.prof != nullptr && lane == 0;
    unsigned long long m_w = 0, m_acc = 0, m_st = 0, m_start = prof ? clock64() : 0;
    auto read_item = [&](int sq) {
      const int slot = sq & (kChainRing - 1);
      mbar_wait(&it_full[slot], static_cast<uint32_t>(sq / kChainRing) & 1u, 210);
      const int v = ring[slot];
      __syncwarp();
      if (elect_one()) mbar_arrive(&it_empty[slot]);
      return v;
    };
    int gi = read_item(0);
    for (int seq = 0; gi >= 0; ++seq) {
      const int4 dsc = __ldg(ca.idesc + gi);
      const int li = dsc.x >> 22;
      const PPArgs& a = ca.L[li];
      const int key = li * kMaxGroup + dsc.w;
      if (key != cur_key) {
        if (cur_key >= 0) wph ^= 1u;
        cur_key = key;
        st = 0;
      }
      unsigned long long q0 = prof ? clock64() : 0;
      mbar_wait(w_full, wph, 211);
      if (prof) {
        const unsigned long long q1 = clock64();
        m_w += q1 - q0;
        q0 = q1;
      }
      mbar_wait(&acc_empty[acc], accph ^ 1u, 212);
      if (prof) {
        const unsigned long long q1 = clock64();
        m_acc += q1 - q0;
      }
      tc_fence_after();
      const uint32_t idesc = make_idesc_f16(kBM, a.nb);
      const uint32_t b_lbo = static_cast<uint32_t>(a.Q * a.R * 16);
      const uint32_t d_tmem = tmem_base + static_cast<uint32_t>(acc * 256);
      const uint32_t sw = smem_u32(sW), sb = sw + a.w_bytes;
      for (int j = 0; j < a.n_pairs + a.n_res_pairs; ++j) {
        const unsigned long long q2 = prof ? clock64() : 0;
        mbar_wait(&st_full[st], (full_ph >> st) & 1u, 213);
        if (prof) m_st += clock64() - q2;
        full_ph ^= 1u << st;
        tc_fence_after();
        const uint64_t b0 = make_desc(sb + static_cast<uint32_t>(st) * a.stage_bytes, b_lbo, 128);
        if (elect_one()) {
          if (j >= a.n_pairs) {
            const uint64_t z0 = make_desc(sw + a.z_off + static_cast<uint32_t>(j - a.n_pairs) * a.z_pair_bytes,
                                          a.z_half_bytes, 128);
            for (int ps = 0; ps < a.ph; ++ps)
              mma_f16_ss(d_tmem, z0 + static_cast<uint32_t>(ps * a.cout), b0 + static_cast<uint32_t>(ps * a.R + 8),
                         idesc, 1u);
            mma_commit(&st_empty[st]);
          } else {
            const uint64_t a0 = make_desc(sw + static_cast<uint32_t>(j) * a.w_pair_bytes, a.w_half_bytes, 128);
            pp_issue_pair(a, d_tmem, a0, b0, idesc, j == 0, &st_empty[st]);
          }
        }
        __syncwarp();
        if (++st == a.n_stages) st = 0;
      }
      if (elect_one()) mma_commit(&acc_full[acc]);
      __syncwarp();
      // the next item (published before the producer's image wait): when it
      // needs another image, release this one once these MMAs retire
      const int nx = read_item(seq + 1);
      if (nx >= 0 && item_key(nx) != key) {
        if (elect_one()) mma_commit(w_empty);
        __syncwarp();
      }
      gi = nx;
      if (++acc == 2) {
        acc = 0;
        accph ^= 1u;
      }
    }
    if (prof) {
      unsigned long long* pr = ca.prof + blockIdx.x * 16;
      pr[5] = m_w;
      pr[6] = m_acc;
      pr[7] = m_st;
      pr[8] = clock64() - m_start;
    }
  } else if (warp == 3) {
    // ------------------------------------------------------------- aggregation
    // (fused K5) chunk beds blockIdx.x, + gridDim.x, ...: once a bed's head-tile halves are all counted
    // (bed_target per launch, counters never reset) its members' partials are summed and the
    // bed's outputs written.  Every CTA of the persistent grid is resident, so the wait ends.
    if (ca.agg) {
      if (!ca.stems_flagged) pdl_wait();
      const uint32_t target = ca.bed_target * (*reinterpret_cast<volatile unsigned*>(ca.sync) + 1u);
      for (int p = static_cast<int>(blockIdx.x); p < ca.n_beds; p += static_cast<int>(gridDim.x)) {
        uint32_t spins = 0;
        while (!__all_sync(0xffffffffu, static_cast<int>(ld_acquire_u32(ca.bed_ctr + p) - target) >= 0)) {
          __nanosleep(128);
          if (++spins == (1u << 26)) asm volatile("trap;");  // a head tile that never lands is a planning bug
        }
        chain_aggregate_bed(ca, ca.bed0 + p, static_cast<int>(lane));
      }
    }
  } else if (warp >= 4) {
    // ------------------------------------------------------------------ epilogue
    const int ew = (static_cast<int>(warp) - 4) >> 2;
    const bool prof = ca.prof != nullptr && warp == 4 && lane == 0;
    unsigned long long e_work = 0, e_start = prof ? clock64() : 0;
    const int eb = ew & 1;     // this warpgroup's accumulator: items of that parity
    const int half = ew >> 1;  // ... and its half of their columns
    const int wq = static_cast<int>(warp) & 3;
    const int row = wq * 32 + static_cast<int>(lane);  // M row = (p', c)
    if (!ca.stems_flagged) pdl_wait();
    const uint32_t taddr = tmem_base + (static_cast<uint32_t>(wq * 32) << 16) + static_cast<uint32_t>(eb * 256);
    for (int seq = eb;; seq += 2) {
      const uint32_t accph = static_cast<uint32_t>(seq >> 1) & 1u;
      const int slot = seq & (kChainRing - 1);
      mbar_wait(&it_full[slot], static_cast<uint32_t>(seq / kChainRing) & 1u, 219);
      const int gi = ring[slot];
      if (gi < 0) break;
      // the producer acquired this item's dependencies: its shortcut rows may be
      // read ahead of the accumulator wait, as K4b does (the ring slot is released
      // only after this wait, so it_ready's phases cannot alias)
      mbar_wait(&it_ready[slot], static_cast<uint32_t>(seq / kChainRing) & 1u, 218);
      mbar_arrive(&it_empty[slot]);
      const int4 dsc = __ldg(ca.idesc + gi);
      const int li = dsc.x >> 22, tile = dsc.x & ((1 << 22) - 1);
      const PPArgs& a = ca.L[li];
      PPTile t;
      t.p = dsc.y;
      t.nt = dsc.z;
      t.g = dsc.w;
      const int c = row & (a.cout - 1);
      const float bias = __ldg(a.bias + static_cast<size_t>(t.g) * a.bias_stride + c);
      // the shortcut rows are written inside this launch: read through L2 (ld.global.cg)
      pp_epi_tile<false, kEpiPartsChain>(a, t, half, wq, static_cast<int>(lane), taddr, &acc_full[eb], accph,
                                         &acc_empty[eb], bias, true, (ca.opts & 4) != 0);
      const unsigned long long e0 = prof ? clock64() : 0;
      if (a.fc_w == nullptr) {  // publish this column half of the tile (+1 of kEpiPartsChain per launch)
        named_bar_sync(2 + ew, 128);
        if (wq == 0 && lane == 0) {
          fence_proxy_async_global();
          __threadfence();
          red_release_add_u32(ca.flags + ca.flag_base[li] + tile, 1u);
        }
      } else if (ca.agg) {  // a head tile's half: count it for the bed (warp 3 of the bed's CTA aggregates)
        named_bar_sync(2 + ew, 128);  // the warpgroup's head partials are stored
        if (wq == 0 && lane == 0) {
          __threadfence();
          red_release_add_u32(ca.bed_ctr + (t.p - t.g * a.Pm), 1u);
        }
      }
      if (ca.trace && wq == 0 && lane == 0) ca.trace[5 * gi + 3 + half] = globaltimer();
      if (prof) e_work += clock64() - e0;
    }
    if (prof) {
      unsigned long long* pr = ca.prof + blockIdx.x * 16;
      pr[9] = e_work;
      pr[10] = clock64() - e_start;
    }
  }

  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_dealloc(tmem_base, 512);
  if (threadIdx.x == 0) {  // the last CTA out resets the queues and advances the epoch
    __threadfence();
    if (atomicAdd(ca.sync + 1, 1u) == gridDim.x - 1) {
      for (int k = 0; k < ca.n_chains; ++k) ca.ctr[k] = 0u;
      ca.sync[1] = 0u;
      if (ca.agg && ca.wpos != nullptr) *ca.wpos += ca.advance;  // the tick's ring cursor (K5's job otherwise)
      __threadfence();
      atomicAdd(ca.sync, 1u);
    }
  }
}

// ------------------------------------------------------------------ host side

int pp_phases(int cout) { return kBM / cout; }

static int pp_taps_per_parity(int cout, int stride) { return kTaps / stride + 2 * (pp_phases(cout) - 1); }

bool pp_shape_ok(int cin, int cout, int stride) {
  if (cout != 16 && cout != 32 && cout != 64) return false;
  if (cin != 16 && cin != 32 && cin != 64) return false;
  return stride == 1 || stride == 2;
}

static size_t pp_conv_wbytes(int cin, int cout, int stride) {
  return static_cast<size_t>(cin / 8) * stride * pp_taps_per_parity(cout, stride) * cout * 16;
}
// Identity-shortcut selection array per 16-channel shortcut group: [half][z][16 B],
// z in [0, (2ph-1)*cout): row (ph-1)*cout + c holds a one at channel c - (16 jr + 8 half).
static size_t pp_z_half_bytes(int cout) { return static_cast<size_t>(2 * pp_phases(cout) - 1) * cout * 16; }

size_t pp_wbytes(int cin, int cout, int stride, int zc) {
  return pp_conv_wbytes(cin, cout, stride) + static_cast<size_t>(zc / 16) * 2 * pp_z_half_bytes(cout);
}

// Weight image [pair j][half h][parity pi][entry e][cout][8 fp16]:
// entry e of parity pi holds tap stride*(e - (ph-1)) + pi (zero outside [0,16)),
// channels 16j + 8h .. +7; then (zc > 0) the shortcut selection arrays.
void pp_pack_weights(const float* w, int cin, int cout, int stride, uint16_t* dst, int zc) {
  const int ph = pp_phases(cout), na = pp_taps_per_parity(cout, stride);
  size_t o = 0;
  for (int j = 0; j < cin / 16; ++j)
    for (int h = 0; h < 2; ++h)
      for (int pi = 0; pi < stride; ++pi)
        for (int e = 0; e < na; ++e) {
          const int t = stride * (e - (ph - 1)) + pi;
          for (int co = 0; co < cout; ++co)
            for (int k = 0; k < 8; ++k) {
              const int ci = 16 * j + 8 * h + k;
              const float v = (t >= 0 && t < kTaps) ? w[(static_cast<size_t>(co) * cin + ci) * kTaps + t] : 0.f;
              const __half hv = __float2half_rn(v);
              uint16_t bits;
              std::memcpy(&bits, &hv, 2);
              dst[o++] = bits;
            }
        }
  const __half one = __float2half_rn(1.f);
  uint16_t one_bits;
  std::memcpy(&one_bits, &one, 2);
  const int zrows = (2 * ph - 1) * cout, z0 = (ph - 1) * cout;
  for (int jr = 0; jr < zc / 16; ++jr)
    for (int h = 0; h < 2; ++h)
      for (int z = 0; z < zrows; ++z)
        for (int k = 0; k < 8; ++k) {
          const int c = z - z0;
          dst[o++] = (c >= 0 && c < cout && c == 16 * jr + 8 * h + k) ? one_bits : 0;
        }
}

using EncodeTiledFnPP = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                     const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                     CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFnPP get_encode_pp() {
  static EncodeTiledFnPP fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFnPP>(p);
  }
  return fn;
}

// Columns per tile: the largest N whose operands fit with >= 2 stages, then
// the one that minimises (waves x per-tile cost) -- small layers at serving
// batch sizes prefer narrower tiles over a ragged last wave.  HB_PP_NB forces.
// Column tile N (a multiple of 16, 64..256): per-tile time ~ N + 171 column
// units (the fixed part measured as N=128 tiles costing 1.4x per column of
// N=256 ones: A is re-read per MMA), times the waves of tiles over the SMs.
// Widths between the powers of two trim the padding of awkward rows (L = 7500
// gives 1875 / 938 / 469 columns: 240-wide tiles instead of 256 drop the
// 9 % padded columns to 2 %).
// The head layer (a member's last conv, fused mean-pool + FC) is the exception:
// its tile width sets how the fp32 pooled sum is split into per-(tile, warp)
// partials, so it is chosen from the layer shape alone (the same model with the
// wave quantisation dropped, i.e. as if the batch were large).  A bed's logit
// is then bit-identical whatever the batch size, shard or grid cap.  HB_PP_NB
// forces a width wherever it fits (elsewhere the model chooses).  The knobs
// are read per plan (tools/abtick.py compares settings in one process).
static int pick_nb(int tiles_per_col_unit, int n_cols, int num_sms, const std::function<bool(int)>& fits,
                   bool maxpool_epi, bool shape_only) {
  const int force = getenv("HB_PP_NB") ? atoi(getenv("HB_PP_NB")) : 0;
  const bool pow2_only = getenv("HB_PP_NB_POW2") && atoi(getenv("HB_PP_NB_POW2"));
  const double fixed_cols = getenv("HB_PP_NB_FIXED") ? atof(getenv("HB_PP_NB_FIXED")) : 171.0;
  // maxpool shortcut in the epilogue at ph >= 4: the epilogue, not the MMA, sets
  // the pace and narrower tiles overlap it better (tools/nb_sweep.py: 160-wide
  // tiles 8-14 % faster on the 32-channel maxpool layers) - a smaller fixed term
  const double fixed_mp = getenv("HB_PP_NB_FIXED_MP") ? atof(getenv("HB_PP_NB_FIXED_MP")) : 60.0;
  if (force >= 64 && force <= 256 && force % 16 == 0 && fits(force)) return force;
  const double fixed = maxpool_epi ? fixed_mp : fixed_cols;
  int best = 0;
  double best_t = 1e30;
  for (int nb = 256; nb >= 64; nb -= 16) {
    if (pow2_only && (nb & (nb - 1))) continue;
    if (!fits(nb)) continue;
    const long col_tiles = (n_cols + nb - 1) / nb;
    const long tiles = static_cast<long>(tiles_per_col_unit) * col_tiles;
    const double waves = shape_only ? static_cast<double>(col_tiles) : static_cast<double>((tiles + num_sms - 1) / num_sms);
    const double tt = waves * (nb + fixed);
    if (tt < best_t - 1e-9) {
      best_t = tt;
      best = nb;
    }
  }
  return best;
}

const char* plan_pp(PPPlan* plan, int G, int Pm, int cin, int cout, int lin, int lout, int stride, int pad,
                    const __half* in, __half* out, int out_q, const uint8_t* wimg, const float* bias,
                    const __half* res, int res_mode, int res_c, int res_len, int res_q, int num_sms, int zc,
                    const float* fc_w, float* head_out, size_t head_g_stride, int prefer_nb) {
  std::memset(plan, 0, sizeof(*plan));
  if (G < 1 || G > kMaxGroup || Pm < 1) return "conv_pp: bad group shape";
  if (!pp_shape_ok(cin, cout, stride)) return "conv_pp: unsupported layer shape";
  if (lout != (lin + stride - 1) / stride) return "conv_pp: lout must be ceil(lin/stride)";
  if (pad < 0 || pad > 8) return "conv_pp: padding out of range";
  if (out_q < 1 || out_q > 32 || (out_q & (out_q - 1))) return "conv_pp: out_q must be a power of two <= 32";
  if (res && (res_q < 1 || res_q > 32 || (res_q & (res_q - 1)))) return "conv_pp: res_q must be a power of two <= 32";
  if (res && res_c > cout) return "conv_pp: shortcut wider than the output";
  PPArgs& a = plan->args;
  a.G = G;
  a.Pm = Pm;
  a.P = G * Pm;
  a.cin = cin;
  a.cout = cout;
  a.stride = stride;
  a.pad = pad;
  a.lin = lin;
  a.lout = lout;
  a.ph = pp_phases(cout);
  a.Q = stride * a.ph;
  a.qs = ilog2(a.Q);
  a.U = stride * (a.ph - 1) + kTaps;
  a.n_pairs = cin / 16;
  const int na = pp_taps_per_parity(cout, stride);
  a.w_par16 = static_cast<uint32_t>(na * cout);  // one parity array, 16-B units
  a.w_half_bytes = static_cast<uint32_t>(stride * na * cout * 16);
  a.w_pair_bytes = 2 * a.w_half_bytes;
  // Identity shortcut as MMAs when the image carries Z for it and x is in this
  // conv's input layout.  Measured (192 rows, L=7500): 32 channels 68 -> 51 us;
  // 64 channels 115 -> 148 us (the 64-channel weights leave 3 B stages for 8
  // loads per tile, and the epilogue path is cheaper there), so only ph >= 4.
  const bool res_mma = res && res_mode == 1 && res_q == a.ph && a.ph >= 4 && res_c % 16 == 0 && zc == res_c &&
                       !(getenv("HB_PP_RES_EPI") && atoi(getenv("HB_PP_RES_EPI")));
  a.n_res_pairs = res_mma ? res_c / 16 : 0;
  a.z_off = static_cast<uint32_t>(pp_conv_wbytes(cin, cout, stride));
  a.z_half_bytes = static_cast<uint32_t>(pp_z_half_bytes(cout));
  a.z_pair_bytes = 2 * a.z_half_bytes;
  a.w_bytes = static_cast<uint32_t>(pp_wbytes(cin, cout, stride, res_mma ? zc : 0));
  a.w_stride = pp_wbytes(cin, cout, stride, zc);
  a.in_lq = lq_Q(lin, a.Q);
  a.out_qs = ilog2(out_q);
  a.out_lq = lq_Q(lout, out_q);
  a.out_rows = act_rows_q(lout, out_q);
  const int n_cols = (a.out_rows + a.ph - 1) / a.ph;
  const int dr_max = (a.U - 1 - pad) >> a.qs;
  const uint32_t fixed = 1024 + static_cast<uint32_t>(G * cout) * 4 + 256;
  if (a.w_bytes + fixed >= kSmemLimit) return "conv_pp: weights do not fit in shared memory";
  const uint32_t budget = kSmemLimit - fixed - a.w_bytes;
  auto fits = [&](int nb) {  // two B stages at least, TMA box rows <= 256
    const int R = round_up(8 + nb + dr_max, 8);
    return (2u * 2u * a.Q * R * 16u <= budget) && R / 8 <= 256;
  };
  // a member's last conv keeps the shape-only tile model: its width sets the fp32 grouping of the
  // mean-pool partials, and a bed's logit stays bit-identical across the chain / per-layer paths
  if (fc_w != nullptr) prefer_nb = 0;
  if (prefer_nb > 0) {
    // K4c: narrower tiles for short layers, whose few tiles per bed otherwise
    // leave a persistent CTA waiting on the previous layer's last tiles
    // (HB_CHAIN_MIN_TILES: column tiles per bed below which the width halves)
    const int min_tiles = getenv("HB_CHAIN_MIN_TILES") ? atoi(getenv("HB_CHAIN_MIN_TILES")) : 2;
    while (prefer_nb > 64 && (n_cols + prefer_nb - 1) / prefer_nb < min_tiles) prefer_nb = round_up(prefer_nb / 2, 16);
  }
  a.nb = (prefer_nb >= 64 && prefer_nb <= 256 && prefer_nb % 16 == 0 && fits(prefer_nb) && !getenv("HB_PP_NB"))
             ? prefer_nb
             : pick_nb(a.P, n_cols, num_sms, fits, res && res_mode == 2 && a.ph >= 4, fc_w != nullptr);
  if (!a.nb) return "conv_pp: no column tile fits in shared memory";
  a.R = round_up(8 + a.nb + dr_max, 8);
  a.stage_bytes = static_cast<uint32_t>(2 * a.Q * a.R * 16);
  a.n_stages = static_cast<int>(budget / a.stage_bytes);
  {
    const int cap = getenv("HB_PP_STAGES") ? atoi(getenv("HB_PP_STAGES")) : 4;
    if (a.n_stages > cap) a.n_stages = cap;
  }
  a.nt_per_p = (n_cols + a.nb - 1) / a.nb;
  a.num_tiles = a.P * a.nt_per_p;
  a.tmem_cols = 32;
  while (a.tmem_cols < static_cast<uint32_t>(2 * a.nb)) a.tmem_cols <<= 1;  // allocation: a power of two
  a.wimg = wimg;
  a.bias = bias;
  a.bias_stride = static_cast<int>(bias_len(cout));
  a.out = out;
  a.fc_w = fc_w;
  a.head_out = head_out;
  a.head_mt = a.nt_per_p * 4 * kHeadParts;  // one partial per (column tile, column quarter, warp)
  a.head_g_stride = head_g_stride ? head_g_stride : static_cast<size_t>(Pm) * a.head_mt;
  a.res = res;
  a.res_mode = (res && !res_mma) ? res_mode : 0;  // the epilogue's share of the shortcut
  a.res_c = res ? res_c : 0;
  a.res_qs = res ? ilog2(res_q) : 0;
  a.res_lq = res ? lq_Q(res_len, res_q) : 0;
  if (a.res && a.res_mode == 2 && act_rows_q(res_len, res_q) < 2 * lout)
    return "conv_pp: maxpool shortcut shorter than the output";
  plan->smem_bytes = a.w_bytes + a.n_stages * a.stage_bytes + fixed;
  plan->grid = a.num_tiles < num_sms ? a.num_tiles : num_sms;
  {  // member-partitioned CTAs when that costs no extra wave (HB_PP_SPLIT=0 disables)
    const int split_on = getenv("HB_PP_SPLIT") ? atoi(getenv("HB_PP_SPLIT")) : 1;
    const int grid = plan->grid, per_g = a.Pm * a.nt_per_p;
    int waves_split = 0;
    for (int g = 0; g < G; ++g) {
      const int n_g = ((g + 1) * grid) / G - (g * grid) / G;
      waves_split = n_g < 1 ? 1 << 30 : std::max(waves_split, (per_g + n_g - 1) / n_g);
    }
    a.member_split = split_on && G > 1 && a.num_tiles > grid && waves_split <= (a.num_tiles + grid - 1) / grid;
  }

  EncodeTiledFnPP enc = get_encode_pp();
  if (!enc) return "conv_pp: cuTensorMapEncodeTiled unavailable";
  // input, Q-phase layout: {64 elems = one 128-B line of 8 rows, lq/8 lines, Q phases, P*cin/8 planes}
  const cuuint64_t lq = static_cast<cuuint64_t>(a.in_lq);
  const cuuint64_t dims[4] = {64, lq / 8, static_cast<cuuint64_t>(a.Q), static_cast<cuuint64_t>(a.P) * (cin / 8)};
  const cuuint64_t strides[3] = {128, lq * 16, static_cast<cuuint64_t>(a.Q) * lq * 16};
  const cuuint32_t box[4] = {64, static_cast<cuuint32_t>(a.R / 8), static_cast<cuuint32_t>(a.Q), 2};
  const cuuint32_t estr[4] = {1, 1, 1, 1};
  const CUresult rc = enc(&plan->tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 4, const_cast<__half*>(in), dims, strides, box,
                          estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                          CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (rc != CUDA_SUCCESS) return "conv_pp: cuTensorMapEncodeTiled rejected the activation view";
  if (res_mma) {  // x: {lines, lq/8, Q = ph phases, P*res_c/8 planes}, the same box as a B stage
    const cuuint64_t xlq = static_cast<cuuint64_t>(lq_Q(res_len, res_q));
    const cuuint64_t xd[4] = {64, xlq / 8, static_cast<cuuint64_t>(res_q), static_cast<cuuint64_t>(a.P) * (res_c / 8)};
    const cuuint64_t xs[3] = {128, xlq * 16, static_cast<cuuint64_t>(res_q) * xlq * 16};
    const CUresult rx = enc(&plan->tmapX, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 4, const_cast<__half*>(res), xd, xs, box,
                            estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (rx != CUDA_SUCCESS) return "conv_pp: cuTensorMapEncodeTiled rejected the shortcut view";
  } else {
    plan->tmapX = plan->tmap;  // unused
  }
  a.dbg = getenv("HB_PP_DBG") ? atoi(getenv("HB_PP_DBG")) : 0;
  return nullptr;
}

cudaError_t init_pp_kernel() {
  cudaError_t e = cudaFuncSetAttribute(conv_pp_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemLimit);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(chain_pp_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemLimit);
  return e;
}

void free_chain(ChainPlan* cp) {
  cudaFree(cp->d_tmaps);
  cudaFree(cp->d_items);
  cudaFree(cp->d_item_off);
  cudaFree(cp->d_flags);
  cudaFree(cp->d_sync);
  cudaFree(cp->d_prof);
  cudaFree(cp->d_trace);
  cudaFree(cp->d_bed);
  cudaFree(cp->d_idesc);
  cudaFree(cp->d_ideps);
  delete cp->args;
  *cp = ChainPlan();
}

// Work of a chain launch: one queue per (chain, group member), layer-major,
// tiles in (patient, column) order, pulled with an atomic counter.  Each CTA
// has a home queue -- CTA blocks in proportion to the queues' MMA work
// (issued MMA columns per tile plus a fixed per-tile term), so members run
// side by side and a CTA changes weight image only at layer boundaries --
// and steals from the other queues once its own is drained, which evens out
// the cost model's error at the end of the launch.
const char* plan_chain(ChainPlan* cp, const ChainLayerIn* in, int n, int num_sms, const ChainStemIn* stems) {
  free_chain(cp);
  if (n < 1 || n > kMaxChainLayers) return "chain: layer count out of range";
  cp->args = new ChainArgs();
  ChainArgs& ca = *cp->args;
  std::memset(&ca, 0, sizeof(ca));
  std::vector<CUtensorMap> tm(2 * n);
  int n_chains = 0, flags = 0;
  for (int i = 0; i < n; ++i) n_chains = std::max(n_chains, in[i].chain + 1);
  // the stems' tile counters first (when they publish them), then the layers'
  std::vector<int> stem_base(n_chains, -1);
  if (stems)
    for (int k = 0; k < n_chains; ++k) {
      stem_base[k] = flags;
      flags += stems[k].rows * stems[k].tiles_per_row;
    }
  // HB_CHAIN_OPTS (experiments): 1 = no proxy fence on the consumer side, 4 = no epilogue math or
  // stores (timing only: the outputs are garbage)
  ca.opts = getenv("HB_CHAIN_OPTS") ? atoi(getenv("HB_CHAIN_OPTS")) : 0;
  uint32_t smem = 0;
  for (int i = 0; i < n; ++i) {
    const PPPlan& p = *in[i].plan;
    if (in[i].dep_in >= i || in[i].dep_res >= i) return "chain: a layer depends on a later one";
    if ((in[i].dep_in == kChainDepStem || in[i].dep_res == kChainDepStem) && !stems)
      return "chain: a stem dependency without stem counters";
    if (p.args.dbg) return "chain: debug knobs (HB_PP_DBG) are per-launch only";
    ca.L[i] = p.args;
    if (ca.L[i].n_stages > kChainStages) ca.L[i].n_stages = kChainStages;
    ca.dep_in[i] = in[i].dep_in;
    ca.dep_res[i] = in[i].dep_res;
    ca.flag_base[i] = flags;
    if (!p.args.fc_w) flags += p.args.num_tiles;
    tm[2 * i] = p.tmap;
    tm[2 * i + 1] = p.tmapX;
    smem = std::max(smem, kChainFixed + p.args.w_bytes + static_cast<uint32_t>(ca.L[i].n_stages) * p.args.stage_bytes);
    n_chains = std::max(n_chains, in[i].chain + 1);
    if (p.args.num_tiles >= (1 << 22)) return "chain: too many tiles in one layer";
  }
  if (smem > kSmemLimit) return "chain: a layer does not fit in shared memory";
  for (int i = 0; i < n; ++i) {  // a dependency must be on the same chain with the same row numbering
    for (int d : {in[i].dep_in, in[i].dep_res})
      if (d >= 0 && (in[d].chain != in[i].chain || ca.L[d].P != ca.L[i].P)) return "chain: bad dependency";
    if (stems && (in[i].dep_in == kChainDepStem || in[i].dep_res == kChainDepStem) &&
        stems[in[i].chain].rows != ca.L[i].P)
      return "chain: stem rows differ from the layer's";
  }
  ca.stems_flagged = stems != nullptr;
  // One queue per (chain, group member): a member's layers use one weight
  // image each, so a CTA drawing from one queue changes image only at layer
  // boundaries.  CTA blocks per queue in proportion to the MMA work (largest
  // remainder, >= 1 each).
  std::vector<int> q_chain, q_member;
  for (int k = 0; k < n_chains; ++k) {
    int G = 0;
    for (int i = 0; i < n; ++i)
      if (in[i].chain == k) G = ca.L[i].G;
    for (int g = 0; g < G; ++g) {
      q_chain.push_back(k);
      q_member.push_back(g);
    }
  }
  const int nq = static_cast<int>(q_chain.size());
  std::vector<double> cost(nq, 0.0);
  for (int q = 0; q < nq; ++q)
    for (int i = 0; i < n; ++i) {
      if (in[i].chain != q_chain[q]) continue;
      const PPArgs& a = ca.L[i];
      const double mmas = a.n_pairs * a.U + a.n_res_pairs * a.ph;
      cost[q] += static_cast<double>(a.Pm * a.nt_per_p) * (mmas * a.nb * 0.5 + 600.0);
    }
  const int grid = num_sms;
  double tot = 0;
  for (double v : cost) tot += v;
  std::vector<int> ctas(nq, 1);
  if (nq > grid) {  // fewer CTAs than queues (a capped grid): one home each, the rest drained by stealing
    for (int q = 0; q < nq; ++q) ctas[q] = q < grid ? 1 : 0;
  } else {
    int left = grid - nq;
    std::vector<std::pair<double, int>> rem;
    for (int q = 0; q < nq; ++q) {
      const double share = cost[q] / tot * grid - 1.0;
      const int whole = std::max(0, std::min(left, static_cast<int>(share)));
      ctas[q] += whole;
      left -= whole;
      rem.push_back({share - whole, q});
    }
    std::sort(rem.begin(), rem.end(), [](const std::pair<double, int>& x, const std::pair<double, int>& y) {
      return x.first > y.first;
    });
    for (size_t r = 0; left > 0; r = (r + 1) % rem.size(), --left) ctas[rem[r].second] += 1;
  }
  // queue items: the member's tiles in (patient, column) order, layer-major -- except that the
  // leading run of large layers (HB_CHAIN_CHUNKS chunks, default 2) goes bed chunk by bed chunk: all those
  // layers over the first chunk's beds, then over the next chunk's, so a layer reads its producer
  // layer's output (and its block input) while they are still in L2.  Every item still follows
  // all the items it depends on (same beds, earlier layers; rows are per bed).
  // default 2: the chain's DRAM reads drop from 1.36 to 1.01 GB per c2 tick (ncu) -- neutral on
  // a cool clock, +1.5-2 % over 1000 power-capped ticks (profiles/r02_ab_chain.txt)
  const int n_chunks = getenv("HB_CHAIN_CHUNKS") ? std::max(1, atoi(getenv("HB_CHAIN_CHUNKS"))) : 2;
  const int chunk_min = getenv("HB_CHAIN_CHUNK_MIN") ? atoi(getenv("HB_CHAIN_CHUNK_MIN")) : 128;
  std::vector<int> items, qoff(nq + 1, 0), home(grid, 0);
  for (int q = 0; q < nq; ++q) {
    qoff[q] = static_cast<int>(items.size());
    std::vector<int> ls;  // this chain's layers, in order
    for (int i = 0; i < n; ++i)
      if (in[i].chain == q_chain[q]) ls.push_back(i);
    size_t pre = 0;  // the chunked prefix: layers with >= chunk_min tiles per (member, chunk)
    while (n_chunks > 1 && pre < ls.size() && ca.L[ls[pre]].Pm * ca.L[ls[pre]].nt_per_p / n_chunks >= chunk_min) ++pre;
    auto emit = [&](int i, int p0, int p1) {
      const int ntp = ca.L[i].nt_per_p;
      const int t0 = (q_member[q] * ca.L[i].Pm + p0) * ntp, t1 = (q_member[q] * ca.L[i].Pm + p1) * ntp;
      for (int t = t0; t < t1; ++t) items.push_back((i << 22) | t);
    };
    if (pre > 0) {
      const int Pm = ca.L[ls[0]].Pm;
      for (int c = 0; c < n_chunks; ++c)
        for (size_t k = 0; k < pre; ++k) emit(ls[k], c * Pm / n_chunks, (c + 1) * Pm / n_chunks);
    }
    for (size_t k = pre; k < ls.size(); ++k) emit(ls[k], 0, ca.L[ls[k]].Pm);
  }
  qoff[nq] = static_cast<int>(items.size());
  {
    int b = 0;
    for (int q = 0; q < nq; ++q)
      for (int j = 0; j < ctas[q]; ++j) home[b++] = q;
  }
  // per item: its decoded tile and the counters of the producer tiles its TMA boxes
  // (input rows [Q(nt*nb - 8), Q(nt*nb - 8 + R)), shortcut rows) cover
  std::vector<int4> idesc(items.size()), ideps(items.size());
  auto dep_range = [&](int dl, int row, long lo, long hi, int* f0, int* f1) {
    *f0 = *f1 = 0;
    if (dl < 0) return;  // written before the launch
    const PPArgs& d = ca.L[dl];
    lo = std::max(lo, 0L);
    hi = std::min(hi, static_cast<long>(d.out_rows));
    if (hi <= lo) return;
    const long ppt = static_cast<long>(d.ph) * d.nb;
    const long t0 = lo / ppt, t1 = std::min((hi - 1) / ppt, static_cast<long>(d.nt_per_p - 1));
    const int base = ca.flag_base[dl] + row * d.nt_per_p;
    *f0 = base + static_cast<int>(t0);
    *f1 = base + static_cast<int>(t1) + 1;
  };
  for (size_t k = 0; k < items.size(); ++k) {
    const int i = items[k] >> 22, tile = items[k] & ((1 << 22) - 1);
    const PPArgs& a = ca.L[i];
    const int per_g = a.Pm * a.nt_per_p;
    const int g = tile / per_g, rem = tile - g * per_g, pl = rem / a.nt_per_p, nt = rem - pl * a.nt_per_p;
    const int p = g * a.Pm + pl;
    idesc[k] = make_int4(items[k], p, nt, g);
    int4 dr = make_int4(0, 0, 0, 0);
    const long r0 = 8L * (nt * (a.nb / 8) - 1);
    // the stem's tiles: 1024-position blocks x groups_per_blk phase groups per block
    auto stem_range = [&](int row, long lo, long hi, int* f0, int* f1) {
      const ChainStemIn& sm = stems[in[i].chain];
      lo = std::max(lo, 0L);
      hi = std::min(hi, static_cast<long>(sm.out_rows));
      *f0 = *f1 = 0;
      if (hi <= lo) return;
      const int base = stem_base[in[i].chain] + row * sm.tiles_per_row;
      *f0 = base + static_cast<int>(lo / 1024) * sm.groups_per_blk;
      *f1 = std::min(base + static_cast<int>((hi - 1) / 1024 + 1) * sm.groups_per_blk, base + sm.tiles_per_row);
    };
    if (ca.dep_in[i] == kChainDepStem) stem_range(p, a.Q * r0, a.Q * (r0 + a.R), &dr.x, &dr.y);
    if (ca.dep_in[i] >= 0) dep_range(ca.dep_in[i], p, a.Q * r0, a.Q * (r0 + a.R), &dr.x, &dr.y);
    if (ca.dep_res[i] == kChainDepStem) {
      const long ppt = static_cast<long>(a.ph) * a.nb;
      if (a.n_res_pairs)
        stem_range(p, a.ph * r0, a.ph * (r0 + a.R), &dr.z, &dr.w);
      else if (a.res_mode == 1)
        stem_range(p, ppt * nt, ppt * (nt + 1), &dr.z, &dr.w);
      else if (a.res_mode == 2)
        stem_range(p, 2 * ppt * nt, 2 * ppt * (nt + 1), &dr.z, &dr.w);
    }
    if (ca.dep_res[i] >= 0) {
      const long ppt = static_cast<long>(a.ph) * a.nb;
      if (a.n_res_pairs)
        dep_range(ca.dep_res[i], p, a.ph * r0, a.ph * (r0 + a.R), &dr.z, &dr.w);
      else if (a.res_mode == 1)
        dep_range(ca.dep_res[i], p, ppt * nt, ppt * (nt + 1), &dr.z, &dr.w);
      else if (a.res_mode == 2)
        dep_range(ca.dep_res[i], p, 2 * ppt * nt, 2 * ppt * (nt + 1), &dr.z, &dr.w);
    }
    if (dr.y - dr.x > kMaxRange || dr.w - dr.z > kMaxRange) return "chain: an item depends on too many tiles";
    ideps[k] = dr;
  }
  auto cpy = [](void** dst, const void* src, size_t bytes) -> bool {
    if (cudaMalloc(dst, bytes) != cudaSuccess) return false;
    return cudaMemcpy(*dst, src, bytes, cudaMemcpyHostToDevice) == cudaSuccess;
  };
  if (!cpy(reinterpret_cast<void**>(&cp->d_idesc), idesc.data(), sizeof(int4) * std::max<size_t>(1, idesc.size())) ||
      !cpy(reinterpret_cast<void**>(&cp->d_ideps), ideps.data(), sizeof(int4) * std::max<size_t>(1, ideps.size())))
    return "chain: device allocation failed";
  ca.idesc = cp->d_idesc;
  ca.ideps = cp->d_ideps;
  std::vector<int> meta(qoff);  // [queue offsets (n_chains + 1)][home (grid)]
  meta.insert(meta.end(), home.begin(), home.end());
  if (!cpy(reinterpret_cast<void**>(&cp->d_tmaps), tm.data(), sizeof(CUtensorMap) * tm.size()) ||
      !cpy(reinterpret_cast<void**>(&cp->d_items), items.data(), sizeof(int) * std::max<size_t>(1, items.size())) ||
      !cpy(reinterpret_cast<void**>(&cp->d_item_off), meta.data(), sizeof(int) * meta.size()))
    return "chain: device allocation failed";
  if (cudaMalloc(&cp->d_flags, sizeof(unsigned) * std::max(1, flags)) != cudaSuccess ||
      cudaMemset(cp->d_flags, 0, sizeof(unsigned) * std::max(1, flags)) != cudaSuccess ||
      cudaMalloc(&cp->d_sync, sizeof(unsigned) * (2 + nq)) != cudaSuccess ||
      cudaMemset(cp->d_sync, 0, sizeof(unsigned) * (2 + nq)) != cudaSuccess)
    return "chain: device allocation failed";
  if (stems)
    for (int k = 0; k < n_chains; ++k) cp->stem_flags.push_back(cp->d_flags + stem_base[k]);
  ca.tmaps = cp->d_tmaps;
  ca.items = cp->d_items;
  ca.queue_off = cp->d_item_off;
  ca.home = cp->d_item_off + nq + 1;
  ca.n_chains = nq;
  ca.ctr = cp->d_sync + 2;
  ca.flags = cp->d_flags;
  ca.sync = cp->d_sync;
  if (getenv("HB_CHAIN_PROF") && atoi(getenv("HB_CHAIN_PROF"))) {
    if (cudaMalloc(&cp->d_prof, sizeof(unsigned long long) * 16 * grid) != cudaSuccess ||
        cudaMemset(cp->d_prof, 0, sizeof(unsigned long long) * 16 * grid) != cudaSuccess)
      return "chain: device allocation failed";
    ca.prof = cp->d_prof;
    if (cudaMalloc(&cp->d_trace, sizeof(unsigned long long) * 5 * std::max<size_t>(1, items.size())) != cudaSuccess)
      return "chain: device allocation failed";
    ca.trace = cp->d_trace;
    cp->n_items = static_cast<int>(items.size());
  }
  cp->grid = grid;
  cp->n_layers = n;
  cp->smem_bytes = smem;
  return nullptr;
}

cudaError_t launch_chain(const ChainPlan& cp, cudaStream_t st) {
  return launch_pdl(chain_pp_kernel, dim3(cp.grid), dim3(kPPThreads), cp.smem_bytes, st, *cp.args);
}

cudaError_t launch_pp(const PPPlan& plan, cudaStream_t st) {
  return launch_pdl(conv_pp_kernel, dim3(plan.grid), dim3(kPPThreads), plan.smem_bytes, st, plan.tmap, plan.tmapX,
                    plan.args);
}

}  // namespace hb
