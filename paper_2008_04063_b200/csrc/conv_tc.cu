// K4: 1-D convolution (16 taps, stride 1|2, "same" padding) as an implicit GEMM
// on tcgen05 tensor cores, with the folded-BN bias / shortcut add / ReLU and the
// optional mean-pool+FC head fused into the TMEM epilogue.
//
//   GEMM view (one tile = 128 output positions of one patient x bn channels):
//     D[m, n] = sum_{t, c} X[s*(l0+m) + t - pad, c] * W[n, c, t]
//   A (positions x K) is never materialised: the producer TMA-loads, per
//   8-channel group, the contiguous run of input rows the tile touches (rows
//   [l0-pad, l0-pad+144) for s=1; for s=2 the even and odd positions as two
//   regions via a 5-D (pair, parity) tensor-map view).  The smem layout is the
//   canonical K-major no-swizzle UMMA layout with rows 16 B apart, so tap t is
//   the same region shifted by t rows: descriptor start + 16*t.  Out-of-range
//   rows (the "same" padding) are zero-filled by TMA.
//   B (weights) is pre-packed on the host into the exact smem image and moved
//   with plain bulk copies; it stays resident in smem across tiles when the
//   whole layer's weights fit.
//
// Roles (256 threads, 1 CTA/SM, persistent over tiles):
//   warp 0  : TMA producer (one elected lane)
//   warp 1  : MMA issuer (one lane), double-buffered TMEM accumulators
//   warp 2  : TMEM allocator
//   warps 4-7: epilogue, thread r <-> TMEM lane r <-> output position l0+r
#include "hb_kernels.cuh"
#include "hb_ptx.cuh"

#include <cstring>
#include <cstdio>
#include <vector>

namespace hb {

__device__ __forceinline__ int floordiv(int a, int b) { return (a >= 0) ? a / b : -((-a + b - 1) / b); }

__global__ void __launch_bounds__(kConvThreads, 1)
    conv_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ ConvArgs a) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sB = smem;
  uint8_t* sA = smem + a.nb_slots * a.b_chunk_bytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sA + a.na_stages * a.a_stage_bytes);
  uint64_t* a_full = bars;
  uint64_t* a_empty = a_full + a.na_stages;
  uint64_t* b_full = a_empty + a.na_stages;
  uint64_t* b_empty = b_full + a.nb_slots;
  uint64_t* acc_full = b_empty + a.nb_slots;
  uint64_t* acc_empty = acc_full + 2;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(acc_empty + 2);
  float* s_head = reinterpret_cast<float*>(tmem_holder + 4);  // [4] per-warp head partials
  uint32_t* s_aoff = reinterpret_cast<uint32_t*>(s_head + 4);  // [ksteps] A descriptor offsets (16 B units)
  uint32_t* s_boff = s_aoff + 64;                              // [ksteps] B descriptor offsets
  float* s_bias = reinterpret_cast<float*>(s_boff + 64);       // [bn]
  float* s_fc = s_bias + 256;                                  // [bn]

  const uint32_t warp = warp_id();
  const uint32_t lane = lane_id();

  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tmA);
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
      mbar_init(&acc_empty[i], 128);
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc(tmem_holder, a.tmem_cols);
  // Per-K-step smem descriptor offsets, so the single MMA-issuing thread does
  // no index arithmetic in its loop.  K-step ks covers (tap t, channel groups
  // g, g+1) for 16+-channel chunks, or taps (t, t+stride) of the one 8-channel
  // group; the A region of tap t is the tile's input rows shifted by t rows.
  if (threadIdx.x < a.ksteps) {
    const int ks = threadIdx.x;
    int t, g;
    if (a.ck >= 16) {
      const int per_tap = a.ck / 16;
      t = ks / per_tap;
      g = 2 * (ks % per_tap);
    } else {
      t = (a.stride == 1) ? 2 * ks : (ks / 2) * 4 + (ks % 2);
      g = 0;
    }
    const int u = t - a.pad;
    const int q = u - a.stride * floordiv(u, a.stride);
    const int row0 = floordiv(u, a.stride) - a.lo;
    const uint32_t region_bytes = static_cast<uint32_t>((a.ck / 8) * a.rows * 16);
    s_aoff[ks] = (static_cast<uint32_t>(q) * region_bytes + static_cast<uint32_t>(g * a.rows * 16 + row0 * 16)) >> 4;
    s_boff[ks] = static_cast<uint32_t>(ks * 2 * a.bn * 16) >> 4;
  }
  for (int i = threadIdx.x; i < a.bn; i += blockDim.x) {
    const int co = i;  // bias / fc are indexed per n-tile below (n_ntiles > 1 reloads per tile)
    s_bias[i] = a.bias[co];
    s_fc[i] = a.fc_w ? a.fc_w[co < a.cout ? co : 0] : 0.f;
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;

  const int tiles_per_nt = a.P * a.mt_per_p;

  if (warp == 0) {
    if (lane == 0) {
      // ------------------------------------------------------------ producer
      int as = 0;
      uint32_t aph = 0;
      int bs = 0;
      uint32_t bph = 0;
      int loaded_nt = -1;
      const int groups = a.ck / 8;
      const uint32_t region_bytes = static_cast<uint32_t>(groups * a.rows * 16);
      for (int tile = blockIdx.x; tile < a.num_tiles; tile += gridDim.x) {
        const int nt = tile / tiles_per_nt;
        const int rem = tile % tiles_per_nt;
        const int p = rem / a.mt_per_p;
        const int l0 = (rem % a.mt_per_p) * kBM;
        const bool load_b = !a.b_resident || nt != loaded_nt;
        loaded_nt = nt;
        for (int kc = 0; kc < a.n_kchunks; ++kc) {
          if (load_b) {
            const int slot = a.b_resident ? kc : bs;
            if (!a.b_resident) mbar_wait(&b_empty[bs], bph ^ 1);
            mbar_arrive_expect_tx(&b_full[slot], a.b_chunk_bytes);
            bulk_load(sB + static_cast<size_t>(slot) * a.b_chunk_bytes,
                      a.wpack + (static_cast<size_t>(nt) * a.n_kchunks + kc) * a.b_chunk_bytes, a.b_chunk_bytes,
                      &b_full[slot]);
            if (!a.b_resident && ++bs == a.nb_slots) {
              bs = 0;
              bph ^= 1;
            }
          }
          mbar_wait(&a_empty[as], aph ^ 1);
          mbar_arrive_expect_tx(&a_full[as], a.a_stage_bytes);
          uint8_t* dst = sA + static_cast<size_t>(as) * a.a_stage_bytes;
          if (a.stride == 1) {
            tma_load_4d(dst, &tmA, &a_full[as], 0, l0 + a.lo, kc * groups, p);
          } else {
            tma_load_5d(dst, &tmA, &a_full[as], 0, 0, l0 + a.lo, kc * groups, p);
            tma_load_5d(dst + region_bytes, &tmA, &a_full[as], 0, 1, l0 + a.lo, kc * groups, p);
          }
          if (++as == a.na_stages) {
            as = 0;
            aph ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ------------------------------------------------------------ MMA issuer
      const uint32_t idesc = make_idesc_f16(kBM, a.bn);
      const uint32_t a_lbo = (a.ck >= 16) ? static_cast<uint32_t>(a.rows * 16) : 16u;
      const uint32_t b_lbo = static_cast<uint32_t>(a.bn * 16);
      int as = 0;
      uint32_t aph = 0;
      int bs = 0;
      uint32_t bph = 0;
      int acc = 0;
      uint32_t accph = 0;
      int loaded_nt = -1;
      uint32_t bres_phase = 0;
      for (int tile = blockIdx.x; tile < a.num_tiles; tile += gridDim.x) {
        const int nt = tile / tiles_per_nt;
        if (a.b_resident && nt != loaded_nt) {
          if (loaded_nt >= 0) bres_phase ^= 1;
          loaded_nt = nt;
        }
        mbar_wait(&acc_empty[acc], accph ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + static_cast<uint32_t>(acc * a.bn);
        for (int kc = 0; kc < a.n_kchunks; ++kc) {
          const int slot = a.b_resident ? kc : bs;
          mbar_wait(&b_full[slot], a.b_resident ? bres_phase : bph);
          mbar_wait(&a_full[as], aph);
          tc_fence_after();
          const uint64_t adesc = make_desc(smem_u32(sA + static_cast<size_t>(as) * a.a_stage_bytes), a_lbo, 128);
          const uint64_t bdesc = make_desc(smem_u32(sB + static_cast<size_t>(slot) * a.b_chunk_bytes), b_lbo, 128);
#pragma unroll 4
          for (int ks = 0; ks < a.ksteps; ++ks) {
            mma_f16_ss(d_tmem, adesc + s_aoff[ks], bdesc + s_boff[ks], idesc, (kc | ks) != 0 ? 1u : 0u);
          }
          mma_commit(&a_empty[as]);
          if (!a.b_resident) {
            mma_commit(&b_empty[bs]);
            if (++bs == a.nb_slots) {
              bs = 0;
              bph ^= 1;
            }
          }
          if (++as == a.na_stages) {
            as = 0;
            aph ^= 1;
          }
        }
        mma_commit(&acc_full[acc]);
        if (++acc == 2) {
          acc = 0;
          accph ^= 1;
        }
      }
    }
  } else if (warp >= 4) {
    // -------------------------------------------------------------- epilogue
    const int wq = static_cast<int>(warp) - 4;
    const int r = wq * 32 + static_cast<int>(lane);
    int acc = 0;
    uint32_t accph = 0;
    const int out_groups = a.cout / 8;
    const int res_groups = a.res_mode ? a.res_c / 8 : 0;
    for (int tile = blockIdx.x; tile < a.num_tiles; tile += gridDim.x) {
      const int nt = tile / tiles_per_nt;
      const int rem = tile % tiles_per_nt;
      const int p = rem / a.mt_per_p;
      const int mt = rem % a.mt_per_p;
      const int l = mt * kBM + r;
      const bool valid = l < a.lout;
      const bool in_buf = l < a.lp_out;
      const int g0 = nt * (a.bn / 8);
      const int ng = min(a.bn / 8, out_groups - g0);
      const __half* res_p = a.res_mode ? a.res + static_cast<size_t>(p) * res_groups * a.lp_res * 8 : nullptr;
      // Shortcut rows are independent of the accumulator: fetch the first 8
      // groups while the MMAs of this tile are still running.
      uint4 rres[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        rres[j] = make_uint4(0u, 0u, 0u, 0u);
        const int g = g0 + j;
        if (j < ng && g < res_groups && valid) {
          const __half* src = res_p + static_cast<size_t>(g) * a.lp_res * 8;
          if (a.res_mode == 1) {
            rres[j] = __ldg(reinterpret_cast<const uint4*>(src + static_cast<size_t>(l) * 8));
          } else {
            const uint4 r0 = __ldg(reinterpret_cast<const uint4*>(src + static_cast<size_t>(2 * l) * 8));
            const uint4 r1 = __ldg(reinterpret_cast<const uint4*>(src + static_cast<size_t>(2 * l + 1) * 8));
            const __half2* h0 = reinterpret_cast<const __half2*>(&r0);
            const __half2* h1 = reinterpret_cast<const __half2*>(&r1);
            __half2* o = reinterpret_cast<__half2*>(&rres[j]);
#pragma unroll
            for (int k = 0; k < 4; ++k) o[k] = __hmax2(h0[k], h1[k]);
          }
        }
      }
      const float* bias_t = (a.n_ntiles == 1) ? s_bias : a.bias + static_cast<size_t>(nt) * a.bn;
      mbar_wait(&acc_full[acc], accph);
      tc_fence_after();
      const uint32_t taddr = tmem_base + (static_cast<uint32_t>(wq * 32) << 16) + static_cast<uint32_t>(acc * a.bn);
      float head = 0.f;
#pragma unroll
      for (int c16 = 0; c16 < 16; ++c16) {
        if (c16 * 2 >= ng) break;
        float v[16];
        tmem_ld16(taddr + static_cast<uint32_t>(c16 * 16), v);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int j = 2 * c16 + h;
          if (j >= ng) break;
          const int g = g0 + j;
          float y[8];
#pragma unroll
          for (int k = 0; k < 8; ++k) y[k] = v[8 * h + k] + bias_t[8 * j + k];
          if (g < res_groups && valid) {
            uint4 rv;
            if (j < 8) {
              rv = rres[j < 8 ? j : 0];
            } else {
              const __half* src = res_p + static_cast<size_t>(g) * a.lp_res * 8;
              if (a.res_mode == 1) {
                rv = __ldg(reinterpret_cast<const uint4*>(src + static_cast<size_t>(l) * 8));
              } else {
                const uint4 r0 = __ldg(reinterpret_cast<const uint4*>(src + static_cast<size_t>(2 * l) * 8));
                const uint4 r1 = __ldg(reinterpret_cast<const uint4*>(src + static_cast<size_t>(2 * l + 1) * 8));
                const __half2* h0 = reinterpret_cast<const __half2*>(&r0);
                const __half2* h1 = reinterpret_cast<const __half2*>(&r1);
                __half2* o = reinterpret_cast<__half2*>(&rv);
#pragma unroll
                for (int k = 0; k < 4; ++k) o[k] = __hmax2(h0[k], h1[k]);
              }
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
            for (int k = 0; k < 8; ++k) y[k] = fmaxf(y[k], 0.f);
          }
          if (a.fc_w != nullptr) {
            if (valid) {
#pragma unroll
              for (int k = 0; k < 8; ++k) head = fmaf(y[k], s_fc[8 * j + k], head);
            }
          } else if (in_buf) {
            uint4 pk;
            __half2* o2 = reinterpret_cast<__half2*>(&pk);
#pragma unroll
            for (int k = 0; k < 4; ++k)
              o2[k] = valid ? __floats2half2_rn(y[2 * k], y[2 * k + 1]) : __floats2half2_rn(0.f, 0.f);
            *reinterpret_cast<uint4*>(a.out + ((static_cast<size_t>(p) * out_groups + g) * a.lp_out + l) * 8) = pk;
          }
        }
      }
      tc_fence_before();
      mbar_arrive(&acc_empty[acc]);
      if (++acc == 2) {
        acc = 0;
        accph ^= 1;
      }
      if (a.fc_w != nullptr) {
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) head += __shfl_xor_sync(0xffffffffu, head, off);
        if (lane == 0) s_head[wq] = head;
        named_bar_sync(1, 128);
        if (wq == 0 && lane == 0) {
          const float sum = ((s_head[0] + s_head[1]) + s_head[2]) + s_head[3];
          a.head_out[static_cast<size_t>(p) * a.mt_per_p + mt] = sum;  // n_ntiles == 1 enforced for heads
        }
        named_bar_sync(1, 128);
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_dealloc(tmem_base, a.tmem_cols);
}

// ------------------------------------------------------------------ host side

int conv_bn(int cout) {
  const int c = round_up(cout < 16 ? 16 : cout, 16);
  if (c <= 256) return c;
  // split N into equal tiles of <= 256 (multiple of 16)
  const int nt = (c + 255) / 256;
  return round_up((c + nt - 1) / nt, 16);
}

constexpr uint32_t kFixedSmem = 1024 + 256 + 512 + 2048;  // barriers, holder, head scratch, K-step tables, bias/fc

// Channels per k-chunk.  Prefer the largest chunk whose whole-layer weights
// stay resident in smem next to two A stages; otherwise the largest chunk that
// streams with two B slots + two A stages.  The host packer and the planner
// both call this, so the B image always matches the kernel's K-step order.
static int pick_ck(int cin, int cout, int stride, int* resident) {
  const int bn = conv_bn(cout);
  const int nnt = (round_up(cout, 16) + bn - 1) / bn;
  const int rows = (stride == 1) ? kBM + 16 : kBM + 8;
  const uint32_t budget = kSmemLimit - kFixedSmem;
  const int cands[4] = {64, 32, 16, 8};
  if (nnt == 1) {
    for (int ck : cands) {
      if (cin % ck || cin / ck > 32) continue;
      const uint32_t b_all = 32u * cin * bn;  // 16 taps * cin * bn * 2 B
      const uint32_t a_stage = static_cast<uint32_t>(stride * rows * ck * 2);
      if (b_all + 2 * a_stage <= budget) {
        *resident = 1;
        return ck;
      }
    }
  }
  for (int ck : cands) {
    if (cin % ck) continue;
    const uint32_t b_chunk = 32u * ck * bn;
    const uint32_t a_stage = static_cast<uint32_t>(stride * rows * ck * 2);
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

// B image per (ntile, kchunk): [kstep][half][bn rows][8 fp16], the K-step
// order matching the MMA issuer (tap-major, then 16-channel sub-chunks; for
// 8-channel chunks taps are paired (t,t+1) for s=1 or (t,t+2) for s=2 — the
// pairing only depends on the consumer's stride, so a stride-specific image
// is built: see pack_weights_strided).
static void pack_weights_strided(const float* w, int cin, int cout, int stride, uint16_t* dst) {
  const int bn = conv_bn(cout);
  const int nnt = (round_up(cout, 16) + bn - 1) / bn;
  int resident;
  const int ck = pick_ck(cin, cout, stride, &resident);
  if (ck == 0) return;
  const int nkc = cin / ck;
  const int ksteps = (ck >= 16) ? ck : 8;
  size_t o = 0;
  for (int nt = 0; nt < nnt; ++nt)
    for (int kc = 0; kc < nkc; ++kc)
      for (int ks = 0; ks < ksteps; ++ks)
        for (int half = 0; half < 2; ++half) {
          int t, c0;
          if (ck >= 16) {
            const int per_tap = ck / 16;
            t = ks / per_tap;
            c0 = kc * ck + 16 * (ks % per_tap) + 8 * half;
          } else {
            const int t0 = (stride == 1) ? 2 * ks : (ks / 2) * 4 + (ks % 2);
            t = t0 + half * stride;
            c0 = kc * ck;
          }
          for (int n = 0; n < bn; ++n)
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

void pack_weights(const float* w, int cin, int cout, int stride, uint16_t* dst) {
  pack_weights_strided(w, cin, cout, stride, dst);
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

const char* plan_conv(ConvPlan* plan, int P, int cin, int cout, int lin, int lout, int stride, int pad,
                      const __half* in, int lp_in, __half* out, const uint8_t* wpack, const float* bias,
                      const __half* res, int res_mode, int res_c, int lp_res, const float* fc_w,
                      float* head_out, int num_sms) {
  std::memset(plan, 0, sizeof(*plan));
  if (cin % 8 || cout % 8) return "conv: channels must be multiples of 8";
  if (stride != 1 && stride != 2) return "conv: stride must be 1 or 2";
  if (stride == 2 && (lp_in % 2)) return "conv: stride-2 input needs even padded length";
  if (lout != (lin + stride - 1) / stride) return "conv: lout must be ceil(lin/stride)";
  ConvArgs& a = plan->args;
  a.P = P;
  a.cin = cin;
  a.cout = cout;
  a.bn = conv_bn(cout);
  a.n_ntiles = (round_up(cout, 16) + a.bn - 1) / a.bn;
  if (fc_w && a.n_ntiles != 1) return "conv: fused head needs cout <= 256";
  a.lin = lin;
  a.lout = lout;
  a.lp_out = round_up(lout, 8);
  a.stride = stride;
  a.pad = pad;
  a.lo = (stride == 1) ? -pad : -((pad + 1) / 2);  // floor(-pad/2)
  int resident = 0;
  a.ck = pick_ck(cin, cout, stride, &resident);
  if (a.ck == 0) return "conv: no k-chunk fits in shared memory";
  a.n_kchunks = cin / a.ck;
  a.ksteps = (a.ck >= 16) ? a.ck : 8;
  a.rows = (stride == 1) ? kBM + 16 : kBM + 8;
  a.mt_per_p = (lout + kBM - 1) / kBM;
  a.num_tiles = a.n_ntiles * P * a.mt_per_p;
  a.a_stage_bytes = static_cast<uint32_t>(stride * (a.ck / 8) * a.rows * 16);
  a.b_chunk_bytes = static_cast<uint32_t>(a.ksteps * 2 * a.bn * 16);
  const uint32_t fixed = kFixedSmem;
  const uint32_t budget = kSmemLimit - fixed;
  const uint32_t b_all = a.b_chunk_bytes * a.n_kchunks;
  a.b_resident = resident;
  a.nb_slots = resident ? a.n_kchunks : 2;
  const uint32_t b_smem = resident ? b_all : 2 * a.b_chunk_bytes;
  a.na_stages = static_cast<int>((budget - b_smem) / a.a_stage_bytes);
  if (a.na_stages > 4) a.na_stages = 4;
  if (a.na_stages < 2) return "conv: k-chunk does not fit in shared memory";
  uint32_t cols = 32;
  while (cols < static_cast<uint32_t>(2 * a.bn)) cols <<= 1;
  a.tmem_cols = cols;
  a.wpack = wpack;
  a.bias = bias;
  a.out = out;
  a.res = res;
  a.res_mode = res_mode;
  a.res_c = res_c;
  a.lp_res = lp_res;
  a.relu = 1;
  a.fc_w = fc_w;
  a.head_out = head_out;
  plan->smem_bytes = a.nb_slots * a.b_chunk_bytes + a.na_stages * a.a_stage_bytes + fixed;
  plan->grid = a.num_tiles < num_sms ? a.num_tiles : num_sms;

  EncodeTiledFn enc = get_encode();
  if (!enc) return "conv: cuTensorMapEncodeTiled unavailable";
  const int G = cin / 8;
  const cuuint32_t estr[5] = {1, 1, 1, 1, 1};
  CUresult rc;
  if (stride == 1) {
    const cuuint64_t dims[4] = {8, static_cast<cuuint64_t>(lp_in), static_cast<cuuint64_t>(G),
                                static_cast<cuuint64_t>(P)};
    const cuuint64_t strides[3] = {16, static_cast<cuuint64_t>(lp_in) * 16,
                                   static_cast<cuuint64_t>(G) * lp_in * 16};
    const cuuint32_t box[4] = {8, static_cast<cuuint32_t>(a.rows), static_cast<cuuint32_t>(a.ck / 8), 1};
    rc = enc(&plan->tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 4, const_cast<__half*>(in), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  } else {
    const cuuint64_t dims[5] = {8, 2, static_cast<cuuint64_t>(lp_in / 2), static_cast<cuuint64_t>(G),
                                static_cast<cuuint64_t>(P)};
    const cuuint64_t strides[4] = {16, 32, static_cast<cuuint64_t>(lp_in) * 16,
                                   static_cast<cuuint64_t>(G) * lp_in * 16};
    const cuuint32_t box[5] = {8, 1, static_cast<cuuint32_t>(a.rows), static_cast<cuuint32_t>(a.ck / 8), 1};
    rc = enc(&plan->tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 5, const_cast<__half*>(in), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
  if (rc != CUDA_SUCCESS) return "conv: cuTensorMapEncodeTiled rejected the activation view";
  return nullptr;
}

cudaError_t init_conv_kernel() {
  return cudaFuncSetAttribute(conv_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemLimit);
}

cudaError_t launch_conv(const ConvPlan& plan, cudaStream_t st) {
  conv_tc_kernel<<<plan.grid, kConvThreads, plan.smem_bytes, st>>>(plan.tmap, plan.args);
  return cudaGetLastError();
}

}  // namespace hb
