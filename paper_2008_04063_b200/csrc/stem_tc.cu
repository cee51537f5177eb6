// K3: the stem conv (1 input channel -> w channels, 16 taps, "same" padding)
// + folded BN bias + ReLU on tcgen05 tensor cores.  Two kernels:
//   stem_pp_kernel (further down, the default for w <= 64): the window segment
//     itself is the MMA operand, the phase shifts live in shifted weight images;
//   stem_tc_kernel (this first part, w = 128 or HB_STEM=0): Toeplitz rows built
//     in shared memory, described here.
//
// With one input channel the whole 16-tap receptive field is exactly one
// kind::f16 K-step, so a tile of 128 output positions is ONE MMA:
//   D[m, c] = sum_t A[m, t] W[c, t],  A[m, t] = x[l0 + m + t - pad]
// A is the Toeplitz (im2col) view of the normalised window; rows overlap by
// one sample, which no TMA box or descriptor stride can express, so each
// producer thread writes its own row (32 B) into the canonical K-major
// no-swizzle layout from a staged window segment.  The kernel is bound by
// writing the w-channel output (HBM), not by math: 2*w*16 FLOP per 2*w bytes.
//
// Persistent and warp-specialised (one CTA per SM) so the phases of a tile
// overlap across tiles:
//   warp 9     TMA: the tile's 144-sample window segment (one 2-D box of the
//              [rows][x_stride] window buffer, zero-filled outside [0, L))
//              into a ring of kStages stages, up to kStages tiles ahead
//   warps 0-7  builders (two warpgroups, alternate tiles): segment ->
//              Toeplitz A rows of the same stage
//   warp 8     TMEM allocator + MMA issuer (one elected lane)
//   warps 12-31 epilogue: five warpgroups, warpgroup e drains accumulator e
//              (every 5th tile): thread r <-> TMEM lane r <-> position l0 + r;
//              bias, ReLU, fp16, 16-byte row stores in the consumer's Q-phase
//              layout.  (One warpgroup for all accumulators was latency-bound:
//              the old one-tile-per-CTA kernel with 12 CTAs/SM beat it.)
// Accumulators rotate over kAcc TMEM buffers.  Every member of the group keeps
// its B image (fp16 weights) and bias resident in smem, so member changes cost
// nothing.
#include <algorithm>
#include <vector>
#include <cstdlib>
#include <cstring>

#include "hb_kernels.cuh"
#include "hb_ptx.cuh"

namespace hb {

constexpr int kStemThreads = 1024;  // warps 0-7 two builder warpgroups, 8 MMA, 9 TMA, 12-31 five epilogue warpgroups
constexpr int kStages = 8;             // segment + A ring depth
constexpr int kAcc = 5;                // TMEM accumulators = epilogue warpgroups (fewer if TMEM is short)
constexpr int kStemA = kBM * 32;       // A tile: 2 K-halves x 128 rows x 16 B
constexpr int kStemSegN = 144;         // staged segment: samples [l0 - 8, l0 + 136)
constexpr int kStemSegB = kStemSegN * 2;  // bytes a segment TMA delivers
constexpr int kStemSegS = 384;         // segment stage stride (TMA destinations 128-B aligned)

struct StemTcArgs {
  StemMember m[kMaxGroup];
  int x_row0[kMaxGroup];  // member g's first window row in the TMA view
  int G, Pm, x_stride, L, out_qs, out_lq, out_rows, cout, n_mma, pad, mt_per_row, num_tiles;
  __half* out;
};

__global__ void __launch_bounds__(kStemThreads, 1)
    stem_tc_kernel(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ StemTcArgs a) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sA = smem;                                                 // [kStages][4 KB]
  __half* sSeg = reinterpret_cast<__half*>(sA + kStages * kStemA);     // [kStages][192] (144 used)
  uint8_t* sB = reinterpret_cast<uint8_t*>(sSeg) + kStages * kStemSegS;  // [G][2][n_mma][16 B]
  const int b_bytes = a.n_mma * 32;
  float* sBias = reinterpret_cast<float*>(sB + a.G * b_bytes);        // [G][cout]
  uint64_t* bars = reinterpret_cast<uint64_t*>(sBias + ((a.G * a.cout + 1) & ~1));
  uint64_t* a_full = bars;
  uint64_t* a_empty = a_full + kStages;
  uint64_t* seg_full = a_empty + kStages;
  uint64_t* d_full = seg_full + kStages;
  uint64_t* d_empty = d_full + kAcc;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(d_empty + kAcc);

  const uint32_t warp = warp_id();
  const int tid = threadIdx.x;
  uint32_t cols = 32;
  while (cols < static_cast<uint32_t>(a.n_mma)) cols <<= 1;
  const int n_acc = static_cast<int>(512 / cols) < kAcc ? static_cast<int>(512 / cols) : kAcc;
  uint32_t tmem_cols = 32;
  while (tmem_cols < cols * n_acc) tmem_cols <<= 1;
  if (tid == 0) {
    for (int i = 0; i < kStages; ++i) {
      mbar_init(&a_full[i], kBM);  // every builder thread arrives after writing its row
      mbar_init(&a_empty[i], 1);
      mbar_init(&seg_full[i], 1);
    }
    for (int i = 0; i < n_acc; ++i) {
      mbar_init(&d_full[i], 1);
      mbar_init(&d_empty[i], kBM);
    }
    fence_barrier_init();
  }
  if (warp == 8) tmem_alloc(tmem_holder, tmem_cols);
  // every member's B image (fp16, [K-half][n][8 taps]) and bias: constants, built before the dependency wait
  for (int i = tid; i < a.G * a.n_mma * 16; i += kStemThreads) {
    const int g = i / (a.n_mma * 16), rem = i - g * a.n_mma * 16;
    const int n = rem >> 4, t = rem & 15;
    const float w = n < a.cout ? a.m[g].w[n * kTaps + t] : 0.f;
    reinterpret_cast<__half*>(sB + g * b_bytes)[((t >> 3) * a.n_mma + n) * 8 + (t & 7)] = __float2half_rn(w);
  }
  for (int i = tid; i < a.G * a.cout; i += kStemThreads) sBias[i] = a.m[i / a.cout].b[i % a.cout];
  fence_proxy_async();  // B images are read by the tensor core
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_holder;
  pdl_wait();  // x is the window kernel's output; our output buffer may still be read upstream
  pdl_trigger();

  if (warp == 9) {
    // ---------------------------------------------------------------- TMA issuer
    if (lane_id() == 0) {
      prefetch_tmap(&tmX);
      int s = 0;
      uint32_t ph = 0;
      for (int tile = blockIdx.x; tile < a.num_tiles; tile += gridDim.x) {
        const int row = tile / a.mt_per_row;
        const int mt = tile - row * a.mt_per_row;
        const int g = row / a.Pm, p = row - g * a.Pm;
        mbar_wait(&a_empty[s], ph ^ 1u, 301);  // the stage's previous MMA (and so its builders) are done
        mbar_arrive_expect_tx(&seg_full[s], kStemSegB);
        tma_load_2d(sSeg + s * (kStemSegS / 2), &tmX, &seg_full[s], mt * kBM - 8, a.x_row0[g] + p);
        if (++s == kStages) {
          s = 0;
          ph ^= 1u;
        }
      }
    }
  } else if (warp < 8) {
    // ---------------------------------------------------------------- builders
    // two warpgroups, alternate tiles (local tile i -> warpgroup i % 2, stage i % kStages)
    const int bw = static_cast<int>(warp) >> 2;
    const int r = tid & 127;
    const int first = r + 8 - a.pad;  // segment index of sample l0 + r - pad
    for (int i = bw;; i += 2) {
      const int tile = blockIdx.x + i * gridDim.x;
      if (tile >= a.num_tiles) break;
      const int s = i % kStages;
      const uint32_t ph = static_cast<uint32_t>(i / kStages) & 1u;
      const __half* sg = sSeg + s * (kStemSegS / 2);
      mbar_wait(&seg_full[s], ph, 302);
      __align__(16) __half v[16];
#pragma unroll
      for (int t = 0; t < 16; ++t) v[t] = sg[first + t];
      const uint4* v4 = reinterpret_cast<const uint4*>(v);
      uint8_t* dst = sA + s * kStemA;
      const int off = (r >> 3) * 128 + (r & 7) * 16;
      *reinterpret_cast<uint4*>(dst + off) = v4[0];
      *reinterpret_cast<uint4*>(dst + kBM * 16 + off) = v4[1];
      fence_proxy_async();  // generic-proxy smem writes -> visible to the tensor core
      mbar_arrive(&a_full[s]);
    }
  } else if (warp == 8) {
    // ------------------------------------------------------------------ MMA issuer
    const uint32_t idesc = make_idesc_f16(kBM, a.n_mma);
    int s = 0, d = 0;
    uint32_t ph = 0, dph = 0;
    for (int tile = blockIdx.x; tile < a.num_tiles; tile += gridDim.x) {
      const int g = (tile / a.mt_per_row) / a.Pm;
      mbar_wait(&a_full[s], ph, 311);
      mbar_wait(&d_empty[d], dph ^ 1u, 312);
      tc_fence_after();
      const uint64_t adesc = make_desc(smem_u32(sA + s * kStemA), kBM * 16, 128);
      const uint64_t bdesc = make_desc(smem_u32(sB + g * b_bytes), a.n_mma * 16, 128);
      if (elect_one()) {
        mma_f16_ss(tmem + static_cast<uint32_t>(d) * cols, adesc, bdesc, idesc, 0u);
        mma_commit(&a_empty[s]);
        mma_commit(&d_full[d]);
      }
      __syncwarp();
      if (++s == kStages) {
        s = 0;
        ph ^= 1u;
      }
      if (++d == n_acc) {
        d = 0;
        dph ^= 1u;
      }
    }
  } else if (warp >= 12) {
    // -------------------------------------------------------------------- epilogue
    const int e = (static_cast<int>(warp) - 12) >> 2;  // warpgroup = accumulator
    const int wq = static_cast<int>(warp) & 3;
    const int r = wq * 32 + static_cast<int>(lane_id());  // TMEM lane quadrant wq
    const int d = e;
    uint32_t dph = 0;
    for (int tile = blockIdx.x + e * gridDim.x; e < n_acc && tile < a.num_tiles; tile += n_acc * gridDim.x) {
      const int row = tile / a.mt_per_row;
      const int mt = tile - row * a.mt_per_row;
      const int g = row / a.Pm;
      const int l = mt * kBM + r;
      const bool in_buf = l < a.out_rows, valid = l < a.L;
      mbar_wait(&d_full[d], dph, 321);
      tc_fence_after();
      const uint32_t taddr = tmem + (static_cast<uint32_t>(wq * 32) << 16) + static_cast<uint32_t>(d) * cols;
      const float* bias = sBias + g * a.cout;
      for (int c16 = 0; c16 * 16 < a.cout; ++c16) {  // warp-collective loads: every lane takes part
        float v[16];
        tmem_ld16(taddr + static_cast<uint32_t>(c16 * 16), v);
        if (c16 * 16 + 16 >= a.cout) {  // last TMEM read of this accumulator
          tc_fence_before();
          mbar_arrive(&d_empty[d]);
        }
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int g8 = c16 * 2 + h;
          if (g8 * 8 >= a.cout || !in_buf) break;
          uint4 pk;
          __half2* o2 = reinterpret_cast<__half2*>(&pk);
#pragma unroll
          for (int k = 0; k < 8; k += 2) {
            const float y0 = fmax_nan(v[8 * h + k] + bias[g8 * 8 + k], 0.f);
            const float y1 = fmax_nan(v[8 * h + k + 1] + bias[g8 * 8 + k + 1], 0.f);
            o2[k / 2] = valid ? __floats2half2_rn(y0, y1) : __floats2half2_rn(0.f, 0.f);
          }
          *reinterpret_cast<uint4*>(a.out + q_off(static_cast<size_t>(row) * (a.cout / 8) + g8, a.out_qs,
                                                  a.out_lq, l)) = pk;
        }
      }
      dph ^= 1u;
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 8) tmem_dealloc(tmem, tmem_cols);
}

static size_t stem_smem_bytes(int G, int n_mma, int cout) {
  return static_cast<size_t>(kStages) * (kStemA + kStemSegS) + static_cast<size_t>(G) * n_mma * 32 +
         static_cast<size_t>((G * cout + 1) & ~1) * 4 + (3 * kStages + 2 * kAcc) * 8 + 16;
}

cudaError_t init_stem_pp_kernel();
cudaError_t init_stem_kernel() {
  const cudaError_t e = cudaFuncSetAttribute(stem_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemLimit);
  return e != cudaSuccess ? e : init_stem_pp_kernel();
}

using EncodeTiledFnStem = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                       const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                       CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static cudaError_t launch_stem_toeplitz(const StemMember* members, int G, int x_stride, int Pm, int L, int out_q,
                                       int cout, int pad, __half* out, cudaStream_t st) {
  if (cout > 128 || cout % 8 || G < 1 || G > kMaxGroup || pad > 8 || (x_stride * 2) % 16) return cudaErrorInvalidValue;
  StemTcArgs a;
  // one 2-D view {L samples, rows} over every member's windows (they share the buffer and its row stride)
  const __half* base = members[0].x;
  for (int g = 1; g < G; ++g) base = members[g].x < base ? members[g].x : base;
  if ((reinterpret_cast<uintptr_t>(base) & 15) != 0) return cudaErrorInvalidValue;
  long long rows = 0;
  for (int g = 0; g < G; ++g) {
    a.m[g] = members[g];
    const long long off = members[g].x - base;
    if (off % x_stride) return cudaErrorInvalidValue;
    a.x_row0[g] = static_cast<int>(off / x_stride);
    rows = a.x_row0[g] + Pm > rows ? a.x_row0[g] + Pm : rows;
  }
  static EncodeTiledFnStem enc = nullptr;
  if (!enc) {
    void* fp = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return cudaErrorNotSupported;
    enc = reinterpret_cast<EncodeTiledFnStem>(fp);
  }
  CUtensorMap tm;
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(L), static_cast<cuuint64_t>(rows)};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(x_stride) * 2};
  const cuuint32_t box[2] = {kStemSegN, 1};
  const cuuint32_t estr[2] = {1, 1};
  if (enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<__half*>(base), dims, strides, box, estr,
          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return cudaErrorInvalidValue;
  a.G = G;
  a.Pm = Pm;
  a.x_stride = x_stride;
  a.L = L;
  a.out_qs = ilog2(out_q);
  a.out_lq = lq_Q(L, out_q);
  a.out_rows = act_rows_q(L, out_q);
  a.cout = cout;
  a.n_mma = cout < 16 ? 16 : cout;  // M=128 needs N >= 16
  a.pad = pad;
  a.mt_per_row = (a.out_rows + kBM - 1) / kBM;
  a.num_tiles = G * Pm * a.mt_per_row;
  a.out = out;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int grid = a.num_tiles < sms ? a.num_tiles : sms;
  return launch_pdl(stem_tc_kernel, dim3(grid), dim3(kStemThreads), stem_smem_bytes(G, a.n_mma, cout), st, tm, a);
}


// ---------------------------------------------------------------------------
// K3, phase-shifted-weights form (the default; HB_STEM=0 selects the builder
// kernel above).  Output position l = l0 + 8n + j, n in [0, 128) on the TMEM
// lanes, phase j in [0, 8) and channel c on the columns:
//   D[n, (j, c)] = sum_k' A[n, k'] B_j[c, k'],  k' in [0, 32)
//   A[n, k'] = x[l0 - 8 + 8n + k'],   B_j[c, k'] = W[c, k' - j - 8 + pad]
// A is the window segment itself: in the canonical K-major no-swizzle layout
// row n of a core matrix sits at 16 B * n (8 samples) and the next K core
// matrix at +16 B, so LBO = 16 B and SBO = 128 B turn the plain sample array
// (one 16-B aligned TMA segment per tile) into the Toeplitz operand; the
// sub-16-B shifts of the 8 phases live in 8 shifted weight images instead
// (TMA coordinates and descriptor addresses are 16-B granular).  Two K=16
// MMAs per phase.  With positions on the lanes the epilogue needs no
// transpose: a thread holds 8 channels of positions l and l + Q (phases j and
// j + Q), the two halves of one 32-B sector of the consumer's Q-phase layout:
// one 256-bit store (Q >= 8: two 128-bit stores into separate sub-planes).
// Warp roles as in K4b: 0 TMA, 1 MMA, 2 TMEM, 4-19 four epilogue warpgroups
// (buffer = ew & 1, half of the tile's (phase pair, 8-channel) units = ew >> 1).
constexpr int kStemPPThreads = 640;
constexpr int kStemSubs = 4;
constexpr int kStemPPStages = 8;
constexpr int kStemSeg = 2560;  // one tile's window segment: 5 boxes of 256 samples (1048 used)

struct StemPPArgs {
  StemMember m[kMaxGroup];
  int x_row0[kMaxGroup];
  int G, Pm, L, C, Ceff, pad, out_qs, out_lq, out_rows;
  int J, dd, paired, groups_per_blk, nt_per_row, num_tiles, n_stages;
  int dbg;  // HB_STEM_DBG (timing experiments only): 1 no stores, 2 no MMA, 4 no TMA
  int ug;   // epilogue units per TMEM load set: 4 (x32, one set; the default where it divides) or 1 (x8, two sets)
  __half* out;
  unsigned* flags;  // per tile counter (+1 per column half after its stores), null = none (see launch_stems)
};
// One launch = up to kStemSubs independent stems (member groups of different
// widths): CTAs [cta0[i], cta0[i+1]) run sub-problem i with its own smem
// layout.  A single launch gives the K4c chain ONE programmatic predecessor.
struct StemPPLaunch {
  CUtensorMap tm[kStemSubs];
  StemPPArgs a[kStemSubs];
  int cta0[kStemSubs + 1];
  int n_sub;
};

// (lo, hi) -> max(0, .) rounded to fp16, lo in the low half (one F2FP.RELU)
__device__ __forceinline__ uint32_t pack_relu_f16x2(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.relu.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}
__device__ __forceinline__ void tmem_ld8_nw(uint32_t taddr, uint32_t* r) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
}
__device__ __forceinline__ void st_global_256(void* p, const uint32_t (&v)[8]) {
  asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(v[0]), "r"(v[1]), "r"(v[2]),
               "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
               : "memory");
}

// Processing order k -> tile index: the group's members interleaved bed by bed
// (row = g * Pm + p in memory), so every member's first beds land first -- the
// K4c chain's per-member queues start on them while the stem still runs.
__device__ __forceinline__ int stem_tile_of(const StemPPArgs& a, int k) {
  const int ro = k / a.nt_per_row, rt = k - ro * a.nt_per_row;
  const int row = (ro % a.G) * a.Pm + ro / a.G;
  return row * a.nt_per_row + rt;
}

__global__ void __launch_bounds__(kStemPPThreads, 1) stem_pp_kernel(const __grid_constant__ StemPPLaunch S) {
  extern __shared__ __align__(1024) uint8_t smem[];
  int sub = 0;
  while (sub + 1 < S.n_sub && static_cast<int>(blockIdx.x) >= S.cta0[sub + 1]) ++sub;
  const StemPPArgs& a = S.a[sub];
  const CUtensorMap* tmX = &S.tm[sub];
  const int bid = static_cast<int>(blockIdx.x) - S.cta0[sub], nbk = S.cta0[sub + 1] - S.cta0[sub];
  const int wimg = a.Ceff * 32;                                   // one (phase, k-step) B image
  uint8_t* sW = smem;                                             // [G][8 phases][2 k-steps][k-half][Ceff][16 B]
  uint8_t* sX = sW + static_cast<size_t>(a.G) * 16 * wimg;        // [n_stages][kStemSeg]
  float* sBias = reinterpret_cast<float*>(sX + a.n_stages * kStemSeg);  // [G][Ceff]
  uint64_t* st_full = reinterpret_cast<uint64_t*>(sBias + a.G * a.Ceff);
  uint64_t* st_empty = st_full + a.n_stages;
  uint64_t* acc_full = st_empty + a.n_stages;
  uint64_t* acc_empty = acc_full + 2;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(acc_empty + 2);
  int* sUnit = reinterpret_cast<int*>(tmem_holder + 4);           // [64] epilogue unit -> (phase ja, c8)
  float* sRaw = reinterpret_cast<float*>(sUnit + 64);             // [G][16][C] staged taps

  const uint32_t warp = warp_id();
  const uint32_t lane = lane_id();
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int i = 0; i < a.n_stages; ++i) {
      mbar_init(&st_full[i], 1);
      mbar_init(&st_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&acc_full[i], 1);
      mbar_init(&acc_empty[i], 256);  // two epilogue warpgroups per buffer
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc(tmem_holder, 512);
  // B images and biases: constants, built before the dependency wait (taps
  // staged through shared memory so the global reads are coalesced)
  for (int i = tid; i < a.G * a.C * kTaps; i += kStemPPThreads) {  // -> [g][tap][channel]: conflict-free reads below
    const int g = i / (a.C * kTaps), rem = i - g * a.C * kTaps;
    const int n = rem >> 4, t = rem & 15;
    sRaw[(g * kTaps + t) * a.C + n] = a.m[g].w[rem];
  }
  for (int i = tid; i < a.G * a.Ceff; i += kStemPPThreads) {
    const int g = i / a.Ceff, c = i - g * a.Ceff;
    sBias[i] = c < a.C ? a.m[g].b[c] : 0.f;
  }
  if (tid < (a.J / 2) * (a.C / 8)) {  // unit u = (phase pair pi, 8-channel group c8), pair = (ja, ja + dd)
    const int pi = tid / (a.C / 8), c8 = tid - pi * (a.C / 8);
    sUnit[tid] = ((pi / a.dd) * 2 * a.dd + (pi % a.dd)) | (c8 << 8);
  }
  __syncthreads();
  const int rows_per_g = 8 * 2 * 2 * a.Ceff;  // 16-B rows: (phase, k-step, k-half, n)
  for (int i = tid; i < a.G * rows_per_g; i += kStemPPThreads) {
    const int g = i / rows_per_g;
    int r = i - g * rows_per_g;
    const int n = r % a.Ceff;
    r /= a.Ceff;
    const int h = r & 1, s = (r >> 1) & 1, j = r >> 2;
    __align__(16) __half v[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const int t = 16 * s + 8 * h + e - j - 8 + a.pad;
      v[e] = __float2half_rn(n < a.C && t >= 0 && t < kTaps ? sRaw[(g * kTaps + t) * a.C + n] : 0.f);
    }
    *reinterpret_cast<uint4*>(sW + static_cast<size_t>(i) * 16) = *reinterpret_cast<const uint4*>(v);
  }
  fence_proxy_async();  // B images are read by the tensor core
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;
  pdl_trigger();
  const int cols_buf = a.J * a.Ceff;

  if (warp == 0) {
    // ------------------------------------------------------------------ TMA
    if (lane == 0) {
      prefetch_tmap(tmX);
      pdl_wait();  // x is the window kernel's output
      int st = 0;
      uint32_t sph = 0;
      for (int k = bid; k < a.num_tiles; k += nbk) {
        const int tile = stem_tile_of(a, k);
        const int row = tile / a.nt_per_row, rt = tile - row * a.nt_per_row;
        const int nb = rt / a.groups_per_blk;
        const int g = row / a.Pm, p = row - g * a.Pm;
        mbar_wait(&st_empty[st], sph ^ 1u, 331);
        if (a.dbg & 4) {
          mbar_arrive(&st_full[st]);
        } else {
          mbar_arrive_expect_tx(&st_full[st], static_cast<uint32_t>(kStemSeg));
          uint8_t* dst = sX + st * kStemSeg;
          for (int b = 0; b < kStemSeg / 512; ++b)  // samples [l0 - 8, l0 + 1272), 16-B aligned start
            tma_load_2d(dst + 512 * b, tmX, &st_full[st], nb * 1024 - 8 + 256 * b, a.x_row0[g] + p);
        }
        if (++st == a.n_stages) {
          st = 0;
          sph ^= 1u;
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------------ MMA
    const uint32_t idesc = make_idesc_f16(kBM, a.Ceff);
    int st = 0, acc = 0;
    uint32_t sph = 0, accph = 0;
    for (int k = bid; k < a.num_tiles; k += nbk) {
      const int tile = stem_tile_of(a, k);
      const int row = tile / a.nt_per_row, rt = tile - row * a.nt_per_row;
      const int g = row / a.Pm, jg = rt % a.groups_per_blk;
      mbar_wait(&st_full[st], sph, 332);
      mbar_wait(&acc_empty[acc], accph ^ 1u, 333);
      tc_fence_after();
      const uint32_t xs = smem_u32(sX + st * kStemSeg);
      const uint32_t ws = smem_u32(sW + static_cast<size_t>(g) * 16 * wimg);
      const uint32_t d0 = tmem_base + static_cast<uint32_t>(acc * cols_buf);
      for (int jj = 0; jj < a.J; ++jj) {
        const int j = jg * a.J + jj;
#pragma unroll
        for (int s = 0; s < 2; ++s) {
          const uint64_t ad = make_desc(xs + static_cast<uint32_t>(32 * s), 16, 128);
          const uint64_t bd = make_desc(ws + static_cast<uint32_t>((j * 2 + s) * wimg), a.Ceff * 16, 128);
          if (!(a.dbg & 2) && elect_one())
            mma_f16_ss(d0 + static_cast<uint32_t>(jj * a.Ceff), ad, bd, idesc, static_cast<uint32_t>(s));
          __syncwarp();
        }
      }
      if (elect_one()) {
        mma_commit(&st_empty[st]);
        mma_commit(&acc_full[acc]);
      }
      __syncwarp();
      if (++st == a.n_stages) {
        st = 0;
        sph ^= 1u;
      }
      if (++acc == 2) {
        acc = 0;
        accph ^= 1u;
      }
    }
  } else if (warp >= 4) {
    // ------------------------------------------------------------- epilogue
    const int ew = (static_cast<int>(warp) - 4) >> 2;
    const int eb = ew & 1;
    const int wq = static_cast<int>(warp) & 3;
    const int n = wq * 32 + static_cast<int>(lane);  // TMEM lane = position block
    const int nc8 = a.C / 8;
    const int units = (a.J / 2) * nc8;  // (phase pair, 8-channel group)
    const int u_lo = (ew >> 1) ? (units + 1) / 2 : 0, u_hi = (ew >> 1) ? units : (units + 1) / 2;
    uint32_t accph = 0;
    pdl_wait();  // the output buffer may still be read by the previous tick's layers
    for (int k = bid + eb * nbk; k < a.num_tiles; k += 2 * nbk) {
      const int tile = stem_tile_of(a, k);
      const int row = tile / a.nt_per_row, rt = tile - row * a.nt_per_row;
      const int nb = rt / a.groups_per_blk, jg = rt - nb * a.groups_per_blk;
      const int g = row / a.Pm;
      const int lbase = nb * 1024 + 8 * n + jg * a.J;
      mbar_wait(&acc_full[eb], accph, 334);
      tc_fence_after();
      const uint32_t tb = tmem_base + (static_cast<uint32_t>(wq * 32) << 16) + static_cast<uint32_t>(eb * cols_buf);
      // Units run through two register sets: the next unit's TMEM loads are in
      // flight while the current one is converted and stored (tcgen05.wait::ld
      // waits for every outstanding load, so the sets alternate).
      auto unit_cols = [&](int u, uint32_t& ca, uint32_t& cb) {
        const int code = sUnit[u];
        ca = tb + static_cast<uint32_t>((code & 255) * a.Ceff + (code >> 8) * 8);
        cb = ca + static_cast<uint32_t>(a.dd * a.Ceff);
      };
      auto issue = [&](int u, uint32_t (&ra)[8], uint32_t (&rb)[8]) {
        uint32_t ca, cb;
        unit_cols(u, ca, cb);
        tmem_ld8_nw(ca, ra);
        tmem_ld8_nw(cb, rb);
      };
      auto store = [&](int u, const uint32_t* ra, const uint32_t* rb) {
        const int code = sUnit[u];
        const int ja = code & 255, c8 = code >> 8, jb = ja + a.dd;
        const float4 b0 = *reinterpret_cast<const float4*>(sBias + g * a.Ceff + c8 * 8);
        const float4 b1 = *reinterpret_cast<const float4*>(sBias + g * a.Ceff + c8 * 8 + 4);
        const float bias[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
        const int la = lbase + ja, lb = lbase + jb;
        uint32_t v[8];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          v[k] = pack_relu_f16x2(__uint_as_float(ra[2 * k]) + bias[2 * k], __uint_as_float(ra[2 * k + 1]) + bias[2 * k + 1]);
          v[4 + k] = pack_relu_f16x2(__uint_as_float(rb[2 * k]) + bias[2 * k], __uint_as_float(rb[2 * k + 1]) + bias[2 * k + 1]);
        }
        if (la >= a.L) v[0] = v[1] = v[2] = v[3] = 0u;  // the layout's zero padding [L, out_rows)
        if (lb >= a.L) v[4] = v[5] = v[6] = v[7] = 0u;
        if (a.dbg & 1) return;
        const size_t plane = static_cast<size_t>(row) * nc8 + c8;
        __half* pa = a.out + q_off(plane, a.out_qs, a.out_lq, la);
        if (a.paired && lb < a.out_rows) {
          st_global_256(pa, v);  // l and l + Q: adjacent rows of one sub-plane
        } else {
          if (la < a.out_rows) *reinterpret_cast<uint4*>(pa) = make_uint4(v[0], v[1], v[2], v[3]);
          if (lb < a.out_rows)
            *reinterpret_cast<uint4*>(a.out + q_off(plane, a.out_qs, a.out_lq, lb)) = make_uint4(v[4], v[5], v[6], v[7]);
        }
      };
      auto release = [&]() {
        tc_fence_before();
        mbar_arrive(&acc_empty[eb]);
      };
      if (a.ug == 4) {
        // four units (one phase pair, 32 consecutive columns per phase) per load
        // set: two waits per tile instead of eight
        uint32_t ra[32], rb[32];
        for (int u = u_lo; u < u_hi; u += 4) {
          uint32_t ca, cb;
          unit_cols(u, ca, cb);
          tmem_ld32_nw(ca, ra);
          tmem_ld32_nw(cb, rb);
          tmem_wait_ld();
          if (u + 4 >= u_hi) release();
#pragma unroll
          for (int k = 0; k < 4; ++k) store(u + k, ra + 8 * k, rb + 8 * k);
        }
      } else {
        uint32_t xa[8], xb[8], ya[8], yb[8];
        if (u_lo < u_hi) issue(u_lo, xa, xb);
        for (int u = u_lo; u < u_hi; u += 2) {
          tmem_wait_ld();  // set x (unit u) landed
          if (u + 1 < u_hi) {
            issue(u + 1, ya, yb);
          } else {
            release();
          }
          store(u, xa, xb);
          if (u + 1 >= u_hi) break;
          tmem_wait_ld();  // set y (unit u + 1) landed
          if (u + 2 < u_hi) {
            issue(u + 2, xa, xb);
          } else {
            release();
          }
          store(u + 1, ya, yb);
        }
      }
      if (u_lo >= u_hi) {  // no units for this warpgroup: release the buffer all the same
        tc_fence_before();
        mbar_arrive(&acc_empty[eb]);
      }
      if (a.flags) {  // publish this half of the tile for the K4c chain (counters grow by 2 per tick)
        named_bar_sync(2 + ew, 128);
        if (wq == 0 && lane == 0) {
          asm volatile("fence.proxy.async.global;" ::: "memory");
          __threadfence();
          asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(a.flags + tile), "r"(1u) : "memory");
        }
      }
      accph ^= 1u;
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_dealloc(tmem_base, 512);
}

cudaError_t init_stem_pp_kernel() {
  return cudaFuncSetAttribute(stem_pp_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemLimit);
}

// One group's stem as stem_pp sub-problems (several when the members' B
// images do not fit one CTA's shared memory).  Returns false when stem_pp does
// not serve the shape (w > 64: the Toeplitz builder kernel).
struct StemPPSub {
  CUtensorMap tm;
  StemPPArgs a;
  size_t smem;
};
static cudaError_t plan_stem_pp(const StemGroup& sg, std::vector<StemPPSub>* subs, bool* served) {
  const StemMember* members = sg.members;
  const int G = sg.G, x_stride = sg.x_stride, Pm = sg.Pm, L = sg.L, out_q = sg.out_q, cout = sg.cout, pad = sg.pad;
  *served = false;
  if (cout > 128 || cout % 8 || G < 1 || G > kMaxGroup || pad < 0 || pad > 8 || (x_stride * 2) % 16 ||
      out_q < 1 || out_q > 32 || (out_q & (out_q - 1)))
    return cudaErrorInvalidValue;
  StemPPArgs a;
  std::memset(&a, 0, sizeof(a));
  a.G = G;
  a.Pm = Pm;
  a.L = L;
  a.C = cout;
  a.Ceff = cout < 16 ? 16 : round_up(cout, 16);
  a.pad = pad;
  a.out_qs = ilog2(out_q);
  a.out_lq = lq_Q(L, out_q);
  a.out_rows = act_rows_q(L, out_q);
  a.J = 8;  // phases per tile (8, 4 or 2): J * Ceff TMEM columns per accumulator
  while (a.J > 2 && a.J * a.Ceff > 256) a.J >>= 1;
  // two phases per tile (C > 64) leave too little per accumulator: the builder kernel is faster there
  if (a.J < 4) return cudaSuccess;
  *served = true;
  a.dd = out_q < a.J ? out_q : 1;  // pair phases j, j + dd
  a.paired = a.dd == out_q;        // ... which are adjacent 16-B rows of the layout
  a.groups_per_blk = 8 / a.J;
  a.nt_per_row = ((a.out_rows + 1023) / 1024) * a.groups_per_blk;
  a.n_stages = kStemPPStages;
  a.dbg = getenv("HB_STEM_DBG") ? atoi(getenv("HB_STEM_DBG")) : 0;
  {  // units per TMEM load set (HB_STEM_UG): a warpgroup's units must split into whole sets of one phase pair
    // (measured, zero data: w32 group 64 beds 24.9 -> 23.1 us, 1024 beds 101 -> 91 us; c2 tick -0.8 %)
    const int want = getenv("HB_STEM_UG") ? atoi(getenv("HB_STEM_UG")) : 4;
    const int nc8 = cout / 8, units = (a.J / 2) * nc8;
    a.ug = (want == 4 && nc8 % 4 == 0 && units % 4 == 0 && ((units + 1) / 2) % 4 == 0) ? 4 : 1;
  }
  // members per launch: every member's 16 B images stay resident
  const size_t per_g = static_cast<size_t>(16) * a.Ceff * 32 + a.Ceff * 4 + static_cast<size_t>(cout) * kTaps * 4;
  const size_t fixed = static_cast<size_t>(a.n_stages) * kStemSeg + (2 * a.n_stages + 4) * 8 + 16 + 64 * 4;
  if ((a.J / 2) * (cout / 8) > 64) return cudaErrorInvalidValue;
  int gmax = static_cast<int>((kSmemLimit - fixed) / per_g);
  if (const char* cap = getenv("HB_STEM_GMAX")) gmax = std::min(gmax, std::max(1, atoi(cap)));  // test knob: split launches
  if (gmax < 1) return cudaErrorInvalidValue;
  static EncodeTiledFnStem enc = nullptr;
  if (!enc) {
    void* fp = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return cudaErrorNotSupported;
    enc = reinterpret_cast<EncodeTiledFnStem>(fp);
  }
  const size_t plane_elems = static_cast<size_t>(a.out_rows) * 8;
  for (int g0 = 0; g0 < G; g0 += gmax) {
    const int Gs = G - g0 < gmax ? G - g0 : gmax;
    const __half* base = members[g0].x;
    for (int g = 1; g < Gs; ++g) base = members[g0 + g].x < base ? members[g0 + g].x : base;
    if ((reinterpret_cast<uintptr_t>(base) & 15) != 0) return cudaErrorInvalidValue;
    long long rows = 0;
    for (int g = 0; g < Gs; ++g) {
      a.m[g] = members[g0 + g];
      const long long off = members[g0 + g].x - base;
      if (off % x_stride) return cudaErrorInvalidValue;
      a.x_row0[g] = static_cast<int>(off / x_stride);
      rows = a.x_row0[g] + Pm > rows ? a.x_row0[g] + Pm : rows;
    }
    StemPPSub sub;
    const cuuint64_t dims[2] = {static_cast<cuuint64_t>(L), static_cast<cuuint64_t>(rows)};
    const cuuint64_t strides[1] = {static_cast<cuuint64_t>(x_stride) * 2};
    const cuuint32_t box[2] = {256, 1};
    const cuuint32_t estr[2] = {1, 1};
    if (enc(&sub.tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<__half*>(base), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return cudaErrorInvalidValue;
    a.G = Gs;
    a.num_tiles = Gs * Pm * a.nt_per_row;
    a.out = sg.out + static_cast<size_t>(g0) * Pm * (cout / 8) * plane_elems;
    // the counters index the group's tiles (rows g * Pm + p over ALL its members)
    a.flags = sg.flags ? sg.flags + static_cast<size_t>(g0) * Pm * a.nt_per_row : nullptr;
    sub.a = a;
    sub.smem = fixed + Gs * per_g;
    subs->push_back(sub);
  }
  return cudaSuccess;
}

int stem_tiles_per_row(int L, int out_q, int cout) {
  const int Ceff = cout < 16 ? 16 : round_up(cout, 16);
  int J = 8;
  while (J > 2 && J * Ceff > 256) J >>= 1;
  if (J < 4) return 0;
  return ((act_rows_q(L, out_q) + 1023) / 1024) * (8 / J);
}

cudaError_t launch_stems(const StemGroup* groups, int n, int grid_cap, cudaStream_t st) {
  const int which = getenv("HB_STEM") ? atoi(getenv("HB_STEM")) : 1;  // read per launch (tests switch it)
  std::vector<StemPPSub> subs;
  for (int i = 0; i < n; ++i) {
    const StemGroup& sg = groups[i];
    bool served = false;
    if (which) {
      const cudaError_t e = plan_stem_pp(sg, &subs, &served);
      if (e != cudaSuccess) return e;
    }
    if (!served) {
      if (sg.flags) return cudaErrorInvalidValue;  // the builder kernel publishes no tile counters
      const cudaError_t e = launch_stem_toeplitz(sg.members, sg.G, sg.x_stride, sg.Pm, sg.L, sg.out_q, sg.cout, sg.pad,
                                                 sg.out, st);
      if (e != cudaSuccess) return e;
    }
  }
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int cap = grid_cap > 0 ? std::min(grid_cap, sms) : sms;
  for (size_t s0 = 0; s0 < subs.size(); s0 += kStemSubs) {
    const int ns = static_cast<int>(std::min<size_t>(kStemSubs, subs.size() - s0));
    StemPPLaunch S;
    std::memset(&S, 0, sizeof(S));
    S.n_sub = ns;
    long tot = 0;
    size_t smem = 0;
    for (int i = 0; i < ns; ++i) {
      S.tm[i] = subs[s0 + i].tm;
      S.a[i] = subs[s0 + i].a;
      tot += S.a[i].num_tiles;
      smem = std::max(smem, subs[s0 + i].smem);
    }
    // CTAs per sub-problem in proportion to its tiles (>= 1 each), at most one per tile
    const int grid = static_cast<int>(std::min<long>(tot, std::max(cap, ns)));
    int given = 0;
    S.cta0[0] = 0;
    for (int i = 0; i < ns; ++i) {
      int c = i + 1 == ns ? grid - given
                          : static_cast<int>(std::max<long>(1, static_cast<long>(grid) * S.a[i].num_tiles / tot));
      c = std::max(1, std::min(c, grid - given - (ns - 1 - i)));
      c = std::min(c, S.a[i].num_tiles);
      given += c;
      S.cta0[i + 1] = given;
    }
    const cudaError_t e = launch_pdl(stem_pp_kernel, dim3(given), dim3(kStemPPThreads), smem, st, S);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

cudaError_t launch_stem(const StemMember* members, int G, int x_stride, int Pm, int L, int out_q, int cout, int pad,
                        __half* out, cudaStream_t st) {
  StemGroup sg{members, G, x_stride, Pm, L, out_q, cout, pad, out, nullptr};
  return launch_stems(&sg, 1, 0, st);
}

}  // namespace hb
