// K3: the stem conv (1 input channel -> w channels, 16 taps, "same" padding)
// + folded BN bias + ReLU on tcgen05 tensor cores.
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
            const float y0 = fmaxf(v[8 * h + k] + bias[g8 * 8 + k], 0.f);
            const float y1 = fmaxf(v[8 * h + k + 1] + bias[g8 * 8 + k + 1], 0.f);
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

cudaError_t init_stem_kernel() {
  return cudaFuncSetAttribute(stem_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemLimit);
}

using EncodeTiledFnStem = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                       const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                       CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

cudaError_t launch_stem(const StemMember* members, int G, int x_stride, int Pm, int L, int out_q, int cout, int pad,
                        __half* out, cudaStream_t st) {
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

}  // namespace hb
