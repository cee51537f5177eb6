// K3: the stem conv (1 input channel -> w channels, 16 taps, "same" padding)
// + folded BN bias + ReLU on tcgen05 tensor cores.
//
// With one input channel the whole 16-tap receptive field is exactly one
// kind::f16 K-step, so a tile of 128 output positions is ONE MMA:
//   D[m, c] = sum_t A[m, t] W[c, t],  A[m, t] = x[l0 + m + t - pad]
// A is the Toeplitz (im2col) view of the normalised window; rows overlap by
// one sample, which no TMA box or descriptor stride can express, so each
// thread writes its own row (32 B) into the canonical K-major no-swizzle
// layout from a staged window segment.  The kernel is bound by writing the
// w-channel output (HBM), not by math: 2*w*16 FLOP per 2*w output bytes.
//
// 128 threads per CTA (thread r <-> TMEM lane r <-> position l0 + r), several
// CTAs per SM overlap each other's phases; persistent over tiles.
#include "hb_kernels.cuh"
#include "hb_ptx.cuh"

namespace hb {

constexpr int kStemTcThreads = 128;
constexpr int kStemSeg = kBM + kTaps;  // window samples one tile touches (143 used)
constexpr int kStemSmemCap = 48 * 1024;  // largest dynamic-smem pad (4 CTAs/SM at 128 TMEM columns)

struct StemTcArgs {
  StemMember m[kMaxGroup];
  int G, Pm, x_stride, L, out_qs, out_lq, out_rows, cout, n_mma, pad, mt_per_row, num_tiles;
  __half* out;
};

// Thread r's share (samples r and r + 128) of a tile's window segment.
__device__ __forceinline__ void seg_load(const StemTcArgs& a, int tile, int r, __half* seg) {
  const int row = tile / a.mt_per_row;
  const int mt = tile - row * a.mt_per_row;
  const int g = row / a.Pm, p = row - g * a.Pm;
  const __half* x = a.m[g].x + static_cast<size_t>(p) * a.x_stride;
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const int i = r + k * kStemTcThreads;
    const int pos = mt * kBM + i - a.pad;
    seg[k] = (i < kStemSeg && pos >= 0 && pos < a.L) ? x[pos] : __float2half_rn(0.f);
  }
}

__global__ void __launch_bounds__(kStemTcThreads) stem_tc_kernel(const __grid_constant__ StemTcArgs a) {
  __shared__ __align__(1024) uint8_t sA[kBM * 32];        // 2 K-halves x 128 rows x 16 B
  __shared__ __align__(1024) uint8_t sB[2 * 128 * 16];    // 2 K-halves x <=128 rows x 16 B
  __shared__ __half sx[kStemSeg];
  __shared__ float sbias[128];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tmem_holder;
  const int r = threadIdx.x;
  const uint32_t warp = warp_id();
  uint32_t cols = 32;
  while (cols < static_cast<uint32_t>(a.n_mma)) cols <<= 1;
  if (r == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc(&tmem_holder, cols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_holder;
  const uint32_t idesc = make_idesc_f16(kBM, a.n_mma);
  const uint64_t adesc = make_desc(smem_u32(sA), kBM * 16, 128);
  const uint64_t bdesc = make_desc(smem_u32(sB), a.n_mma * 16, 128);
  pdl_wait();  // x is the window kernel's output
  pdl_trigger();
  int cur_g = -1;
  uint32_t phase = 0;
  __half seg[2];
  for (int tile = blockIdx.x; tile < a.num_tiles; tile += gridDim.x) {
    const int row = tile / a.mt_per_row;  // g * Pm + p
    const int mt = tile - row * a.mt_per_row;
    const int g = row / a.Pm, p = row - g * a.Pm;
    const int l0 = mt * kBM;
    const StemMember& mb = a.m[g];
    if (g != cur_g) {  // this member's weights as the B operand image (fp16) + bias
      for (int i = r; i < a.n_mma * 16; i += kStemTcThreads) {
        const int n = i >> 4, t = i & 15;
        const float w = n < a.cout ? mb.w[n * kTaps + t] : 0.f;
        reinterpret_cast<__half*>(sB)[((t >> 3) * a.n_mma + n) * 8 + (t & 7)] = __float2half_rn(w);
      }
      for (int i = r; i < a.cout; i += kStemTcThreads) sbias[i] = mb.b[i];
      cur_g = g;
    }
    if (tile == static_cast<int>(blockIdx.x)) seg_load(a, tile, r, seg);  // first tile: no prefetch yet
    sx[r] = seg[0];
    if (r + kStemTcThreads < kStemSeg) sx[r + kStemTcThreads] = seg[1];
    __syncthreads();
    {  // row r of the Toeplitz tile: samples r .. r+15 of the segment
      __align__(16) __half v[16];
#pragma unroll
      for (int t = 0; t < 16; ++t) v[t] = sx[r + t];
      const uint4* v4 = reinterpret_cast<const uint4*>(v);
      const int off = (r >> 3) * 128 + (r & 7) * 16;
      *reinterpret_cast<uint4*>(sA + off) = v4[0];
      *reinterpret_cast<uint4*>(sA + kBM * 16 + off) = v4[1];
    }
    fence_proxy_async();  // generic-proxy smem writes -> visible to the tensor core
    __syncthreads();
    if (warp == 0) {
      tc_fence_after();
      if (elect_one()) {
        mma_f16_ss(tmem, adesc, bdesc, idesc, 0u);
        mma_commit(&bar);
      }
      __syncwarp();
    }
    // prefetch the next tile's window segment while the MMA runs
    if (tile + static_cast<int>(gridDim.x) < a.num_tiles) seg_load(a, tile + gridDim.x, r, seg);
    mbar_wait(&bar, phase);
    phase ^= 1;
    tc_fence_after();
    const int l = l0 + r;
    const bool in_buf = l < a.out_rows, valid = l < a.L;
    const uint32_t taddr = tmem + (static_cast<uint32_t>(warp * 32) << 16);
    for (int c16 = 0; c16 * 16 < a.cout; ++c16) {  // warp-collective loads: every lane takes part
      float v[16];
      tmem_ld16(taddr + static_cast<uint32_t>(c16 * 16), v);
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int g8 = c16 * 2 + h;
        if (g8 * 8 >= a.cout || !in_buf) break;
        uint4 pk;
        __half2* o2 = reinterpret_cast<__half2*>(&pk);
#pragma unroll
        for (int k = 0; k < 8; k += 2) {
          const float y0 = fmaxf(v[8 * h + k] + sbias[g8 * 8 + k], 0.f);
          const float y1 = fmaxf(v[8 * h + k + 1] + sbias[g8 * 8 + k + 1], 0.f);
          o2[k / 2] = valid ? __floats2half2_rn(y0, y1) : __floats2half2_rn(0.f, 0.f);
        }
        *reinterpret_cast<uint4*>(a.out + q_off(static_cast<size_t>(row) * (a.cout / 8) + g8, a.out_qs, a.out_lq, l)) = pk;
      }
    }
    tc_fence_before();
    __syncthreads();  // sA, sx and the accumulator are reused by the next tile
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) tmem_dealloc(tmem, cols);
}

cudaError_t init_stem_kernel() {
  return cudaFuncSetAttribute(stem_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kStemSmemCap);
}

cudaError_t launch_stem(const StemMember* members, int G, int x_stride, int Pm, int L, int out_q, int cout, int pad,
                        __half* out, cudaStream_t st) {
  if (cout > 128 || cout % 8 || G < 1 || G > kMaxGroup) return cudaErrorInvalidValue;
  StemTcArgs a;
  for (int g = 0; g < G; ++g) a.m[g] = members[g];
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
  // Residency per SM is capped through (unused) dynamic shared memory so all
  // resident CTAs' TMEM allocations fit at once: 512 / columns, at most 12
  // (register file).  More CTAs hide the per-tile load -> MMA -> store chain.
  int cols = 32;
  while (cols < a.n_mma) cols <<= 1;
  int per_sm = 512 / cols;
  if (per_sm > 12) per_sm = 12;
  const size_t pad_smem = 232448 / per_sm - 10 * 1024;
  int grid = sms * per_sm;
  if (grid > a.num_tiles) grid = a.num_tiles;
  return launch_pdl(stem_tc_kernel, dim3(grid), dim3(kStemTcThreads), pad_smem, st, a);
}

}  // namespace hb
