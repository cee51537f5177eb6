// K1/K2 (ring append, window gather, z-normalisation) and K5 (head + ensemble
// aggregation).  Both memory-bound or tiny.  (K3, the stem, is stem_tc.cu.)
//
// Reference counterparts (behaviour, not code):
//   K1/K2 replace `Aggregator.add` buffering + `WindowBatch` materialisation
//         (`pkg/src/zooserve/runtime.py:76-115`): at hop == window the gathered
//         window k is exactly samples [k*W, (k+1)*W) of the stream.
//   K5    replaces `_WindowScorer.draw`'s mean latent (`runtime.py:131-136`)
//         and `ensemble_scores` (`cohort.py:89-97`): mean over the selected
//         members in zoo order, normalised by popcount; it also emits the mean
//         of member sigmoids (north star).  Fixed order, no float atomics.
#include "hb_kernels.cuh"
#include "hb_ptx.cuh"

#include <cstdint>
#include <cstdlib>

namespace hb {

constexpr int kWinThreads = 1024;

__device__ __forceinline__ float block_sum(float v, float* red) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  float s = 0.f;
  if (threadIdx.x == 0) {
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) s += red[i];  // fixed order
    red[32] = s;
  }
  __syncthreads();
  return red[32];
}

// One CTA per (patient, lead) stream.
__global__ void __launch_bounds__(kWinThreads) ingest_window_kernel(const float* __restrict__ staged,
                                                                    float* __restrict__ ring,
                                                                    const long long* __restrict__ wpos_p, int P,
                                                                    int leads, int n_new, int R, int W,
                                                                    __half* __restrict__ xn, int xn_rows, int xn_stride,
                                                                    float* __restrict__ raw_out,
                                                                    float* __restrict__ stats) {
  extern __shared__ float win[];  // [W] when gathering
  __shared__ float red[33];
  const int s = blockIdx.x;  // stream = p*leads + lead
  const int p = s / leads, lead = s % leads;
  pdl_wait();  // the ring cursor / rings / staging buffer belong to the previous tick's chain
  pdl_trigger();
  const long long wpos = *wpos_p;
  float* rs = ring + static_cast<size_t>(s) * (R + W);
  const float* src = staged + static_cast<size_t>(s) * n_new;
  const int w0 = static_cast<int>(wpos % R);
  for (int i = threadIdx.x; i < n_new; i += blockDim.x) {
    const float v = src[i];
    int j = w0 + i;
    if (j >= R) j -= R;
    rs[j] = v;
    if (j < W) rs[R + j] = v;  // mirror: any window is then a contiguous run of [0, R + W)
    if (xn != nullptr && i >= n_new - W) win[W - n_new + i] = v;  // newest samples straight from staging
  }
  if (xn == nullptr) return;
  // window = samples [end - W, end) with end = wpos + n_new; the part older
  // than this tick's append comes from the ring (written by earlier ticks)
  const long long start = wpos + n_new - W;
  const int old_n = W > n_new ? W - n_new : 0;
  int r0 = static_cast<int>(((start % R) + R) % R);
  for (int i = threadIdx.x; i < old_n; i += blockDim.x) {
    int j = r0 + i;
    if (j >= R) j -= R;
    win[i] = (start + i >= 0) ? rs[j] : 0.f;
  }
  __syncthreads();
  float part = 0.f;
  for (int i = threadIdx.x; i < W; i += blockDim.x) part += win[i];
  const float mean = block_sum(part, red) / static_cast<float>(W);
  float sq = 0.f;
  for (int i = threadIdx.x; i < W; i += blockDim.x) {
    const float d = win[i] - mean;
    sq += d * d;
  }
  const float var = block_sum(sq, red) / static_cast<float>(W);
  const float sd = sqrtf(var);
  const float rstd = 1.f / fmaxf(sd, 1e-6f);
  __half* dst = xn + (static_cast<size_t>(lead) * xn_rows + p) * xn_stride;
  if ((W & 1) == 0) {
    __half2* d2 = reinterpret_cast<__half2*>(dst);
    for (int i = threadIdx.x; i < W / 2; i += blockDim.x)
      d2[i] = __floats2half2_rn((win[2 * i] - mean) * rstd, (win[2 * i + 1] - mean) * rstd);
  } else {
    for (int i = threadIdx.x; i < W; i += blockDim.x) dst[i] = __float2half_rn((win[i] - mean) * rstd);
  }
  if (raw_out) {
    float* r = raw_out + static_cast<size_t>(s) * W;
    for (int i = threadIdx.x; i < W; i += blockDim.x) r[i] = win[i];
  }
  if (stats && threadIdx.x == 0) {
    stats[2 * s] = mean;
    stats[2 * s + 1] = sd;
  }
}

// Register-resident variant (ingest_window_reg): T threads per stream, thread
// t holds window samples t, t+T, ... (PER of them).  The ring carries a mirror
// of its first W slots after slot R-1, so after this tick's append the window
// is one contiguous run: PER loads at a constant stride from one base register
// (80 registers -> three 256-thread streams per SM).  Same arithmetic as the
// shared-memory kernel above except the two block sums (fixed order, T/32
// partials).
template <int T>
__device__ __forceinline__ float block_sum_t(float v, float* red) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) red[w] = v;
  __syncthreads();
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < T / 32; ++i) s += red[i];
  __syncthreads();
  return s;
}

template <int T, int PER>
__global__ void __launch_bounds__(T, 3) ingest_window_reg_kernel(const float* __restrict__ staged,
                                                              float* __restrict__ ring,
                                                              const long long* __restrict__ wpos_p, int leads,
                                                              int n_new, int R, int W, __half* __restrict__ xn,
                                                              int xn_rows, int xn_stride,
                                                              float* __restrict__ raw_out,
                                                              float* __restrict__ stats) {
  __shared__ float red[T / 32];
  const int s = blockIdx.x;
  const int p = s / leads, lead = s % leads;
  pdl_wait();
  pdl_trigger();
  const long long wpos = *wpos_p;
  float* rs = ring + static_cast<size_t>(s) * (R + W);
  const float* src = staged + static_cast<size_t>(s) * n_new;
  const long long start = wpos + n_new - W;
  const int r0 = static_cast<int>(((start % R) + R) % R);
  // append this tick's samples (and their mirror), then read the whole window
  // as one contiguous run of the mirrored ring: PER loads at a constant stride
  // from one base (few live registers -> more streams per SM)
  const int w0 = static_cast<int>(wpos % R);
  for (int i = threadIdx.x; i < n_new; i += T) {
    int j = w0 + i;
    if (j >= R) j -= R;
    const float v = src[i];
    rs[j] = v;
    if (j < W) rs[R + j] = v;
  }
  __syncthreads();
  const float* win = rs + r0 + threadIdx.x;
  float v[PER];
#pragma unroll
  for (int k = 0; k < PER; ++k) {
    const int i = threadIdx.x + k * T;
    v[k] = (i < W && start + i >= 0) ? win[k * T] : 0.f;
  }
  float part = 0.f;
#pragma unroll
  for (int k = 0; k < PER; ++k) part += v[k];
  const float mean = block_sum_t<T>(part, red) / static_cast<float>(W);
  float sq = 0.f;
#pragma unroll
  for (int k = 0; k < PER; ++k) {
    const int i = threadIdx.x + k * T;
    const float d = v[k] - mean;
    sq += (i < W) ? d * d : 0.f;
  }
  const float var = block_sum_t<T>(sq, red) / static_cast<float>(W);
  const float sd = sqrtf(var);
  const float rstd = 1.f / fmaxf(sd, 1e-6f);
  __half* dst = xn + (static_cast<size_t>(lead) * xn_rows + p) * xn_stride;
  float* rw = raw_out ? raw_out + static_cast<size_t>(s) * W : nullptr;
#pragma unroll
  for (int k = 0; k < PER; ++k) {
    const int i = threadIdx.x + k * T;
    if (i < W) {
      dst[i] = __float2half_rn((v[k] - mean) * rstd);
      if (rw) rw[i] = v[k];
    }
  }
  if (stats && threadIdx.x == 0) {
    stats[2 * s] = mean;
    stats[2 * s + 1] = sd;
  }
}

__global__ void advance_kernel(long long* wpos, int n) {
  pdl_wait();
  *wpos += n;
}

cudaError_t launch_ingest_window(const float* staged, float* ring, const long long* wpos, int P, int leads,
                                 int n_new, int R, int window, __half* xn, int xn_rows, float* raw_out, float* stats,
                                 cudaStream_t st) {
  const int xn_stride = round_up(window, 8);  // 16-B aligned rows (the stem's TMA view)
  // the register-resident variant whenever the window fits (measured faster at
  // 64 and 1024 beds: 13.7 vs 17.5 us, 87 vs 128 us); HB_WIN=1 forces the
  // shared-memory kernel (also used for hb_ingest and windows > 8192 samples).
  static const int force = getenv("HB_WIN") ? atoi(getenv("HB_WIN")) : 0;
  const bool reg = xn != nullptr && n_new <= window && window <= 256 * 32 && force != 1;
  if (reg)
    return launch_pdl(ingest_window_reg_kernel<256, 32>, dim3(P * leads), dim3(256), 0, st, staged, ring, wpos,
                      leads, n_new, R, window, xn, xn_rows, xn_stride, raw_out, stats);
  const size_t smem = xn ? static_cast<size_t>(window) * sizeof(float) : 0;
  return launch_pdl(ingest_window_kernel, dim3(P * leads), dim3(kWinThreads), smem, st, staged, ring, wpos, P, leads,
                    n_new, R, window, xn, xn_rows, xn_stride, raw_out, stats);
}

cudaError_t init_stream_kernels() {
  const cudaError_t e = cudaFuncSetAttribute(ingest_window_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             200 * 1024);
  return e != cudaSuccess ? e : init_stem_kernel();
}

cudaError_t launch_advance(long long* wpos, int n, cudaStream_t st) {
  return launch_pdl(advance_kernel, dim3(1), dim3(1), 0, st, wpos, n);
}

// ------------------------------------------------------------------ K5 aggregate
// One CTA per patient; warp w handles members w, w+8, ...; lanes sum the
// member's per-tile head partials (fixed shuffle tree), then thread 0 combines
// members in zoo order.
__global__ void __launch_bounds__(256) aggregate_kernel(const HeadMember* __restrict__ mem, int M, int P,
                                                        float* __restrict__ member_logits,
                                                        float* __restrict__ ens_prob,
                                                        float* __restrict__ ens_logit,
                                                        float* __restrict__ ens_sums, long long* wpos,
                                                        int advance) {
  __shared__ float s_logit[kMaxMembers];
  const int p = blockIdx.x;
  pdl_wait();
  pdl_trigger();
  // the tick's ring cursor advance rides on the last kernel of the tick
  if (wpos != nullptr && p == 0 && threadIdx.x == 0) *wpos += advance;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int m = warp; m < M; m += 8) {
    const HeadMember hm = mem[m];
    float s = 0.f;
    for (int i = lane; i < hm.mt; i += 32) s += hm.partial[static_cast<size_t>(p) * hm.mt + i];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
    if (lane == 0) s_logit[m] = hm.fc_b + s * hm.inv_len;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    float sp = 0.f, sl = 0.f;
    for (int m = 0; m < M; ++m) {
      const float lg = s_logit[m];
      member_logits[static_cast<size_t>(p) * M + m] = lg;
      sp += 1.f / (1.f + expf(-lg));
      sl += lg;
    }
    ens_prob[p] = sp / static_cast<float>(M);
    ens_logit[p] = sl / static_cast<float>(M);
    ens_sums[p] = sp;       // member-sharded serving reduces these across ranks
    ens_sums[P + p] = sl;
  }
}

cudaError_t launch_aggregate(const HeadMember* members_dev, int M, int P, float* member_logits, float* ens_prob,
                             float* ens_logit, float* ens_sums, long long* wpos, int advance, cudaStream_t st) {
  if (M < 1 || M > kMaxMembers) return cudaErrorInvalidValue;
  return launch_pdl(aggregate_kernel, dim3(P), dim3(256), 0, st, members_dev, M, P, member_logits, ens_prob,
                    ens_logit, ens_sums, wpos, advance);
}

// Member-sharded finish: sums[2][P] reduced over ranks -> means over the total popcount.
__global__ void finalize_kernel(const float* __restrict__ sums, int P, float inv_m, float* __restrict__ prob,
                                float* __restrict__ logit) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= P) return;
  prob[p] = sums[p] * inv_m;
  logit[p] = sums[P + p] * inv_m;
}

cudaError_t launch_finalize(const float* sums, int P, int m_total, float* prob, float* logit, cudaStream_t st) {
  finalize_kernel<<<(P + 255) / 256, 256, 0, st>>>(sums, P, 1.f / static_cast<float>(m_total), prob, logit);
  return cudaGetLastError();
}

}  // namespace hb
