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

// TMA-staged persistent variant (the default, K1/K2): grid = 3 CTAs per SM,
// each CTA walks streams blockIdx.x, +gridDim.x, ...  The part of a window
// that earlier ticks wrote (W - n_new samples, one contiguous run of the
// mirrored ring) is fetched by ONE bulk copy (cp.async.bulk, 16-B aligned: from
// r0 - A, A = r0 & 3) into a 2-deep shared-memory ring, issued one stream
// ahead, so the HBM reads of the next stream overlap this stream's reduction
// and stores; this tick's n_new samples come from the staging buffer (loaded
// into registers one stream ahead, appended to the ring and dropped into the
// shared window behind the bulk copy).  Window sample k is buffer float A + k.
// Statistics in one pass over conflict-free 16-B shared reads: sums of (x - K)
// and (x - K)^2, K = the window's first sample (the variance's cancellation
// stays small and a constant window gives exactly zero); two block barriers
// per stream.  Output: 8 samples per thread shifted by A (a compile-time
// selection in a 4-way switch around the output loop only -- per-A copies of
// the whole loop cost up to 8 us per launch in instruction fetch, ncu
// "no_instructions"), z-normalised, one 16-B fp16 store each.
constexpr int kWinTmaThreads = 256, kWinTmaQuads = 8;  // quads of 4 floats per thread: W + A <= 8192

// Output of one stream's window from the shared buffer (see window_tma_loop):
// octet o = buffer floats [8o + A, 8o + A + 8) -> 8 z-normalised halves, one
// 16-B store.
template <int A, int KO>
__device__ __forceinline__ void window_octets_out(const float* wb, int nq, int W, long long start, float rstd,
                                                  float shift, __half* __restrict__ dst, float* __restrict__ rw) {
  const int oct = (W + 7) / 8;
#pragma unroll
  for (int k = 0; k < KO; ++k) {
    const int o = static_cast<int>(threadIdx.x) + k * kWinTmaThreads;
    if (o >= oct) break;
    float t[12];
    *reinterpret_cast<float4*>(&t[0]) = 2 * o < nq ? *reinterpret_cast<const float4*>(wb + 8 * o) : make_float4(0.f, 0.f, 0.f, 0.f);
    *reinterpret_cast<float4*>(&t[4]) = 2 * o + 1 < nq ? *reinterpret_cast<const float4*>(wb + 8 * o + 4) : make_float4(0.f, 0.f, 0.f, 0.f);
    if constexpr (A != 0)
      *reinterpret_cast<float4*>(&t[8]) = 2 * o + 2 < nq ? *reinterpret_cast<const float4*>(wb + 8 * o + 8) : make_float4(0.f, 0.f, 0.f, 0.f);
    float x[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) x[j] = t[A + j];
    if (start + 8 * o < 0) {  // before the stream's first sample (first ticks only)
#pragma unroll
      for (int j = 0; j < 8; ++j)
        if (start + 8 * o + j < 0) x[j] = 0.f;
    }
    uint4 pk;
    __half2* h2 = reinterpret_cast<__half2*>(&pk);
    if (8 * o + 7 < W) {
#pragma unroll
      for (int j = 0; j < 4; ++j) h2[j] = __floats2half2_rn(fmaf(x[2 * j], rstd, shift), fmaf(x[2 * j + 1], rstd, shift));
    } else {
#pragma unroll
      for (int j = 0; j < 4; ++j)
        h2[j] = __floats2half2_rn(8 * o + 2 * j < W ? fmaf(x[2 * j], rstd, shift) : 0.f,
                                  8 * o + 2 * j + 1 < W ? fmaf(x[2 * j + 1], rstd, shift) : 0.f);
    }
    *reinterpret_cast<uint4*>(dst + 8 * o) = pk;
    if (rw) {
#pragma unroll
      for (int j = 0; j < 8; ++j)
        if (8 * o + j < W) rw[8 * o + j] = x[j];
    }
  }
}

template <int NB>
__device__ __forceinline__ void window_tma_loop(const float* __restrict__ staged, float* __restrict__ ring,
                                                int S, int n_new, int R, int W, int w0, int r0, int A, long long start,
                                                __half* __restrict__ xn, int leads, int xn_rows, int xn_stride,
                                                float* __restrict__ raw_out, float* __restrict__ stats,
                                                float* wbuf, int buf_floats, uint64_t* full, float* red) {
  constexpr int T = kWinTmaThreads, KO = kWinTmaQuads / 2, NW = T / 32;
  const int old_n = W - n_new;                                    // samples earlier ticks wrote
  const uint32_t old_bytes = static_cast<uint32_t>(((A + old_n + 3) & ~3) * 4);  // 16-B multiple
  const int n_iter = (S - static_cast<int>(blockIdx.x) + static_cast<int>(gridDim.x) - 1) / static_cast<int>(gridDim.x);
  auto issue = [&](int i) {  // thread 0: stream i's old part into buffer i % NB
    const int s = static_cast<int>(blockIdx.x) + i * static_cast<int>(gridDim.x);
    if (i >= n_iter || old_n <= 0) return;
    uint64_t* bar = &full[i % NB];
    float* dst = wbuf + static_cast<size_t>(i % NB) * buf_floats;
    const float* src = ring + static_cast<size_t>(s) * (R + W) + (r0 - A);
    fence_proxy_async();  // this buffer's previous generic reads/writes before the async write
    mbar_arrive_expect_tx(bar, old_bytes);
    for (uint32_t off = 0; off < old_bytes; off += 32768u)
      bulk_load(reinterpret_cast<uint8_t*>(dst) + off, reinterpret_cast<const uint8_t*>(src) + off,
                (old_bytes - off) < 32768u ? (old_bytes - off) : 32768u, bar);
  };
  if (threadIdx.x == 0)
    for (int i = 0; i < NB - 1; ++i) issue(i);
  const int nq = (A + W + 3) / 4;  // 16-B quads of the buffer that hold window samples
  // this tick's samples of the NEXT stream are loaded into registers one
  // iteration ahead (n_new <= NP*T; else loaded in place), so the staging
  // read's latency is off the per-stream critical path
  constexpr int NP = 2;
  const bool pre = n_new <= NP * T;
  float nxt[NP];
  auto load_new = [&](int i) {
    const int s = static_cast<int>(blockIdx.x) + i * static_cast<int>(gridDim.x);
    const float* src = staged + static_cast<size_t>(s) * n_new;
#pragma unroll
    for (int q = 0; q < NP; ++q) {
      const int j = static_cast<int>(threadIdx.x) + q * T;
      nxt[q] = (i < n_iter && j < n_new) ? src[j] : 0.f;
    }
  };
  if (pre) load_new(0);
  const int warp = static_cast<int>(threadIdx.x) >> 5, lane = static_cast<int>(threadIdx.x) & 31;
  for (int i = 0; i < n_iter; ++i) {
    const int s = static_cast<int>(blockIdx.x) + i * static_cast<int>(gridDim.x);
    float* rs = ring + static_cast<size_t>(s) * (R + W);
    float* wb = wbuf + static_cast<size_t>(i % NB) * buf_floats;
    float cur[NP];
#pragma unroll
    for (int q = 0; q < NP; ++q) cur[q] = nxt[q];
    if (pre) load_new(i + 1);
    if constexpr (NB == 1) {  // one buffer: every thread is done with stream i-1's before its refill
      if (i > 0) __syncthreads();
      if (threadIdx.x == 0) issue(i);
    }
    if (old_n > 0) mbar_wait(&full[i % NB], static_cast<uint32_t>(i / NB) & 1u, 130);
    auto put = [&](int j, float x) {  // append (+ mirror) and the window's newest samples
      int q = w0 + j;
      if (q >= R) q -= R;
      rs[q] = x;
      if (q < W) rs[R + q] = x;
      wb[A + old_n + j] = x;
    };
    if (pre) {
#pragma unroll
      for (int q = 0; q < NP; ++q) {
        const int j = static_cast<int>(threadIdx.x) + q * T;
        if (j < n_new) put(j, cur[q]);
      }
    } else {
      const float* src = staged + static_cast<size_t>(s) * n_new;
      for (int j = threadIdx.x; j < n_new; j += T) put(j, src[j]);
    }
    __syncthreads();  // (1) the window is complete in shared memory; every thread is past iteration i-1
    // buffer (i-1) % NB is no longer read by anyone: stream i + NB - 1 goes there
    if (NB > 1 && threadIdx.x == 0) issue(i + NB - 1);
    // Conflict-free shared reads: thread t holds the buffer's 16-B quads
    // i = t + k*T (float f of the buffer = window sample f - A).
    // Octet mapping: thread t owns output octets o = t + k*T (window samples
    // [8o, 8o+8) = buffer floats [8o + A, 8o + A + 8), inside buffer quads 2o,
    // 2o+1, 2o+2).  Stats run over the buffer's aligned octets (quads 2o, 2o+1;
    // floats outside the window masked), the output reads the three quads again
    // and shifts by A with a compile-time selection (a 4-way switch around the
    // output loop only: small code).  16-B fp16 stores.
    auto ldq = [&](int qi) {
      return qi < nq ? *reinterpret_cast<const float4*>(wb + 4 * qi) : make_float4(0.f, 0.f, 0.f, 0.f);
    };
    const float K = start < 0 ? 0.f : wb[A];
    float s1 = 0.f, s2 = 0.f;
#pragma unroll
    for (int k = 0; k < KO; ++k) {
      const int o = static_cast<int>(threadIdx.x) + k * T;
      const float4 q0 = ldq(2 * o), q1 = ldq(2 * o + 1);
      float d[8] = {q0.x - K, q0.y - K, q0.z - K, q0.w - K, q1.x - K, q1.y - K, q1.z - K, q1.w - K};
      const int f0 = 8 * o - A;  // window sample of this octet's first float
      if (f0 < 0 || f0 + 7 >= W || start + f0 < 0) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          if (f0 + j < 0 || f0 + j >= W) d[j] = 0.f;
          else if (start + f0 + j < 0) d[j] = -K;  // before the stream's first sample: a zero sample
        }
      }
      s1 += ((d[0] + d[1]) + (d[2] + d[3])) + ((d[4] + d[5]) + (d[6] + d[7]));
      s2 += (fmaf(d[0], d[0], d[1] * d[1]) + fmaf(d[2], d[2], d[3] * d[3])) +
            (fmaf(d[4], d[4], d[5] * d[5]) + fmaf(d[6], d[6], d[7] * d[7]));
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      s1 += __shfl_xor_sync(0xffffffffu, s1, off);
      s2 += __shfl_xor_sync(0xffffffffu, s2, off);
    }
    float* rd = red + (i & 1) * 2 * NW;  // double-buffered: no barrier needed before the next write
    if (lane == 0) {
      rd[warp] = s1;
      rd[NW + warp] = s2;
    }
    __syncthreads();  // (2)
    float t1 = 0.f, t2 = 0.f;
#pragma unroll
    for (int w = 0; w < NW; ++w) {  // fixed order
      t1 += rd[w];
      t2 += rd[NW + w];
    }
    const float inv_w = 1.f / static_cast<float>(W);
    const float m1 = t1 * inv_w;
    const float mean = K + m1;
    const float var = fmaxf(fmaf(-m1, m1, t2 * inv_w), 0.f);
    const float sd = sqrtf(var);
    const float rstd = 1.f / fmaxf(sd, 1e-6f);
    const float shift = -mean * rstd;
    const int p = s / leads, lead = s - (s / leads) * leads;
    __half* dst = xn + (static_cast<size_t>(lead) * xn_rows + p) * xn_stride;
    float* rw = raw_out ? raw_out + static_cast<size_t>(s) * W : nullptr;
    switch (A) {
      case 0: window_octets_out<0, KO>(wb, nq, W, start, rstd, shift, dst, rw); break;
      case 1: window_octets_out<1, KO>(wb, nq, W, start, rstd, shift, dst, rw); break;
      case 2: window_octets_out<2, KO>(wb, nq, W, start, rstd, shift, dst, rw); break;
      default: window_octets_out<3, KO>(wb, nq, W, start, rstd, shift, dst, rw); break;
    }
    if (stats && threadIdx.x == 0) {
      stats[2 * s] = mean;
      stats[2 * s + 1] = sd;
    }
  }
}

template <int NB, int MB>
__global__ void __launch_bounds__(kWinTmaThreads, MB) ingest_window_tma_kernel(
    const float* __restrict__ staged, float* __restrict__ ring, const long long* __restrict__ wpos_p, int S,
    int leads, int n_new, int R, int W, __half* __restrict__ xn, int xn_rows, int xn_stride,
    float* __restrict__ raw_out, float* __restrict__ stats, int buf_floats) {
  extern __shared__ __align__(128) float wbuf[];  // [NB][buf_floats]
  __shared__ __align__(8) uint64_t full[NB];
  __shared__ float red[4 * (kWinTmaThreads / 32)];
  if (threadIdx.x == 0) {
    for (int b = 0; b < NB; ++b) mbar_init(&full[b], 1);
    fence_barrier_init();
  }
  __syncthreads();
  pdl_wait();
  pdl_trigger();
  const unsigned long long wpos = static_cast<unsigned long long>(*wpos_p);
  const long long start = static_cast<long long>(wpos) + n_new - W;
  const int w0 = static_cast<int>(wpos % static_cast<unsigned>(R));
  int r0 = w0 + n_new - W;
  while (r0 < 0) r0 += R;
  while (r0 >= R) r0 -= R;
  // one code path for every window misalignment A (per-A template copies of this
  // loop quadrupled the code, and the instruction fetch of a cold copy cost up to
  // 8 us per launch: ncu "no_instructions" stalls)
  window_tma_loop<NB>(staged, ring, S, n_new, R, W, w0, r0, r0 & 3, start, xn, leads, xn_rows, xn_stride, raw_out,
                      stats, wbuf, buf_floats, full, red);
}

__global__ void advance_kernel(long long* wpos, int n) {
  pdl_wait();
  *wpos += n;
}

cudaError_t launch_ingest_window(const float* staged, float* ring, const long long* wpos, int P, int leads,
                                 int n_new, int R, int window, __half* xn, int xn_rows, float* raw_out, float* stats,
                                 cudaStream_t st) {
  const int xn_stride = round_up(window, 8);  // 16-B aligned rows (the stem's TMA view)
  // Default: the TMA-staged persistent kernel (16-B aligned ring rows, W <= 8189,
  // hop >= 2).  At 1024 beds (ncu, cold L2, tools/gpu_win5.sh) it moves the
  // window's 141.6 MB in 25.5-30 us (0.79 of the measured copy bandwidth) vs
  // 36 us for the scalar register kernel; HB_WIN_NB picks its buffers per CTA
  // (2 = one stream of look-ahead at 3 CTAs/SM, the default; 3 = two streams at
  // 2 CTAs/SM; 1 = none at 6 CTAs/SM, all measured slower).  HB_WIN=1 forces
  // the shared-memory kernel (also used for hb_ingest and windows > 8192
  // samples), HB_WIN=2 the scalar register kernel.
  static const int force = getenv("HB_WIN") ? atoi(getenv("HB_WIN")) : 0;
  const bool reg = xn != nullptr && n_new <= window && window <= 256 * 32 && force != 1;
  const bool tma = reg && force != 2 && R % 4 == 0 && window % 4 == 0 && n_new >= 2 &&
                   window + 3 <= kWinTmaThreads * kWinTmaQuads * 4;
  static const int win_nb = getenv("HB_WIN_NB") ? atoi(getenv("HB_WIN_NB")) : 2;
  if (tma) {
    static int num_sms = 0;
    if (!num_sms) {
      int dev = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, dev);
    }
    const int S = P * leads, buf_floats = round_up(window + 16, 32);
    auto go = [&](auto kern, int nb, int per_sm) {
      const int g = S < per_sm * num_sms ? S : per_sm * num_sms;
      return launch_pdl(kern, dim3(g), dim3(kWinTmaThreads), static_cast<size_t>(nb) * buf_floats * sizeof(float), st,
                        staged, ring, wpos, S, leads, n_new, R, window, xn, xn_rows, xn_stride, raw_out, stats,
                        buf_floats);
    };
    if (win_nb == 3) return go(ingest_window_tma_kernel<3, 2>, 3, 2);
    if (win_nb == 1) return go(ingest_window_tma_kernel<1, 6>, 1, 6);
    return go(ingest_window_tma_kernel<2, 3>, 2, 3);
  }
  if (reg)
    return launch_pdl(ingest_window_reg_kernel<256, 32>, dim3(P * leads), dim3(256), 0, st, staged, ring, wpos,
                      leads, n_new, R, window, xn, xn_rows, xn_stride, raw_out, stats);
  const size_t smem = xn ? static_cast<size_t>(window) * sizeof(float) : 0;
  return launch_pdl(ingest_window_kernel, dim3(P * leads), dim3(kWinThreads), smem, st, staged, ring, wpos, P, leads,
                    n_new, R, window, xn, xn_rows, xn_stride, raw_out, stats);
}

cudaError_t init_stream_kernels() {
  cudaError_t e = cudaFuncSetAttribute(ingest_window_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       200 * 1024);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(ingest_window_tma_kernel<3, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 110 * 1024);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(ingest_window_tma_kernel<2, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 74 * 1024);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(ingest_window_tma_kernel<1, 6>, cudaFuncAttributeMaxDynamicSharedMemorySize, 37 * 1024);
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
