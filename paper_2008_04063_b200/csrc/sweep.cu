// K6: the profiler sweep — exact ROC-AUC of every candidate ensemble's mean
// score over a recorded cohort, one CTA per candidate (persistent over
// candidates).
//
// Reference behaviour being reproduced (not code):
//   exhaustive_search: ens = (scores @ bits.T) / popcount, then
//   roc_auc_many(labels, ens)                 (pkg/src/zooserve/composer.py:614-619)
//   ensemble_roc_auc: roc_auc(labels, scores[:, idx].mean(axis=1))
//                                             (cohort.py:89-102)
//   roc_auc = (R_pos - n_pos(n_pos+1)/2) / (n_pos n_neg), R_pos the midrank
//   sum of the positives, ties averaged       (metrics.py:30-60)
//
// Exactness.  The ensemble mean is summed in fp64 in increasing column order
// and divided by the popcount — numpy's axis-1 mean order exactly, and
// OpenBLAS dgemm's order for every candidate outside its N%8 tail kernel
// (tests/golden pins the resulting AUCs bit-for-bit).  The rank statistic is
// an exact integer: with the smaller class sorted,
//   2U = sum over the larger class of (lo + hi)         [sorted class = negatives]
//   2U = sum over the larger class of (2m - lo - hi)    [sorted class = positives]
// where lo/hi = lower/upper bound of the element in the sorted class, i.e.
// "strictly below" counts twice and a tie once — the midrank convention.
// AUC = (2U/2) / (n_pos n_neg) is then the same correctly rounded division the
// reference performs.
//
// Layout on the device (built once per cohort): scores column-major
// [n][N] fp64 with the rows permuted so the smaller class occupies rows
// [0, m) — every per-candidate pass is a coalesced column read (L2-resident:
// 20000 x 10 x 8 B = 1.6 MB).  Keys are order-preserving uint64 images of the
// fp64 means (-0.0 canonicalised to +0.0, so the two compare equal as in numpy).
// The sorted class lives in shared memory (bitonic sort, m <= 16384) or, for
// larger cohorts, in a per-CTA global scratch region with the same code.
#include "../../include/holmes_b200.h"
#include "hb_kernels.cuh"

#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

namespace hb {

constexpr int kSweepThreads = 1024;
constexpr int kSmemKeys = 16384;   // 128 KB of sorted keys in shared memory
constexpr int kMaxCols = 256;      // selector width supported by the column list

__device__ __forceinline__ unsigned long long order_key(double v) {
  v = v + 0.0;  // -0.0 -> +0.0
  const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(v));
  return (b & 0x8000000000000000ull) ? ~b : (b | 0x8000000000000000ull);
}

struct SweepArgs {
  const double* cols;    // [n][N] permuted (smaller class first)
  int N, n, m;           // m = size of the smaller class
  int sorted_is_pos;     // 1: rows [0, m) are the positives
  int p2;                // power of two >= m (bitonic length)
  long long n_pos, n_neg;
  // candidates: either explicit bit rows [S][n] or integer values first + s
  const uint8_t* bits;
  unsigned long long first;
  long long S;
  unsigned long long* gscratch;  // [grid][p2] when p2 > kSmemKeys
  double* auc;                   // [S]
  double* ens_out;               // optional: ensemble means of candidate 0, original permuted order [N]
};

__device__ __forceinline__ int lower_bound_u64(const unsigned long long* a, int n, unsigned long long k) {
  int lo = 0, len = n;
  while (len > 0) {
    const int half = len >> 1;
    if (a[lo + half] < k) {
      lo += half + 1;
      len -= half + 1;
    } else {
      len = half;
    }
  }
  return lo;
}
__device__ __forceinline__ int upper_bound_u64(const unsigned long long* a, int n, unsigned long long k) {
  int lo = 0, len = n;
  while (len > 0) {
    const int half = len >> 1;
    if (a[lo + half] <= k) {
      lo += half + 1;
      len -= half + 1;
    } else {
      len = half;
    }
  }
  return lo;
}

// Register-level bitonic stages for one merge level k0 (k0 >= 128: only the
// j = 32..1 stages; k0 == 2: every level k = 2..64, i.e. sort each 64-key block).
__device__ __forceinline__ void cmp_keep(unsigned long long& e, int idx, int j, int k) {
  const unsigned long long o = __shfl_xor_sync(0xffffffffu, e, j);
  const bool lower = (idx & j) == 0, up = (idx & k) == 0;
  const unsigned long long mn = e < o ? e : o, mx = e < o ? o : e;
  e = (lower == up) ? mn : mx;
}
template <typename KeyPtr>
__device__ __forceinline__ void reg_pass(KeyPtr keys, int p2, int k0, int tid) {
  const int lane = tid & 31, warp = tid >> 5;
  for (int base = warp * 64; base < p2; base += (kSweepThreads / 32) * 64) {
    unsigned long long e0 = keys[base + lane], e1 = keys[base + 32 + lane];
    const int i0 = base + lane, i1 = base + 32 + lane;
    const int k_first = (k0 == 2) ? 2 : k0, k_last = (k0 == 2) ? 64 : k0;
    for (int k = k_first; k <= k_last; k <<= 1) {
      for (int j = (k >> 1 < 32 ? k >> 1 : 32); j > 0; j >>= 1) {
        if (j == 32) {
          const bool up = (i0 & k) == 0;
          if ((e0 > e1) == up) {
            const unsigned long long t = e0;
            e0 = e1;
            e1 = t;
          }
        } else {
          cmp_keep(e0, i0, j, k);
          cmp_keep(e1, i1, j, k);
        }
      }
    }
    keys[base + lane] = e0;
    keys[base + 32 + lane] = e1;
  }
}

// kShared: the sorted class lives in shared memory (typed LDS/STS); else in
// this CTA's global scratch slice (L2-resident), same code.
template <bool kShared>
__global__ void __launch_bounds__(kSweepThreads, 1) sweep_auc_kernel(const SweepArgs a) {
  extern __shared__ __align__(16) unsigned long long s_keys[];
  __shared__ int s_cols[kMaxCols];
  __shared__ int s_pop;
  __shared__ unsigned long long s_red[32];
  unsigned long long* keys = kShared ? s_keys : a.gscratch + static_cast<size_t>(blockIdx.x) * a.p2;
  const int tid = threadIdx.x;

  for (long long s = blockIdx.x; s < a.S; s += gridDim.x) {
    __syncthreads();
    if (tid == 0) {
      int pop = 0;
      if (a.bits) {
        const uint8_t* row = a.bits + static_cast<size_t>(s) * a.n;
        for (int k = 0; k < a.n; ++k)
          if (row[k]) s_cols[pop++] = k;
      } else {
        const unsigned long long v = a.first + static_cast<unsigned long long>(s);
        for (int k = 0; k < a.n; ++k)
          if ((v >> k) & 1ull) s_cols[pop++] = k;
      }
      s_pop = pop;
    }
    __syncthreads();
    const int pop = s_pop;
    const double dpop = static_cast<double>(pop);
    // ---- keys of the smaller class (+ sentinels up to p2)
    for (int j = tid; j < a.p2; j += kSweepThreads) {
      unsigned long long k = ~0ull;
      if (j < a.m) {
        double acc = 0.0;
        for (int c = 0; c < pop; ++c) acc = acc + a.cols[static_cast<size_t>(s_cols[c]) * a.N + j];
        const double mean = acc / dpop;
        if (a.ens_out && s == 0) a.ens_out[j] = mean;
        k = order_key(mean);
      }
      keys[j] = k;
    }
    __syncthreads();
    // ---- bitonic sort, ascending.  Stages with partner distance j <= 32 run
    // in registers: each warp owns 64-key blocks (2 keys per lane: idx and
    // idx + 32), j = 32 swaps within a lane, j < 32 by shuffle.  Only the
    // j >= 64 stages go through shared memory (45 instead of 105 passes at
    // 16384 keys).
    if (a.p2 >= 64) {
      reg_pass(keys, a.p2, 2, tid);  // k = 2..64: sort every 64-key block
      __syncthreads();
      for (int kk = 128; kk <= a.p2; kk <<= 1) {
        for (int j = kk >> 1; j >= 64; j >>= 1) {
          for (int i = tid; i < (a.p2 >> 1); i += kSweepThreads) {
            const int lo = 2 * i - (i & (j - 1));
            const int hi = lo + j;
            const unsigned long long x = keys[lo], y = keys[hi];
            const bool up = (lo & kk) == 0;
            if ((x > y) == up) {
              keys[lo] = y;
              keys[hi] = x;
            }
          }
          __syncthreads();
        }
        reg_pass(keys, a.p2, kk, tid);  // j = 32 .. 1 of this merge level
        __syncthreads();
      }
    } else {
      for (int kk = 2; kk <= a.p2; kk <<= 1) {
        for (int j = kk >> 1; j > 0; j >>= 1) {
          for (int i = tid; i < (a.p2 >> 1); i += kSweepThreads) {
            const int lo = 2 * i - (i & (j - 1));
            const int hi = lo + j;
            const unsigned long long x = keys[lo], y = keys[hi];
            const bool up = (lo & kk) == 0;
            if ((x > y) == up) {
              keys[lo] = y;
              keys[hi] = x;
            }
          }
          __syncthreads();
        }
      }
    }
    // ---- rank statistic over the larger class
    unsigned long long u2 = 0;
    for (int j = a.m + tid; j < a.N; j += kSweepThreads) {
      double acc = 0.0;
      for (int c = 0; c < pop; ++c) acc = acc + a.cols[static_cast<size_t>(s_cols[c]) * a.N + j];
      const double mean = acc / dpop;
      if (a.ens_out && s == 0) a.ens_out[j] = mean;
      const unsigned long long k = order_key(mean);
      const unsigned long long lo = lower_bound_u64(keys, a.m, k);
      const unsigned long long hi = upper_bound_u64(keys, a.m, k);
      u2 += a.sorted_is_pos ? (2ull * a.m - lo - hi) : (lo + hi);
    }
    for (int off = 16; off > 0; off >>= 1) u2 += __shfl_xor_sync(0xffffffffu, u2, off);
    if ((tid & 31) == 0) s_red[tid >> 5] = u2;
    __syncthreads();
    if (tid == 0) {
      unsigned long long t = 0;
      for (int w = 0; w < kSweepThreads / 32; ++w) t += s_red[w];
      const double u = static_cast<double>(t) * 0.5;
      a.auc[s] = u / static_cast<double>(a.n_pos * a.n_neg);
    }
  }
}

// ---------------------------------------------------------------------------
// Radix variant (m <= kRadixMax): the smaller class is sorted by an LSD radix
// sort in shared memory (8-bit digits, passes over constant bytes skipped),
// stable per pass: each warp owns a contiguous block of keys and ranks equal
// digits with __match_any_sync in lane order; offsets = exclusive scan over
// (digit, warp).  No power-of-two padding, ~6-8 passes instead of 105 bitonic
// stages.  Everything else (keys, exact rank statistic) is as above.
constexpr int kRadixMax = 12288;                       // keys: 2 x 96 KB + counters
constexpr int kRadixRounds = kRadixMax / kSweepThreads;  // keys per lane

__device__ __forceinline__ unsigned long long* radix_sort_block(unsigned long long* a, unsigned long long* b, int m,
                                                                unsigned* cnt, unsigned* base,
                                                                unsigned long long diff) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int per_warp = (m + 31) / 32;
  const int w0 = warp * per_warp;
  const int w1 = min(m, w0 + per_warp);
  const unsigned lt = (1u << lane) - 1u;
  for (int shift = 0; shift < 64; shift += 8) {
    if (((diff >> shift) & 0xFFull) == 0) continue;  // every key has the same byte here
    for (int i = tid; i < 32 * 256; i += kSweepThreads) cnt[i] = 0;
    __syncthreads();
    unsigned rank[kRadixRounds];
#pragma unroll
    for (int r = 0; r < kRadixRounds; ++r) {
      const int i = w0 + r * 32 + lane;
      const bool ok = i < w1;
      const int d = ok ? static_cast<int>((a[i] >> shift) & 0xFFull) : 256 + lane;
      const unsigned mm = __match_any_sync(0xffffffffu, d);
      const unsigned before = ok ? cnt[warp * 256 + d] : 0u;
      rank[r] = before + __popc(mm & lt);
      __syncwarp();
      if (ok && (mm & lt) == 0) cnt[warp * 256 + d] = before + __popc(mm);  // the group's first lane
      __syncwarp();
    }
    __syncthreads();
    if (tid < 256) {  // per digit: exclusive prefix over warps (in place), total -> base
      unsigned run = 0;
      for (int w = 0; w < 32; ++w) {
        const unsigned c = cnt[w * 256 + tid];
        cnt[w * 256 + tid] = run;
        run += c;
      }
      base[tid] = run;
    }
    __syncthreads();
    if (warp == 0) {  // exclusive scan of the 256 digit totals (8 per lane)
      unsigned v[8], sum = 0;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        v[k] = base[lane * 8 + k];
        sum += v[k];
      }
      unsigned incl = sum;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const unsigned t = __shfl_up_sync(0xffffffffu, incl, off);
        if (lane >= off) incl += t;
      }
      unsigned run = incl - sum;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        base[lane * 8 + k] = run;
        run += v[k];
      }
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < kRadixRounds; ++r) {
      const int i = w0 + r * 32 + lane;
      if (i < w1) {  // (the key is re-read from smem: registers are capped at 64 per thread here)
        const unsigned long long k = a[i];
        const int d = static_cast<int>((k >> shift) & 0xFFull);
        b[base[d] + cnt[warp * 256 + d] + rank[r]] = k;
      }
    }
    __syncthreads();
    unsigned long long* t = a;
    a = b;
    b = t;
  }
  return a;
}

__global__ void __launch_bounds__(kSweepThreads, 1) sweep_auc_radix_kernel(const SweepArgs a) {
  extern __shared__ __align__(16) unsigned long long s_ra[];  // [2][m] keys, then counters
  unsigned long long* ka = s_ra;
  unsigned long long* kb = s_ra + a.m;
  unsigned* cnt = reinterpret_cast<unsigned*>(s_ra + 2 * a.m);  // [32][256]
  unsigned* base = cnt + 32 * 256;                               // [256]
  __shared__ int s_cols[kMaxCols];
  __shared__ int s_pop;
  __shared__ unsigned long long s_red[32];
  const int tid = threadIdx.x;
  for (long long s = blockIdx.x; s < a.S; s += gridDim.x) {
    __syncthreads();
    if (tid == 0) {
      int pop = 0;
      if (a.bits) {
        const uint8_t* row = a.bits + static_cast<size_t>(s) * a.n;
        for (int k = 0; k < a.n; ++k)
          if (row[k]) s_cols[pop++] = k;
      } else {
        const unsigned long long v = a.first + static_cast<unsigned long long>(s);
        for (int k = 0; k < a.n; ++k)
          if ((v >> k) & 1ull) s_cols[pop++] = k;
      }
      s_pop = pop;
    }
    __syncthreads();
    const int pop = s_pop;
    const double dpop = static_cast<double>(pop);
    for (int j = tid; j < a.m; j += kSweepThreads) {
      double acc = 0.0;
      for (int c = 0; c < pop; ++c) acc = acc + a.cols[static_cast<size_t>(s_cols[c]) * a.N + j];
      const double mean = acc / dpop;
      if (a.ens_out && s == 0) a.ens_out[j] = mean;
      ka[j] = order_key(mean);
    }
    __syncthreads();
    // bytes that differ between keys (passes over the others are no-ops)
    unsigned long long diff = 0;
    const unsigned long long k0 = ka[0];
    for (int j = tid; j < a.m; j += kSweepThreads) diff |= ka[j] ^ k0;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) diff |= __shfl_xor_sync(0xffffffffu, diff, off);
    if ((tid & 31) == 0) s_red[tid >> 5] = diff;
    __syncthreads();
    diff = 0;
#pragma unroll
    for (int w = 0; w < kSweepThreads / 32; ++w) diff |= s_red[w];
    __syncthreads();
    const unsigned long long* keys = radix_sort_block(ka, kb, a.m, cnt, base, diff);
    unsigned long long u2 = 0;
    for (int j = a.m + tid; j < a.N; j += kSweepThreads) {
      double acc = 0.0;
      for (int c = 0; c < pop; ++c) acc = acc + a.cols[static_cast<size_t>(s_cols[c]) * a.N + j];
      const double mean = acc / dpop;
      if (a.ens_out && s == 0) a.ens_out[j] = mean;
      const unsigned long long k = order_key(mean);
      const int lo = lower_bound_u64(keys, a.m, k);
      // upper bound: walk the (usually empty) run of equal keys; a long run (tie-heavy
      // cohorts) falls back to the binary search
      int hi = lo;
      while (hi < a.m && hi - lo < 8 && keys[hi] == k) ++hi;
      if (hi - lo == 8) hi = upper_bound_u64(keys, a.m, k);
      u2 += a.sorted_is_pos ? (2ull * a.m - static_cast<unsigned long long>(lo + hi))
                            : static_cast<unsigned long long>(lo + hi);
    }
    for (int off = 16; off > 0; off >>= 1) u2 += __shfl_xor_sync(0xffffffffu, u2, off);
    if ((tid & 31) == 0) s_red[tid >> 5] = u2;
    __syncthreads();
    if (tid == 0) {
      unsigned long long t = 0;
      for (int w = 0; w < kSweepThreads / 32; ++w) t += s_red[w];
      const double u = static_cast<double>(t) * 0.5;
      a.auc[s] = u / static_cast<double>(a.n_pos * a.n_neg);
    }
  }
}

size_t radix_smem(int m) { return sizeof(unsigned long long) * 2 * m + sizeof(unsigned) * (32 * 256 + 256); }
bool radix_on(int m) {
  static const bool env_on = !(getenv("HB_SWEEP_RADIX") && atoi(getenv("HB_SWEEP_RADIX")) == 0);
  return env_on && m <= kRadixMax;
}

}  // namespace hb

// ------------------------------------------------------------------ C-ABI

using namespace hb;

struct hb_cohort {
  int device = 0, N = 0, n = 0, m = 0, sorted_is_pos = 0, p2 = 1, num_sms = 148;
  long long n_pos = 0, n_neg = 0;
  double* cols = nullptr;           // device [n][N] permuted
  std::vector<int> perm;            // device row r <- original row perm[r]
  unsigned long long* scratch = nullptr;
  int scratch_ctas = 0;
  uint8_t* d_bits = nullptr;
  size_t d_bits_cap = 0;
  double* d_auc = nullptr;
  size_t d_auc_cap = 0;
  double* d_ens = nullptr;
  cudaStream_t st = nullptr;
  std::string err;
};

namespace {

thread_local std::string g_cohort_err;

int cfail(hb_cohort* c, int code, const std::string& msg) {
  if (c) c->err = msg;
  g_cohort_err = msg;
  return code;
}

#define CKC(c, expr)                                                                                 \
  do {                                                                                               \
    cudaError_t e_ = (expr);                                                                         \
    if (e_ != cudaSuccess) return cfail(c, HB_E_CUDA, std::string(#expr) + ": " + cudaGetErrorString(e_)); \
  } while (0)

int grid_for(const hb_cohort* c, long long S) {
  long long g = c->num_sms;
  if (S < g) g = S;
  return static_cast<int>(g < 1 ? 1 : g);
}

int run(hb_cohort* c, const uint8_t* d_bits, unsigned long long first, long long S, double* host_auc,
        double* host_ens) {
  if (S <= 0) return HB_OK;
  cudaSetDevice(c->device);
  const int grid = grid_for(c, S);
  if (c->p2 > kSmemKeys && grid > c->scratch_ctas) {
    cudaFree(c->scratch);
    c->scratch = nullptr;
    CKC(c, cudaMalloc(&c->scratch, sizeof(unsigned long long) * static_cast<size_t>(grid) * c->p2));
    c->scratch_ctas = grid;
  }
  if (static_cast<size_t>(S) > c->d_auc_cap) {
    cudaFree(c->d_auc);
    c->d_auc = nullptr;
    CKC(c, cudaMalloc(&c->d_auc, sizeof(double) * S));
    c->d_auc_cap = static_cast<size_t>(S);
  }
  if (host_ens && !c->d_ens) CKC(c, cudaMalloc(&c->d_ens, sizeof(double) * c->N));
  SweepArgs a;
  std::memset(&a, 0, sizeof(a));
  a.cols = c->cols;
  a.N = c->N;
  a.n = c->n;
  a.m = c->m;
  a.sorted_is_pos = c->sorted_is_pos;
  a.p2 = c->p2;
  a.n_pos = c->n_pos;
  a.n_neg = c->n_neg;
  a.bits = d_bits;
  a.first = first;
  a.S = S;
  a.gscratch = c->scratch;
  a.auc = c->d_auc;
  a.ens_out = host_ens ? c->d_ens : nullptr;
  const size_t smem = (c->p2 <= kSmemKeys) ? sizeof(unsigned long long) * c->p2 : 0;
  if (radix_on(c->m))
    sweep_auc_radix_kernel<<<grid, kSweepThreads, radix_smem(c->m), c->st>>>(a);
  else if (c->p2 <= kSmemKeys)
    sweep_auc_kernel<true><<<grid, kSweepThreads, smem, c->st>>>(a);
  else
    sweep_auc_kernel<false><<<grid, kSweepThreads, smem, c->st>>>(a);
  CKC(c, cudaGetLastError());
  if (host_auc) CKC(c, cudaMemcpyAsync(host_auc, c->d_auc, sizeof(double) * S, cudaMemcpyDeviceToHost, c->st));
  std::vector<double> ens_perm;
  if (host_ens) {
    ens_perm.resize(c->N);
    CKC(c, cudaMemcpyAsync(ens_perm.data(), c->d_ens, sizeof(double) * c->N, cudaMemcpyDeviceToHost, c->st));
  }
  CKC(c, cudaStreamSynchronize(c->st));
  if (host_ens)
    for (int r = 0; r < c->N; ++r) host_ens[c->perm[r]] = ens_perm[r];
  return HB_OK;
}

}  // namespace

extern "C" {

const char* hb_cohort_last_error(const hb_cohort* c) { return c ? c->err.c_str() : g_cohort_err.c_str(); }

int hb_cohort_create(int device, const double* scores, const int8_t* labels, int N, int n, hb_cohort** out) {
  if (!scores || !labels || !out) return cfail(nullptr, HB_E_INVALID, "null argument");
  if (N < 1) return cfail(nullptr, HB_E_INVALID, "need at least one sample");
  if (n < 1 || n > kMaxCols) return cfail(nullptr, HB_E_INVALID, "cohort width must be in [1, 256]");
  long long npos = 0;
  for (int i = 0; i < N; ++i) {
    if (labels[i] != 0 && labels[i] != 1) return cfail(nullptr, HB_E_INVALID, "labels must be 0 or 1");
    npos += labels[i];
  }
  for (size_t i = 0; i < static_cast<size_t>(N) * n; ++i)
    if (!std::isfinite(scores[i])) return cfail(nullptr, HB_E_INVALID, "scores must be finite");
  const long long nneg = N - npos;
  if (npos == 0 || nneg == 0) return cfail(nullptr, HB_E_METRIC, "roc_auc needs both classes present");
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    return cfail(nullptr, HB_E_CUDA, "no CUDA device (there is no CPU fallback)");
  if (device < 0 || device >= ndev) return cfail(nullptr, HB_E_INVALID, "device ordinal out of range");
  cudaSetDevice(device);
  hb_cohort* c = new hb_cohort();
  c->device = device;
  c->N = N;
  c->n = n;
  c->n_pos = npos;
  c->n_neg = nneg;
  c->sorted_is_pos = npos <= nneg ? 1 : 0;
  c->m = static_cast<int>(c->sorted_is_pos ? npos : nneg);
  while (c->p2 < c->m) c->p2 <<= 1;
  cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device);
  const int8_t small_label = c->sorted_is_pos ? 1 : 0;
  c->perm.reserve(N);
  for (int i = 0; i < N; ++i)
    if (labels[i] == small_label) c->perm.push_back(i);
  for (int i = 0; i < N; ++i)
    if (labels[i] != small_label) c->perm.push_back(i);
  std::vector<double> colmajor(static_cast<size_t>(n) * N);
  for (int k = 0; k < n; ++k)
    for (int r = 0; r < N; ++r) colmajor[static_cast<size_t>(k) * N + r] = scores[static_cast<size_t>(c->perm[r]) * n + k];
  int rc = HB_OK;
  if (cudaStreamCreateWithFlags(&c->st, cudaStreamNonBlocking) != cudaSuccess ||
      cudaMalloc(&c->cols, sizeof(double) * colmajor.size()) != cudaSuccess ||
      cudaMemcpy(c->cols, colmajor.data(), sizeof(double) * colmajor.size(), cudaMemcpyHostToDevice) != cudaSuccess)
    rc = cfail(nullptr, HB_E_CUDA, "cohort device allocation failed");
  if (rc == HB_OK && c->p2 <= kSmemKeys &&
      cudaFuncSetAttribute(sweep_auc_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           static_cast<int>(sizeof(unsigned long long) * kSmemKeys)) != cudaSuccess)
    rc = cfail(nullptr, HB_E_CUDA, "sweep kernel attribute setup failed");
  if (rc == HB_OK && radix_on(c->m) &&
      cudaFuncSetAttribute(sweep_auc_radix_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           static_cast<int>(radix_smem(kRadixMax))) != cudaSuccess)
    rc = cfail(nullptr, HB_E_CUDA, "sweep radix kernel attribute setup failed");
  if (rc != HB_OK) {
    hb_cohort_destroy(c);
    return rc;
  }
  *out = c;
  return HB_OK;
}

int hb_cohort_destroy(hb_cohort* c) {
  if (!c) return HB_OK;
  cudaSetDevice(c->device);
  if (c->st) cudaStreamSynchronize(c->st);
  cudaFree(c->cols);
  cudaFree(c->scratch);
  cudaFree(c->d_bits);
  cudaFree(c->d_auc);
  cudaFree(c->d_ens);
  if (c->st) cudaStreamDestroy(c->st);
  delete c;
  return HB_OK;
}

int hb_cohort_auc(hb_cohort* c, const uint8_t* bits, int S, double* auc_out) {
  if (!c || (S > 0 && (!bits || !auc_out))) return cfail(c, HB_E_INVALID, "null argument");
  if (S < 0) return cfail(c, HB_E_INVALID, "S must be >= 0");
  for (size_t s = 0; s < static_cast<size_t>(S); ++s) {
    int pop = 0;
    for (int k = 0; k < c->n; ++k) {
      const uint8_t b = bits[s * c->n + k];
      if (b > 1) return cfail(c, HB_E_INVALID, "selector bits must be 0 or 1");
      pop += b;
    }
    if (pop == 0) return cfail(c, HB_E_EMPTY, "cannot score an empty ensemble");
  }
  if (S == 0) return HB_OK;
  cudaSetDevice(c->device);
  const size_t need = static_cast<size_t>(S) * c->n;
  if (need > c->d_bits_cap) {
    cudaFree(c->d_bits);
    c->d_bits = nullptr;
    CKC(c, cudaMalloc(&c->d_bits, need));
    c->d_bits_cap = need;
  }
  CKC(c, cudaMemcpyAsync(c->d_bits, bits, need, cudaMemcpyHostToDevice, c->st));
  return run(c, c->d_bits, 0, S, auc_out, nullptr);
}

int hb_cohort_auc_range(hb_cohort* c, unsigned long long first, long long count, double* auc_out) {
  if (!c || (count > 0 && !auc_out)) return cfail(c, HB_E_INVALID, "null argument");
  if (c->n > 63) return cfail(c, HB_E_INVALID, "integer selectors need n <= 63");
  if (count < 0) return cfail(c, HB_E_INVALID, "count must be >= 0");
  if (count == 0) return HB_OK;
  if (first == 0) return cfail(c, HB_E_EMPTY, "cannot score an empty ensemble");
  const unsigned long long last = first + static_cast<unsigned long long>(count) - 1;
  if (last >> c->n) return cfail(c, HB_E_INVALID, "selector value out of range for the cohort width");
  return run(c, nullptr, first, count, auc_out, nullptr);
}

int hb_cohort_ensemble(hb_cohort* c, const uint8_t* bits, double* ens_out, double* auc_out) {
  if (!c || !bits || !ens_out) return cfail(c, HB_E_INVALID, "null argument");
  int pop = 0;
  for (int k = 0; k < c->n; ++k) {
    if (bits[k] > 1) return cfail(c, HB_E_INVALID, "selector bits must be 0 or 1");
    pop += bits[k];
  }
  if (pop == 0) return cfail(c, HB_E_EMPTY, "cannot score an empty ensemble");
  cudaSetDevice(c->device);
  if (static_cast<size_t>(c->n) > c->d_bits_cap) {
    cudaFree(c->d_bits);
    c->d_bits = nullptr;
    CKC(c, cudaMalloc(&c->d_bits, c->n));
    c->d_bits_cap = c->n;
  }
  CKC(c, cudaMemcpyAsync(c->d_bits, bits, c->n, cudaMemcpyHostToDevice, c->st));
  double auc = 0.0;
  const int rc = run(c, c->d_bits, 0, 1, &auc, ens_out);
  if (rc == HB_OK && auc_out) *auc_out = auc;
  return rc;
}

int hb_sweep_auc(int device, const double* scores, const int8_t* labels, int N, int n, const uint32_t* selectors,
                 int S, double* auc_out) {
  if (n > 32) return cfail(nullptr, HB_E_INVALID, "hb_sweep_auc: n must be <= 32 (use hb_cohort_auc)");
  hb_cohort* c = nullptr;
  int rc = hb_cohort_create(device, scores, labels, N, n, &c);
  if (rc) return rc;
  std::vector<uint8_t> bits(static_cast<size_t>(S) * n);
  for (int s = 0; s < S; ++s)
    for (int k = 0; k < n; ++k) bits[static_cast<size_t>(s) * n + k] = (selectors[s] >> k) & 1u;
  rc = hb_cohort_auc(c, bits.data(), S, auc_out);
  if (rc) g_cohort_err = c->err;
  hb_cohort_destroy(c);
  return rc;
}

}  // extern "C"
