// K7: arrival-curve construction for the latency profiler's queueing bound
// (SURVEY §8f "next" row 3).  The reference builds the empirical max-plus
// envelope of a query trace with quadratic numpy loops
// (pkg/src/zooserve/latency.py:198-239):
//   exact  (m <= 8000 events):  width[c-1] = min_i (ts[i+c-1] - ts[i]),   c = 1..m
//   binned (longer traces):     best[k-1]  = max_j (csum[j+k] - csum[j]), k = 1..n_bins
// Both are embarrassingly parallel over c / k: one CTA per output, a strided
// fp64 min / max reduction over the trace (L2-resident: 16k events = 128 kB).
// Subtractions are the same IEEE fp64 operations numpy performs and min / max
// are exact, so the device curve equals the reference's bit for bit.
#include "../../include/holmes_b200.h"
#include "hb_kernels.cuh"

#include <cmath>
#include <string>

namespace hb {

constexpr int kCurveThreads = 256;

__device__ __forceinline__ double warp_min(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// out[c-1] for c = blockIdx.x + 1 (+ gridDim.x strides): min over i of ts[i + c - 1] - ts[i]
__global__ void __launch_bounds__(kCurveThreads) exact_widths_kernel(const double* __restrict__ ts, int m,
                                                                      double* __restrict__ out) {
  __shared__ double red[kCurveThreads / 32];
  for (int c = blockIdx.x + 1; c <= m; c += gridDim.x) {
    double v = INFINITY;
    for (int i = threadIdx.x; i + c - 1 < m; i += kCurveThreads) v = fmin(v, ts[i + c - 1] - ts[i]);
    v = warp_min(v);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x < 32) {
      double w = threadIdx.x < kCurveThreads / 32 ? red[threadIdx.x] : INFINITY;
      w = warp_min(w);
      if (threadIdx.x == 0) out[c - 1] = w;
    }
    __syncthreads();
  }
}

// out[k-1] for k = 1..n: max over j of csum[j + k] - csum[j]   (csum has n + 1 entries)
__global__ void __launch_bounds__(kCurveThreads) binned_best_kernel(const double* __restrict__ csum, int n,
                                                                    double* __restrict__ out) {
  __shared__ double red[kCurveThreads / 32];
  for (int k = blockIdx.x + 1; k <= n; k += gridDim.x) {
    double v = -INFINITY;
    for (int j = threadIdx.x; j + k <= n; j += kCurveThreads) v = fmax(v, csum[j + k] - csum[j]);
    v = warp_max(v);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x < 32) {
      double w = threadIdx.x < kCurveThreads / 32 ? red[threadIdx.x] : -INFINITY;
      w = warp_max(w);
      if (threadIdx.x == 0) out[k - 1] = w;
    }
    __syncthreads();
  }
}

}  // namespace hb

using namespace hb;

namespace {
thread_local std::string g_curve_err;

int run_curve(bool exact, const double* in, int n_in, int n_out, double* out_host) {
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    g_curve_err = "no CUDA device (there is no CPU fallback)";
    return HB_E_CUDA;
  }
  double *d_in = nullptr, *d_out = nullptr;
  cudaStream_t st = nullptr;
  cudaError_t e = cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaMalloc(&d_in, sizeof(double) * n_in);
  if (e == cudaSuccess) e = cudaMalloc(&d_out, sizeof(double) * n_out);
  if (e == cudaSuccess) e = cudaMemcpyAsync(d_in, in, sizeof(double) * n_in, cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int grid = n_out < sms * 8 ? n_out : sms * 8;
    if (exact)
      exact_widths_kernel<<<grid, kCurveThreads, 0, st>>>(d_in, n_in, d_out);
    else
      binned_best_kernel<<<grid, kCurveThreads, 0, st>>>(d_in, n_out, d_out);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) e = cudaMemcpyAsync(out_host, d_out, sizeof(double) * n_out, cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  cudaFree(d_in);
  cudaFree(d_out);
  if (st) cudaStreamDestroy(st);
  if (e != cudaSuccess) {
    g_curve_err = cudaGetErrorString(e);
    return HB_E_CUDA;
  }
  return HB_OK;
}
}  // namespace

extern "C" {

const char* hb_curve_last_error(void) { return g_curve_err.c_str(); }

int hb_arrival_widths(const double* ts, int m, double* widths_out) {
  if (!ts || !widths_out || m < 1) {
    g_curve_err = "bad argument";
    return HB_E_INVALID;
  }
  for (int i = 1; i < m; ++i)
    if (!(ts[i] >= ts[i - 1])) {
      g_curve_err = "timestamps must be sorted non-decreasing";
      return HB_E_INVALID;
    }
  return run_curve(true, ts, m, m, widths_out);
}

int hb_binned_best(const double* csum, int n_bins, double* best_out) {
  if (!csum || !best_out || n_bins < 1) {
    g_curve_err = "bad argument";
    return HB_E_INVALID;
  }
  return run_curve(false, csum, n_bins + 1, n_bins, best_out);
}

}  // extern "C"
