// metrics.cu — per-model test metrics on the device.
//
// Mirrors bbcount/metrics.py as experiment.train_one applies it
// (experiment.py:128-152):
//   mse      = mean((pred - actual)^2) in the normalised space   (metrics.py:33-38)
//   pearson  = sample Pearson of the de-normalised predictions
//              pred*(y_max-y_min)+y_min (traces.py:311-313) vs the raw test
//              counts; undefined (NaN here, None there) when either vector
//              is constant; clamped to [-1, 1]                     (metrics.py:41-52)
//   spearman = Pearson of fractional ranks, ties -> average rank  (metrics.py:55-76)
// Task fields (bbml_pred_task reused): row_begin = first test row of the
// model's series in actual_norm / actual_raw, w_offset = first prediction of
// the model in pred, norm_offset = [x_min(d), x_max(d), y_min, y_max] in norm,
// out_offset = 4 outputs {mse, pearson, spearman, spearman_done}, n = rows.
// One CTA per model.  Ranks come from a bitonic sort of (value, index) in
// shared memory -- index as the tie-break gives numpy's stable argsort order;
// tie groups then get 0.5*(first+last)+1.  Models with more than
// kMetricsMaxN test rows get out[3] = 0 (Spearman left to the caller).
#include <algorithm>

#include "common.cuh"
#include "launch.h"

namespace bbml {

constexpr int MET_NT = 256;
constexpr int kMetricsMaxN = 4096;

__device__ __forceinline__ double met_sum(double v, double* red) {
#pragma unroll
  for (int m = 16; m >= 1; m >>= 1) v += __shfl_xor_sync(0xffffffffu, v, m);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  double s = 0.0;
#pragma unroll
  for (int w = 0; w < MET_NT / 32; ++w) s += red[w];
  return s;
}

// Pearson of a[0..n) and b[0..n) (shared or global), NaN when undefined
__device__ double met_pearson(const double* a, const double* b, int n, double* red) {
  double sa = 0.0, sb = 0.0;
  for (int i = threadIdx.x; i < n; i += MET_NT) {
    sa += a[i];
    sb += b[i];
  }
  const double ma = met_sum(sa, red) / n;
  const double mb = met_sum(sb, red) / n;
  double ab = 0.0, aa = 0.0, bb = 0.0;
  for (int i = threadIdx.x; i < n; i += MET_NT) {
    const double da = a[i] - ma, db = b[i] - mb;
    ab = fma(da, db, ab);
    aa = fma(da, da, aa);
    bb = fma(db, db, bb);
  }
  const double sab = met_sum(ab, red);
  const double saa = met_sum(aa, red);
  const double sbb = met_sum(bb, red);
  const double den = sqrt(saa) * sqrt(sbb);
  if (den == 0.0) return __longlong_as_double(0x7ff8000000000000LL);
  return fmin(1.0, fmax(-1.0, sab / den));
}

// fractional ranks of v[0..n) into rk[0..n); key/idx: shared sort buffers of
// size np (power of two >= n)
__device__ void met_ranks(const double* v, int n, int np, double* key, int* idx, double* rk) {
  for (int i = threadIdx.x; i < np; i += MET_NT) {
    key[i] = i < n ? v[i] : __longlong_as_double(0x7ff0000000000000LL);
    idx[i] = i;
  }
  __syncthreads();
  for (int k = 2; k <= np; k <<= 1)
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < np; i += MET_NT) {
        const int l = i ^ j;
        if (l > i) {
          const bool up = (i & k) == 0;
          const double ki = key[i], kl = key[l];
          const int ii = idx[i], il = idx[l];
          const bool gt = ki > kl || (ki == kl && ii > il);
          if (gt == up) {
            key[i] = kl;
            key[l] = ki;
            idx[i] = il;
            idx[l] = ii;
          }
        }
      }
      __syncthreads();
    }
  for (int s = threadIdx.x; s < n; s += MET_NT) {
    int lo = s, hi = s;
    while (lo > 0 && key[lo - 1] == key[s]) --lo;
    while (hi + 1 < n && key[hi + 1] == key[s]) ++hi;
    rk[idx[s]] = 0.5 * (lo + hi) + 1.0;
  }
  __syncthreads();
}

__global__ void __launch_bounds__(MET_NT)
    metrics_kernel(const bbml_pred_task* __restrict__ tasks, const double* __restrict__ pred,
                   const double* __restrict__ actual_norm, const double* __restrict__ actual_raw,
                   const double* __restrict__ norm, double* __restrict__ out, int cap) {
  extern __shared__ __align__(16) unsigned char met_smem[];
  __shared__ double red[MET_NT / 32];
  const bbml_pred_task tk = tasks[blockIdx.x];
  const int n = tk.n;
  double* o = out + tk.out_offset;
  const double* p = pred + tk.w_offset;  // predictions of this model
  const double* an = actual_norm + tk.row_begin;
  const double* ar = actual_raw + tk.row_begin;
  const double nan = __longlong_as_double(0x7ff8000000000000LL);
  if (n <= 0) {
    if (threadIdx.x == 0) o[0] = o[1] = o[2] = nan, o[3] = 1.0;
    return;
  }
  double se = 0.0;
  for (int i = threadIdx.x; i < n; i += MET_NT) {
    const double e = p[i] - an[i];
    se = fma(e, e, se);
  }
  const double mse = met_sum(se, red) / n;
  const double ylo = norm[tk.norm_offset + 2 * tk.d], yhi = norm[tk.norm_offset + 2 * tk.d + 1];
  const bool fits = n <= cap;
  int np = 1;
  while (np < n) np <<= 1;
  double* key = (double*)met_smem;  // np
  double* pr = key + cap;           // n: de-normalised predictions
  double* ra = pr + cap;            // n: ranks of pr
  double* rb = ra + cap;            // n: ranks of actual_raw
  int* idx = (int*)(rb + cap);      // np
  double pear = nan, spear = nan;
  if (n >= 2) {
    if (fits) {
      for (int i = threadIdx.x; i < n; i += MET_NT)
        pr[i] = __dadd_rn(__dmul_rn(p[i], __dsub_rn(yhi, ylo)), ylo);
      __syncthreads();
      pear = met_pearson(pr, ar, n, red);
      met_ranks(pr, n, np, key, idx, ra);
      met_ranks(ar, n, np, key, idx, rb);
      spear = met_pearson(ra, rb, n, red);
    }
  }
  if (threadIdx.x == 0) {
    o[0] = mse;
    o[1] = pear;
    o[2] = spear;
    o[3] = (fits || n < 2) ? 1.0 : 0.0;
  }
}

bbml_status metrics_launch(const bbml_pred_task* tasks, int32_t n_tasks, const double* pred,
                           const double* actual_norm, const double* actual_raw, const double* norm,
                           double* out, cudaStream_t stream) {
  int max_n = 0;
  for (int i = 0; i < n_tasks; ++i) {
    const bbml_pred_task& t = tasks[i];
    max_n = std::max(max_n, t.n);
    if (t.n < 0 || t.d < 1 || t.d > BBML_MAX_INPUTS || t.row_begin < 0 || t.w_offset < 0 ||
        t.out_offset < 0 || t.norm_offset < 0) {
      set_error("metrics task %d: invalid field", i);
      return BBML_ERR_INVALID;
    }
  }
  if (n_tasks == 0) return BBML_OK;
  ScratchBuffer scratch(stream);
  bbml_pred_task* d_tasks = nullptr;
  bbml_status st;
  if ((st = scratch.alloc(&d_tasks, n_tasks)) != BBML_OK) return st;
  if ((st = scratch.upload(d_tasks, tasks, n_tasks)) != BBML_OK) return st;
  int cap = 32;  // sort capacity: power of two >= the longest test set (<= kMetricsMaxN)
  while (cap < std::min(max_n, kMetricsMaxN)) cap <<= 1;
  const size_t smem = (size_t)cap * (4 * sizeof(double) + sizeof(int));
  cudaError_t e = cudaFuncSetAttribute(metrics_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return cuda_status(e, "metrics smem");
  metrics_kernel<<<n_tasks, MET_NT, smem, stream>>>(d_tasks, pred, actual_norm, actual_raw, norm,
                                                     out, cap);
  e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_status(e, "metrics launch");
  return scratch.release();
}

}  // namespace bbml

extern "C" bbml_status bbml_metrics(const bbml_pred_task* tasks, int32_t n_tasks,
                                    const double* pred, const double* actual_norm,
                                    const double* actual_raw, const double* norm, double* out,
                                    void* stream) {
  using namespace bbml;
  if (n_tasks == 0) return BBML_OK;
  if (!tasks || !pred || !actual_norm || !actual_raw || !norm || !out || n_tasks < 0) {
    set_error("bbml_metrics: NULL argument or n_tasks < 0");
    return BBML_ERR_INVALID;
  }
  return metrics_launch(tasks, n_tasks, pred, actual_norm, actual_raw, norm, out,
                        (cudaStream_t)stream);
}
