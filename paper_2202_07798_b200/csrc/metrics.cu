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
// kMetricsMaxN test rows take the segment path below (counting ranks in
// global memory); out[3] = 1.0 once Pearson / Spearman are written.
#include <algorithm>
#include <vector>

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
  if (n >= 2 && fits) {
    for (int i = threadIdx.x; i < n; i += MET_NT)
      pr[i] = __dadd_rn(__dmul_rn(p[i], __dsub_rn(yhi, ylo)), ylo);
    __syncthreads();
    pear = met_pearson(pr, ar, n, red);
    met_ranks(pr, n, np, key, idx, ra);
    met_ranks(ar, n, np, key, idx, rb);
    spear = met_pearson(ra, rb, n, red);
  }
  if (threadIdx.x == 0) {
    o[0] = mse;
    o[1] = pear;
    o[2] = spear;
    o[3] = (fits || n < 2) ? 1.0 : 0.0;
  }
}

// ---------------------------------------------------------------------------
// Segment path (any n): test sets longer than kMetricsMaxN and the pooled
// per-(app, kind) vectors of experiment.summarize (experiment.py:180-206).
// Values are gathered de-normalised into contiguous scratch (a = predicted
// counts, b = raw counts), ranked by COUNTING -- rank(x_i) = 0.5 (2 #{x_j <
// x_i} + #{x_j == x_i} - 1) + 1, the reference's tie-averaged stable-sort
// rank, exact in integers, O(n^2) compares streamed through shared-memory
// tiles (~24k^2 for the largest pooled app) -- then one CTA per segment
// forms Pearson of (a, b) and of the ranks.
// ---------------------------------------------------------------------------
struct MetSeg {
  int64_t off;   // first element in a / b / ranks
  int64_t n;
  int64_t out;   // out[out] = pearson, out[out + 1] = spearman
  int64_t flag;  // >= 0: out[flag] = 1.0 when done
};

constexpr int RANK_TILE = 2048;

// one CTA per task: de-normalised predictions and raw counts into a / b at dst[task]
__global__ void __launch_bounds__(MET_NT)
    met_gather_kernel(const bbml_pred_task* __restrict__ tasks, const int64_t* __restrict__ dst,
                      const double* __restrict__ pred, const double* __restrict__ actual_raw,
                      const double* __restrict__ norm, double* __restrict__ a, double* __restrict__ b) {
  const bbml_pred_task tk = tasks[blockIdx.x];
  const double ylo = norm[tk.norm_offset + 2 * tk.d], yhi = norm[tk.norm_offset + 2 * tk.d + 1];
  const int64_t o = dst[blockIdx.x];
  for (int i = threadIdx.x; i < tk.n; i += MET_NT) {
    a[o + i] = __dadd_rn(__dmul_rn(pred[tk.w_offset + i], __dsub_rn(yhi, ylo)), ylo);
    b[o + i] = actual_raw[tk.row_begin + i];
  }
}

// grid (chunks of MET_NT elements, segments): ranks of a and b within the segment
__global__ void __launch_bounds__(MET_NT)
    met_rank_kernel(const MetSeg* __restrict__ segs, const double* __restrict__ a,
                    const double* __restrict__ b, double* __restrict__ ra, double* __restrict__ rb) {
  __shared__ double ta[RANK_TILE], tb[RANK_TILE];
  const MetSeg sg = segs[blockIdx.y];
  const int64_t i = (int64_t)blockIdx.x * MET_NT + threadIdx.x;
  if ((int64_t)blockIdx.x * MET_NT >= sg.n) return;  // whole CTA past the segment
  const bool live = i < sg.n;
  const double xa = live ? a[sg.off + i] : 0.0, xb = live ? b[sg.off + i] : 0.0;
  long long lta = 0, eqa = 0, ltb = 0, eqb = 0;
  for (int64_t t0 = 0; t0 < sg.n; t0 += RANK_TILE) {
    const int m = (int)(sg.n - t0 < RANK_TILE ? sg.n - t0 : RANK_TILE);
    __syncthreads();
    for (int k = threadIdx.x; k < m; k += MET_NT) {
      ta[k] = a[sg.off + t0 + k];
      tb[k] = b[sg.off + t0 + k];
    }
    __syncthreads();
    for (int k = 0; k < m; ++k) {
      const double va = ta[k], vb = tb[k];
      lta += va < xa;
      eqa += va == xa;
      ltb += vb < xb;
      eqb += vb == xb;
    }
  }
  if (live) {
    ra[sg.off + i] = 0.5 * (double)(2 * lta + eqa - 1) + 1.0;
    rb[sg.off + i] = 0.5 * (double)(2 * ltb + eqb - 1) + 1.0;
  }
}

__global__ void __launch_bounds__(MET_NT)
    met_corr_kernel(const MetSeg* __restrict__ segs, const double* __restrict__ a,
                    const double* __restrict__ b, const double* __restrict__ ra,
                    const double* __restrict__ rb, double* __restrict__ out) {
  __shared__ double red[MET_NT / 32];
  const MetSeg sg = segs[blockIdx.x];
  const double nan = __longlong_as_double(0x7ff8000000000000LL);
  double pear = nan, spear = nan;
  if (sg.n >= 2) {
    pear = met_pearson(a + sg.off, b + sg.off, (int)sg.n, red);
    spear = met_pearson(ra + sg.off, rb + sg.off, (int)sg.n, red);
  }
  if (threadIdx.x == 0) {
    out[sg.out] = pear;
    out[sg.out + 1] = spear;
    if (sg.flag >= 0) out[sg.flag] = 1.0;
  }
}

// gather + rank + correlate the segments made of `tasks` (task i belongs to
// segment seg_of[i]; tasks of a segment are concatenated in task order)
static bbml_status segment_metrics(const bbml_pred_task* tasks, int32_t n_tasks, const int32_t* seg_of,
                                   int32_t n_seg, const int64_t* seg_out, const int64_t* seg_flag,
                                   const double* pred, const double* actual_raw, const double* norm,
                                   double* out, ScratchBuffer& scratch, cudaStream_t stream) {
  std::vector<int64_t> seg_n(n_seg, 0);
  for (int i = 0; i < n_tasks; ++i) seg_n[seg_of[i]] += tasks[i].n;
  std::vector<MetSeg> segs(n_seg);
  int64_t total = 0, max_n = 0;
  for (int s = 0; s < n_seg; ++s) {
    segs[s] = MetSeg{total, seg_n[s], seg_out[s], seg_flag ? seg_flag[s] : -1};
    total += seg_n[s];
    max_n = std::max(max_n, seg_n[s]);
  }
  std::vector<int64_t> dst(n_tasks);
  std::vector<int64_t> fill(n_seg, 0);
  for (int i = 0; i < n_tasks; ++i) {
    dst[i] = segs[seg_of[i]].off + fill[seg_of[i]];
    fill[seg_of[i]] += tasks[i].n;
  }
  bbml_pred_task* d_tasks = nullptr;
  int64_t* d_dst = nullptr;
  MetSeg* d_segs = nullptr;
  double *a = nullptr, *b = nullptr, *ra = nullptr, *rb = nullptr;
  bbml_status st;
  if ((st = scratch.alloc(&d_tasks, n_tasks)) != BBML_OK) return st;
  if ((st = scratch.alloc(&d_dst, n_tasks)) != BBML_OK) return st;
  if ((st = scratch.alloc(&d_segs, n_seg)) != BBML_OK) return st;
  for (double** p : {&a, &b, &ra, &rb})
    if ((st = scratch.alloc(p, std::max<int64_t>(total, 1))) != BBML_OK) return st;
  if ((st = scratch.upload(d_tasks, tasks, n_tasks)) != BBML_OK) return st;
  if ((st = scratch.upload(d_dst, dst.data(), n_tasks)) != BBML_OK) return st;
  if ((st = scratch.upload(d_segs, segs.data(), n_seg)) != BBML_OK) return st;
  met_gather_kernel<<<n_tasks, MET_NT, 0, stream>>>(d_tasks, d_dst, pred, actual_raw, norm, a, b);
  if (max_n > 0)
    for (int s0 = 0; s0 < n_seg; s0 += 65535) {  // grid.y limit
      dim3 grid((unsigned)ceil_div(max_n, MET_NT), (unsigned)std::min(65535, n_seg - s0));
      met_rank_kernel<<<grid, MET_NT, 0, stream>>>(d_segs + s0, a, b, ra, rb);
    }
  met_corr_kernel<<<n_seg, MET_NT, 0, stream>>>(d_segs, a, b, ra, rb, out);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? BBML_OK : cuda_status(e, "segment metrics launch");
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
  // test sets beyond the shared-memory sort: counting ranks in global memory
  std::vector<bbml_pred_task> big;
  std::vector<int64_t> big_out, big_flag;
  for (int i = 0; i < n_tasks; ++i)
    if (tasks[i].n > kMetricsMaxN) {
      big.push_back(tasks[i]);
      big_out.push_back(tasks[i].out_offset + 1);
      big_flag.push_back(tasks[i].out_offset + 3);
    }
  if (!big.empty()) {
    std::vector<int32_t> seg_of(big.size());
    for (size_t i = 0; i < big.size(); ++i) seg_of[i] = (int32_t)i;
    if ((st = segment_metrics(big.data(), (int32_t)big.size(), seg_of.data(), (int32_t)big.size(),
                              big_out.data(), big_flag.data(), pred, actual_raw, norm, out, scratch,
                              stream)) != BBML_OK)
      return st;
  }
  return scratch.release();
}

// pooled Pearson / Spearman over groups of models (experiment.summarize)
bbml_status pooled_metrics_launch(const bbml_pred_task* tasks, int32_t n_tasks, const int32_t* seg_of,
                                  int32_t n_seg, const double* pred, const double* actual_raw,
                                  const double* norm, double* out, cudaStream_t stream) {
  for (int i = 0; i < n_tasks; ++i) {
    const bbml_pred_task& t = tasks[i];
    if (t.n < 0 || t.d < 1 || t.d > BBML_MAX_INPUTS || t.row_begin < 0 || t.w_offset < 0 ||
        t.norm_offset < 0 || seg_of[i] < 0 || seg_of[i] >= n_seg) {
      set_error("pooled metrics task %d: invalid field", i);
      return BBML_ERR_INVALID;
    }
  }
  if (n_seg == 0) return BBML_OK;
  ScratchBuffer scratch(stream);
  std::vector<int64_t> seg_out(n_seg);
  for (int s = 0; s < n_seg; ++s) seg_out[s] = 2 * (int64_t)s;
  bbml_status st = segment_metrics(tasks, n_tasks, seg_of, n_seg, seg_out.data(), nullptr, pred,
                                   actual_raw, norm, out, scratch, stream);
  if (st != BBML_OK) return st;
  return scratch.release();
}

// ---------------------------------------------------------------------------
// Per-model heatmaps (metrics.heatmap_data, metrics.py:145-156, written per
// model by experiment.py:417-424): square bins over [0, max(pred, actual)]
// (1.0 when that max is <= 0), edges = numpy.linspace(0, hi, bins + 1)
// (i * (hi / bins), last edge exactly hi), counts of histogram2d: bin =
// searchsorted(edges, v, 'right') - 1, a value equal to the last edge goes to
// the last bin, values outside [0, hi] are dropped.  One CTA per model,
// shared-memory counters.
// ---------------------------------------------------------------------------
__device__ __forceinline__ int hm_bin(const double* edges, int bins, double v) {
  int lo = 0, hi = bins + 1;  // searchsorted 'right': first index with edges[idx] > v
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (edges[mid] <= v) lo = mid + 1;
    else hi = mid;
  }
  int idx = lo;
  if (v == edges[bins]) idx -= 1;
  return (idx >= 1 && idx <= bins) ? idx - 1 : -1;
}

__global__ void __launch_bounds__(MET_NT)
    heatmap_kernel(const bbml_pred_task* __restrict__ tasks, const double* __restrict__ pred,
                   const double* __restrict__ actual_raw, const double* __restrict__ norm, int bins,
                   double* __restrict__ edges_out, int32_t* __restrict__ counts_out) {
  extern __shared__ __align__(16) unsigned char hm_smem[];
  __shared__ double red[MET_NT / 32];
  double* edges = (double*)hm_smem;
  int* cnt = (int*)(edges + bins + 1);
  const bbml_pred_task tk = tasks[blockIdx.x];
  const double ylo = norm[tk.norm_offset + 2 * tk.d], yhi = norm[tk.norm_offset + 2 * tk.d + 1];
  double m = -__longlong_as_double(0x7ff0000000000000LL);
  for (int i = threadIdx.x; i < tk.n; i += MET_NT) {
    const double pv = __dadd_rn(__dmul_rn(pred[tk.w_offset + i], __dsub_rn(yhi, ylo)), ylo);
    m = fmax(m, fmax(pv, actual_raw[tk.row_begin + i]));
  }
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  for (int k = threadIdx.x; k < bins * bins; k += MET_NT) cnt[k] = 0;
  __syncthreads();
  double hi = red[0];
  for (int w = 1; w < MET_NT / 32; ++w) hi = fmax(hi, red[w]);
  if (!(hi > 0.0)) hi = 1.0;
  const double step = hi / bins;
  for (int k = threadIdx.x; k <= bins; k += MET_NT) edges[k] = k == bins ? hi : (double)k * step;
  __syncthreads();
  for (int i = threadIdx.x; i < tk.n; i += MET_NT) {
    const double pv = __dadd_rn(__dmul_rn(pred[tk.w_offset + i], __dsub_rn(yhi, ylo)), ylo);
    const int bp = hm_bin(edges, bins, pv), ba = hm_bin(edges, bins, actual_raw[tk.row_begin + i]);
    if (bp >= 0 && ba >= 0) atomicAdd(&cnt[bp * bins + ba], 1);
  }
  __syncthreads();
  double* eo = edges_out + (int64_t)blockIdx.x * (bins + 1);
  int32_t* co = counts_out + (int64_t)blockIdx.x * bins * bins;
  for (int k = threadIdx.x; k <= bins; k += MET_NT) eo[k] = edges[k];
  for (int k = threadIdx.x; k < bins * bins; k += MET_NT) co[k] = cnt[k];
}

bbml_status heatmap_launch(const bbml_pred_task* tasks, int32_t n_tasks, const double* pred,
                           const double* actual_raw, const double* norm, int32_t bins,
                           double* edges, int32_t* counts, cudaStream_t stream) {
  if (bins < 2 || bins > 200) {  // bins^2 int counters in shared memory
    set_error("bbml_heatmaps: bins=%d outside [2, 200]", bins);
    return BBML_ERR_INVALID;
  }
  for (int i = 0; i < n_tasks; ++i) {
    const bbml_pred_task& t = tasks[i];
    if (t.n < 1 || t.d < 1 || t.d > BBML_MAX_INPUTS || t.row_begin < 0 || t.w_offset < 0 ||
        t.norm_offset < 0) {
      set_error("heatmap task %d: invalid field (n >= 1 required)", i);
      return BBML_ERR_INVALID;
    }
  }
  if (n_tasks == 0) return BBML_OK;
  ScratchBuffer scratch(stream);
  bbml_pred_task* d_tasks = nullptr;
  bbml_status st;
  if ((st = scratch.alloc(&d_tasks, n_tasks)) != BBML_OK) return st;
  if ((st = scratch.upload(d_tasks, tasks, n_tasks)) != BBML_OK) return st;
  const size_t smem = (size_t)(bins + 1) * sizeof(double) + (size_t)bins * bins * sizeof(int);
  cudaError_t e = cudaFuncSetAttribute(heatmap_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return cuda_status(e, "heatmap smem");
  heatmap_kernel<<<n_tasks, MET_NT, smem, stream>>>(d_tasks, pred, actual_raw, norm, bins, edges,
                                                    counts);
  e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_status(e, "heatmap launch");
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

namespace bbml {

// ---------------------------------------------------------------------------
// Per-series count KDE (metrics.kde, metrics.py:95-118, one curve per series
// in run_experiment): Scott bandwidth n^(-1/5) * std(ddof = 1), grid =
// linspace(min - 3 bw, max + 3 bw, G), density = sum exp(-z^2 / 2) /
// (n bw sqrt(2 pi)).  One CTA per series: block reductions for mean / spread /
// range, then one grid point per thread over the series' counts staged in
// shared memory.  bw = 0 (no spread, n < 2) marks "no curve" (the reference
// raises BandwidthError and skips the file).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(MET_NT)
    kde_kernel(const int64_t* __restrict__ off, const double* __restrict__ vals, int G, int cap,
               double* __restrict__ grid_out, double* __restrict__ dens_out, double* __restrict__ bw_out) {
  extern __shared__ __align__(16) double kx[];
  __shared__ double red[MET_NT / 32];
  const int64_t a = off[blockIdx.x], n = off[blockIdx.x + 1] - a;
  double* go = grid_out + (int64_t)blockIdx.x * G;
  double* dout = dens_out + (int64_t)blockIdx.x * G;
  double sum = 0.0, lo = __longlong_as_double(0x7ff0000000000000LL), hi = -lo;
  for (int64_t i = threadIdx.x; i < n; i += MET_NT) {
    const double v = vals[a + i];
    if (i < cap) kx[i] = v;
    sum += v;
    lo = fmin(lo, v);
    hi = fmax(hi, v);
  }
  const double mean = met_sum(sum, red) / (double)n;
  double ss = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += MET_NT) {
    const double dv = vals[a + i] - mean;
    ss = fma(dv, dv, ss);
  }
  const double var = n > 1 ? met_sum(ss, red) / (double)(n - 1) : 0.0;
  // block min / max
  for (int o = 16; o >= 1; o >>= 1) {
    lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
  }
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = lo;
  __syncthreads();
  double blo = red[0];
  for (int w = 1; w < MET_NT / 32; ++w) blo = fmin(blo, red[w]);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = hi;
  __syncthreads();
  double bhi = red[0];
  for (int w = 1; w < MET_NT / 32; ++w) bhi = fmax(bhi, red[w]);
  const double spread = sqrt(var);
  if (!(spread > 0.0)) {
    if (threadIdx.x == 0) bw_out[blockIdx.x] = 0.0;
    return;
  }
  // numpy's rounding order (no contraction): linspace = g * step + start,
  // z = (x - v) / bw, exp(-0.5 * z**2)
  const double bw = __dmul_rn(pow((double)n, -1.0 / 5.0), spread);
  const double g0 = __dsub_rn(blo, __dmul_rn(3.0, bw)), g1 = __dadd_rn(bhi, __dmul_rn(3.0, bw));
  const double step = __ddiv_rn(__dsub_rn(g1, g0), (double)(G - 1));
  const double norm = __dmul_rn(__dmul_rn((double)n, bw), 2.5066282746310002);  // sqrt(2 pi)
  for (int g = threadIdx.x; g < G; g += MET_NT) {
    const double x = g == G - 1 ? g1 : __dadd_rn(__dmul_rn((double)g, step), g0);
    double acc = 0.0;
    for (int64_t i = 0; i < n; ++i) {
      const double z = __ddiv_rn(__dsub_rn(x, i < cap ? kx[i] : vals[a + i]), bw);
      acc += exp(__dmul_rn(-0.5, __dmul_rn(z, z)));
    }
    go[g] = x;
    dout[g] = __ddiv_rn(acc, norm);
  }
  if (threadIdx.x == 0) bw_out[blockIdx.x] = bw;
}

bbml_status kde_launch(const int64_t* off, int32_t n_series, const double* vals, int32_t G,
                       double* grid, double* dens, double* bw, cudaStream_t stream) {
  if (G < 2) {
    set_error("bbml_kde: grid_points=%d < 2", G);
    return BBML_ERR_INVALID;
  }
  if (n_series == 0) return BBML_OK;
  int64_t max_n = 0;
  for (int i = 0; i < n_series; ++i) {
    if (off[i + 1] < off[i]) {
      set_error("bbml_kde: offsets not monotone at %d", i);
      return BBML_ERR_INVALID;
    }
    max_n = std::max<int64_t>(max_n, off[i + 1] - off[i]);
  }
  ScratchBuffer scratch(stream);
  int64_t* d_off = nullptr;
  bbml_status st;
  if ((st = scratch.alloc(&d_off, n_series + 1)) != BBML_OK) return st;
  if ((st = scratch.upload(d_off, off, n_series + 1)) != BBML_OK) return st;
  const int cap = (int)std::min<int64_t>(max_n, 12288);  // counts staged in shared memory (96 KB)
  const size_t smem = (size_t)std::max(cap, 1) * sizeof(double);
  cudaError_t e = cudaFuncSetAttribute(kde_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return cuda_status(e, "kde smem");
  kde_kernel<<<n_series, MET_NT, smem, stream>>>(d_off, vals, G, cap, grid, dens, bw);
  e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_status(e, "kde launch");
  return scratch.release();
}

}  // namespace bbml

extern "C" bbml_status bbml_kde(const int64_t* offsets, int32_t n_series, const double* values,
                                int32_t grid_points, double* grid, double* density, double* bandwidth,
                                void* stream) {
  using namespace bbml;
  if (n_series == 0) return BBML_OK;
  if (!offsets || !values || !grid || !density || !bandwidth || n_series < 0) {
    set_error("bbml_kde: NULL argument or n_series < 0");
    return BBML_ERR_INVALID;
  }
  return kde_launch(offsets, n_series, values, grid_points, grid, density, bandwidth,
                    (cudaStream_t)stream);
}

extern "C" bbml_status bbml_pooled_metrics(const bbml_pred_task* tasks, int32_t n_tasks,
                                           const int32_t* seg_of, int32_t n_seg, const double* pred,
                                           const double* actual_raw, const double* norm,
                                           double* out, void* stream) {
  using namespace bbml;
  if (n_seg == 0) return BBML_OK;
  if (!tasks || !seg_of || !pred || !actual_raw || !norm || !out || n_tasks < 0 || n_seg < 0) {
    set_error("bbml_pooled_metrics: NULL argument or negative count");
    return BBML_ERR_INVALID;
  }
  return pooled_metrics_launch(tasks, n_tasks, seg_of, n_seg, pred, actual_raw, norm, out,
                               (cudaStream_t)stream);
}

extern "C" bbml_status bbml_heatmaps(const bbml_pred_task* tasks, int32_t n_tasks, const double* pred,
                                     const double* actual_raw, const double* norm, int32_t bins,
                                     double* edges, int32_t* counts, void* stream) {
  using namespace bbml;
  if (n_tasks == 0) return BBML_OK;
  if (!tasks || !pred || !actual_raw || !norm || !edges || !counts || n_tasks < 0) {
    set_error("bbml_heatmaps: NULL argument or n_tasks < 0");
    return BBML_ERR_INVALID;
  }
  return heatmap_launch(tasks, n_tasks, pred, actual_raw, norm, bins, edges, counts,
                        (cudaStream_t)stream);
}
