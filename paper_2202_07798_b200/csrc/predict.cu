// predict.cu — batched inference / extrapolation and unit-level kernels.
//
// bbml_predict mirrors persist.SavedModel.predict_counts (persist.py:40-43):
//   Xn = (x - x_min) / span  (span <= 0 -> feature forced to 0, no clamping;
//        traces.py:293-302)
//   y  = pnn.forward (pnn.py:108-118) | brbpnn.forward (brbpnn.py:85-91)
//   out = y * (y_max - y_min) + y_min   (traces.py:311-313)
// and, with norm_offset = -1, predict_normalized (persist.py:35-38).
#include <algorithm>
#include <vector>

#include "common.cuh"
#include "launch.h"

namespace bbml {

constexpr int PRED_NT = 128;
constexpr int PRED_MAXP = BBML_LM_MAX_PARAMS + BBML_PNN_MAX_HIDDEN * (BBML_MAX_INPUTS + 2) + 1;

__device__ __forceinline__ double pnn_forward_row(const double* w, const double* x, int d, int h,
                                                  double eps) {
  const int hd = h * d;
  double z = 0.0;
  for (int j = 0; j < h; ++j) {
    double pre = 0.0;
    for (int k = 0; k < d; ++k) pre = fma(x[k], w[j * d + k], pre);
    pre = __dadd_rn(pre, w[hd + j]);
    z = fma(tanh(pre), w[hd + h + j], z);
  }
  z = __dadd_rn(z, w[hd + 2 * h]);
  return __dadd_rn(softplus(z), eps);
}

__device__ __forceinline__ double br_forward_row(const double* w, const double* x, int d, int h) {
  const int hd = h * d;
  double out = 0.0;
  for (int j = 0; j < h; ++j) {
    double pre = 0.0;
    for (int k = 0; k < d; ++k) pre = fma(x[k], w[j * d + k], pre);
    pre = __dadd_rn(pre, w[hd + j]);
    out = fma(tansig(pre), w[hd + h + j], out);
  }
  return __dadd_rn(out, w[hd + 2 * h]);
}

__global__ void __launch_bounds__(PRED_NT)
    predict_kernel(const bbml_pred_task* __restrict__ tasks, const double* __restrict__ Xq,
                   int xs, const double* __restrict__ weights, const double* __restrict__ norm,
                   double* __restrict__ out) {
  const bbml_pred_task tk = tasks[blockIdx.x];
  const int d = tk.d, h = tk.h;
  const int P = h * (d + 2) + 1;
  extern __shared__ double sw[];
  double* nrm = sw + P;  // x_min[d], x_max[d], y_min, y_max
  for (int i = threadIdx.x; i < P; i += blockDim.x) sw[i] = weights[tk.w_offset + i];
  const bool use_norm = tk.norm_offset >= 0;
  if (use_norm)
    for (int i = threadIdx.x; i < 2 * d + 2; i += blockDim.x) nrm[i] = norm[tk.norm_offset + i];
  __syncthreads();
  double x[BBML_MAX_INPUTS];
  const int64_t step = (int64_t)gridDim.y * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.y * blockDim.x + threadIdx.x; i < tk.n; i += step) {
    const double* xr = Xq + (tk.row_begin + i) * xs;
    for (int k = 0; k < d; ++k) {
      double v = __ldg(xr + k);
      if (use_norm) {
        const double lo = nrm[k], span = __dsub_rn(nrm[d + k], lo);
        v = span > 0.0 ? __ddiv_rn(__dsub_rn(v, lo), span) : 0.0;
      }
      x[k] = v;
    }
    double y = tk.kind == 0 ? pnn_forward_row(sw, x, d, h, tk.eps) : br_forward_row(sw, x, d, h);
    if (use_norm) {
      const double ylo = nrm[2 * d], yhi = nrm[2 * d + 1];
      y = __dadd_rn(__dmul_rn(y, __dsub_rn(yhi, ylo)), ylo);
    }
    out[tk.out_offset + i] = y;
  }
}

bbml_status predict_launch(const bbml_pred_task* tasks, int32_t n_tasks, const double* Xq,
                           int32_t x_stride, const double* weights, const double* norm,
                           double* out, cudaStream_t stream) {
  int64_t max_n = 0;
  int max_p = 0;
  for (int i = 0; i < n_tasks; ++i) {
    const bbml_pred_task& t = tasks[i];
    if (t.n < 0 || t.d < 1 || t.h < 1 || t.d > BBML_MAX_INPUTS || (t.kind != 0 && t.kind != 1) ||
        t.row_begin < 0 || t.w_offset < 0 || t.out_offset < 0) {
      set_error("predict task %d: invalid field", i);
      return BBML_ERR_INVALID;
    }
    if (t.d > x_stride) {  // the query rows must carry every input the model reads
      set_error("predict task %d: d=%d exceeds the query row stride %d", i, t.d, x_stride);
      return BBML_ERR_INVALID;
    }
    if (t.norm_offset >= 0 && norm == nullptr) {
      set_error("predict task %d: normalizer requested but norm == NULL", i);
      return BBML_ERR_INVALID;
    }
    const int P = t.h * (t.d + 2) + 1;
    if (P > PRED_MAXP) {
      set_error("predict task %d: %d parameters exceed %d", i, P, PRED_MAXP);
      return BBML_ERR_UNSUPPORTED;
    }
    max_n = std::max<int64_t>(max_n, t.n);
    max_p = std::max(max_p, P);
  }
  if (n_tasks == 0 || max_n == 0) return BBML_OK;
  ScratchBuffer scratch(stream);
  bbml_pred_task* d_tasks = nullptr;
  bbml_status st;
  if ((st = scratch.alloc(&d_tasks, n_tasks)) != BBML_OK) return st;
  if ((st = scratch.upload(d_tasks, tasks, n_tasks)) != BBML_OK) return st;
  const int ychunks = (int)std::min<int64_t>(ceil_div(max_n, PRED_NT), 65535);
  const size_t smem = (size_t)(max_p + 2 * BBML_MAX_INPUTS + 2) * sizeof(double);
  dim3 grid(n_tasks, ychunks);
  predict_kernel<<<grid, PRED_NT, smem, stream>>>(d_tasks, Xq, x_stride, weights, norm, out);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_status(e, "predict launch");
  return scratch.release();
}

}  // namespace bbml
