// launch.h — launch descriptors shared by the kernels and the C-ABI layer.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <vector>

#include "../../include/bbml.h"
#include "common.cuh"

namespace bbml {

struct PnnLaunch {
  const bbml_pnn_task* tasks;  // device, sorted by (bucket, cost desc)
  const int32_t* orig_index;   // device, position of each sorted task in the caller's table
  const int64_t* perm_offset;  // device, per sorted task offset into perm_global
  int32_t n_tasks;
  int32_t x_stride;
  const double* X;
  const double* y;
  const float* Xf;  // FP32 kernels: rows converted once per launch (scratch)
  const float* yf;
  int32_t xf_stride;  // floats per Xf row: 4 when x_stride <= 4 (16-byte rows), else x_stride
  int32_t y_in_x;     // 1: Xf rows are {x0, x1, x2, y} (x_stride <= 3), one 16-byte load per sample
  double* weights;
  double* history;
  bbml_model_status* status;
  int32_t* perm_global;    // global double-buffer workspace (used when smem cannot hold it)
  int32_t perm_in_smem;    // 1: permutation double buffers live in shared memory
  int32_t perm_cap;        // elements per smem permutation buffer (max n of the launch)
  int32_t groups_per_cta;  // models per CTA (consumer groups; producer lane i serves group i)
  int32_t poll_cap_ns;     // producer poll back-off cap (ns)
  int32_t stage_off;       // FP64 kernel: byte offset of the row staging area in shared memory
  const double2* bc;       // FP64 kernel: Adam bias corrections {1 - 0.9^t, 1 - 0.999^t}, t = 1..bc_len
  int32_t bc_len;          //   (host libm pow, as the reference's Python float pow); 1.0 beyond
  const double* rows;      // FP64 kernel: row records [x_0..x_{rec_y-1}, y, pad] (TMA staging)
  int32_t rec;             //   doubles per record (even: 16-byte multiple)
  int32_t rec_y;           //   index of y in a record
};

struct LmLaunch {
  const bbml_lm_task* tasks;
  const int32_t* orig_index;
  int32_t n_tasks;
  int32_t x_stride;
  int32_t pmax;  // max P in this launch (smem sizing)
  const double* X;
  const double* y;
  double* weights;
  double* history;
  bbml_model_status* status;
  int* queue;  // persistent warp kernels: next-task counter (nullptr: static grid)
};

// The library's stream-ordered memory pool for the current device: the
// device's default pool trims freed blocks back to the driver at every
// host synchronisation (release threshold 0), which measured 0.1-0.9 s
// stalls in the caller's first synchronise after a step; this pool keeps
// them cached (release threshold = unlimited).
cudaMemPool_t scratch_pool();

// Stream-ordered scratch: cudaMallocFromPoolAsync on the call's stream,
// released with cudaFreeAsync on the same stream after the kernels are
// enqueued.
class ScratchBuffer {
 public:
  explicit ScratchBuffer(cudaStream_t s) : s_(s) {}
  ~ScratchBuffer() { release(); }
  template <typename T>
  bbml_status alloc(T** p, int64_t count) {
    void* q = nullptr;
    size_t bytes = (size_t)(count > 0 ? count : 1) * sizeof(T);
    cudaError_t e = cudaMallocFromPoolAsync(&q, bytes, scratch_pool(), s_);
    if (e != cudaSuccess) return cuda_status(e, "cudaMallocAsync(scratch)");
    ptrs_.push_back(q);
    *p = (T*)q;
    return BBML_OK;
  }
  template <typename T>
  bbml_status upload(T* dst, const T* src, int64_t count) {
    if (count <= 0) return BBML_OK;
    cudaError_t e = cudaMemcpyAsync(dst, src, (size_t)count * sizeof(T), cudaMemcpyHostToDevice, s_);
    return e == cudaSuccess ? BBML_OK : cuda_status(e, "cudaMemcpyAsync(scratch upload)");
  }
  bbml_status release() {
    bbml_status st = BBML_OK;
    for (void* p : ptrs_) {
      cudaError_t e = cudaFreeAsync(p, s_);
      if (e != cudaSuccess) st = cuda_status(e, "cudaFreeAsync(scratch)");
    }
    ptrs_.clear();
    return st;
  }

 private:
  cudaStream_t s_;
  std::vector<void*> ptrs_;
};

// Fork/join of the caller's stream so the independent per-shape launches of
// one call (e.g. hidden-1 and hidden-10 LM buckets) run concurrently instead
// of back to back.  Child streams/events come from a per-thread, per-device
// pool created on first use (non-blocking streams, timing-disabled events).
class StreamFork {
 public:
  StreamFork(cudaStream_t parent, int n);
  cudaStream_t child(int i) const { return n_ > 1 ? kids_[i] : parent_; }
  bbml_status join();

 private:
  cudaStream_t parent_;
  int n_;
  std::vector<cudaStream_t> kids_;
  std::vector<cudaEvent_t> done_;
};

bbml_status pnn_train_launch(const bbml_pnn_task* tasks, int32_t n_tasks, const double* X,
                             const double* y, int32_t x_stride, double* weights, double* history,
                             bbml_model_status* status, int32_t precision, cudaStream_t stream);
bbml_status lm_train_launch(const bbml_lm_task* tasks, int32_t n_tasks, const double* X,
                            const double* y, int32_t x_stride, double* weights, double* history,
                            bbml_model_status* status, cudaStream_t stream);
bbml_status predict_launch(const bbml_pred_task* tasks, int32_t n_tasks, const double* Xq,
                           int32_t x_stride, const double* weights, const double* norm,
                           double* out, cudaStream_t stream);

}  // namespace bbml
