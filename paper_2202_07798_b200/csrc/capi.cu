// capi.cu — extern "C" entry points of libbbml.so (see include/bbml.h).
#include <stdarg.h>
#include <stdio.h>
#include <string.h>

#include <mutex>

#include "../../include/bbml.h"
#include "common.cuh"
#include "launch.h"
#include "pcg64.cuh"

namespace bbml {

static thread_local char g_err[512] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

bbml_status cuda_status(cudaError_t e, const char* what) {
  set_error("%s: %s (%s)", what, cudaGetErrorName(e), cudaGetErrorString(e));
  return BBML_ERR_CUDA;
}

cudaMemPool_t scratch_pool() {
  static std::mutex mu;
  static std::vector<cudaMemPool_t> pools;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lock(mu);
  if ((int)pools.size() <= dev) pools.resize(dev + 1, nullptr);
  if (!pools[dev]) {
    cudaMemPoolProps props{};
    props.allocType = cudaMemAllocationTypePinned;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = dev;
    cudaMemPool_t p = nullptr;
    if (cudaMemPoolCreate(&p, &props) != cudaSuccess) {
      cudaGetLastError();
      cudaDeviceGetDefaultMemPool(&p, dev);  // still stream-ordered; trims at syncs
    } else {
      uint64_t keep = ~0ull;
      cudaMemPoolSetAttribute(p, cudaMemPoolAttrReleaseThreshold, &keep);
    }
    pools[dev] = p;
  }
  return pools[dev];
}

namespace {
struct ForkPool {
  std::vector<cudaStream_t> streams;
  std::vector<cudaEvent_t> events;
  cudaEvent_t fork = nullptr;
  unsigned cursor = 0;
};
// Child streams are handed out round-robin from kForkStreams, so two calls in
// flight at once (bbml_lm_train on one stream and bbml_pnn_train on another,
// as batch.DeviceWorkload.step issues them) get disjoint children instead of
// queueing a PNN bucket behind an LM bucket on a shared child stream.
constexpr int kForkStreams = 16;
thread_local std::vector<ForkPool> g_pools;  // per device, per host thread
}  // namespace

StreamFork::StreamFork(cudaStream_t parent, int n) : parent_(parent), n_(n) {
  if (n_ <= 1) return;
  int dev = 0;
  cudaGetDevice(&dev);
  if ((int)g_pools.size() <= dev) g_pools.resize(dev + 1);
  ForkPool& p = g_pools[dev];
  if (!p.fork) cudaEventCreateWithFlags(&p.fork, cudaEventDisableTiming);
  while ((int)p.events.size() < n_) {
    cudaEvent_t e;
    cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
    p.events.push_back(e);
  }
  cudaEventRecord(p.fork, parent_);
  for (int i = 0; i < n_; ++i) {
    const int k = (int)(p.cursor++ % kForkStreams);
    if ((int)p.streams.size() <= k) {
      cudaStream_t s;
      cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
      p.streams.push_back(s);
    }
    cudaStreamWaitEvent(p.streams[k], p.fork, 0);
    kids_.push_back(p.streams[k]);
    done_.push_back(p.events[i]);
  }
}

bbml_status StreamFork::join() {
  if (n_ <= 1) return BBML_OK;
  for (int i = 0; i < n_; ++i) {
    cudaEventRecord(done_[i], kids_[i]);
    cudaStreamWaitEvent(parent_, done_[i], 0);
  }
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? BBML_OK : cuda_status(e, "stream fork/join");
}

bbml_status pnn_loss_grad_launch(const bbml_pred_task*, int32_t, const double*, const double*,
                                 int32_t, const double*, double, double*, double*, cudaStream_t);
bbml_status lm_jacobian_launch(const bbml_pred_task*, int32_t, const double*, const double*,
                               int32_t, const double*, const int64_t*, double*, double*, double*,
                               cudaStream_t);
bbml_status adam_launch(double*, const double*, double*, double*, int64_t, const int64_t*, int,
                        double, double, double, double, double, double, int32_t*, cudaStream_t);
bbml_status tansig_launch(const double*, double*, int64_t, cudaStream_t);
bbml_status fma_peak_launch(int, int, int, void*, cudaStream_t);
bbml_status gram_launch(const int32_t*, const int32_t*, int32_t, const int64_t*, const int64_t*,
                        const int64_t*, const int64_t*, const double*, const double*, double*,
                        double*, cudaStream_t);
bbml_status lm_unit_launch(int, const int32_t*, int32_t, const int64_t*, const int64_t*,
                           const double*, const double*, const double*, const double*, int,
                           double*, double*, int32_t*, cudaStream_t);

}  // namespace bbml

using namespace bbml;

#define BBML_CHECK_PTR(p)                          \
  do {                                             \
    if (!(p)) {                                    \
      set_error("%s: NULL pointer '%s'", __func__, #p); \
      return BBML_ERR_INVALID;                     \
    }                                              \
  } while (0)

extern "C" {

int32_t bbml_abi_version(void) { return BBML_ABI_VERSION; }

int64_t bbml_struct_size(int32_t which) {
  switch (which) {
    case 0: return (int64_t)sizeof(bbml_seed);
    case 1: return (int64_t)sizeof(bbml_pnn_task);
    case 2: return (int64_t)sizeof(bbml_lm_task);
    case 3: return (int64_t)sizeof(bbml_pred_task);
    case 4: return (int64_t)sizeof(bbml_model_status);
    default: return -1;
  }
}

const char* bbml_version(void) { return "bbml-b200 0.1.0 (sm_100a)"; }

const char* bbml_last_error(void) { return g_err; }

bbml_status bbml_seedseq_generate(const uint32_t* words, int32_t n_words, uint32_t* out,
                                  int32_t n_out) {
  BBML_CHECK_PTR(words);
  BBML_CHECK_PTR(out);
  if (n_words < 1 || n_out < 0) {
    set_error("bbml_seedseq_generate: n_words=%d n_out=%d", n_words, n_out);
    return BBML_ERR_INVALID;
  }
  SeedSeq s;
  s.init(words, n_words);
  s.generate(out, n_out);
  return BBML_OK;
}

bbml_status bbml_pcg64_state(const bbml_seed* seed, uint64_t* out4) {
  BBML_CHECK_PTR(seed);
  BBML_CHECK_PTR(out4);
  if (seed->n_words < 1 || seed->n_words > BBML_MAX_ENTROPY_WORDS) {
    set_error("bbml_pcg64_state: n_words=%d", seed->n_words);
    return BBML_ERR_INVALID;
  }
  Pcg64 r;
  r.seed(*seed);
  out4[0] = (uint64_t)(r.state >> 64);
  out4[1] = (uint64_t)r.state;
  out4[2] = (uint64_t)(r.inc >> 64);
  out4[3] = (uint64_t)r.inc;
  return BBML_OK;
}

bbml_status bbml_pnn_train(const bbml_pnn_task* tasks, int32_t n_tasks, const double* X,
                           const double* y, int32_t x_stride, double* weights, double* history,
                           bbml_model_status* status, int32_t precision, void* stream) {
  if (n_tasks == 0) return BBML_OK;
  BBML_CHECK_PTR(tasks);
  BBML_CHECK_PTR(X);
  BBML_CHECK_PTR(y);
  BBML_CHECK_PTR(weights);
  BBML_CHECK_PTR(status);
  if (n_tasks < 0 || x_stride < 1 || (precision != 32 && precision != 64)) {
    set_error("bbml_pnn_train: n_tasks=%d x_stride=%d precision=%d", n_tasks, x_stride, precision);
    return BBML_ERR_INVALID;
  }
  for (int i = 0; i < n_tasks; ++i)
    if (tasks[i].d > x_stride) {
      set_error("bbml_pnn_train: task %d has d=%d > x_stride=%d", i, tasks[i].d, x_stride);
      return BBML_ERR_INVALID;
    }
  return pnn_train_launch(tasks, n_tasks, X, y, x_stride, weights, history, status, precision,
                          (cudaStream_t)stream);
}

bbml_status bbml_lm_train(const bbml_lm_task* tasks, int32_t n_tasks, const double* X,
                          const double* y, int32_t x_stride, double* weights, double* history,
                          bbml_model_status* status, void* stream) {
  if (n_tasks == 0) return BBML_OK;
  BBML_CHECK_PTR(tasks);
  BBML_CHECK_PTR(X);
  BBML_CHECK_PTR(y);
  BBML_CHECK_PTR(weights);
  BBML_CHECK_PTR(status);
  if (n_tasks < 0 || x_stride < 1) {
    set_error("bbml_lm_train: n_tasks=%d x_stride=%d", n_tasks, x_stride);
    return BBML_ERR_INVALID;
  }
  for (int i = 0; i < n_tasks; ++i)
    if (tasks[i].d > x_stride) {
      set_error("bbml_lm_train: task %d has d=%d > x_stride=%d", i, tasks[i].d, x_stride);
      return BBML_ERR_INVALID;
    }
  return lm_train_launch(tasks, n_tasks, X, y, x_stride, weights, history, status,
                         (cudaStream_t)stream);
}

bbml_status bbml_predict(const bbml_pred_task* tasks, int32_t n_tasks, const double* Xq,
                         int32_t x_stride, const double* weights, const double* norm, double* out,
                         void* stream) {
  if (n_tasks == 0) return BBML_OK;
  BBML_CHECK_PTR(tasks);
  BBML_CHECK_PTR(Xq);
  BBML_CHECK_PTR(weights);
  BBML_CHECK_PTR(out);
  if (n_tasks < 0 || x_stride < 1) {
    set_error("bbml_predict: n_tasks=%d x_stride=%d", n_tasks, x_stride);
    return BBML_ERR_INVALID;
  }
  return predict_launch(tasks, n_tasks, Xq, x_stride, weights, norm, out, (cudaStream_t)stream);
}

bbml_status bbml_pnn_loss_grad(const bbml_pred_task* tasks, int32_t n_tasks, const double* X,
                               const double* y, int32_t x_stride, const double* weights,
                               double nll_eps, double* loss, double* grads, void* stream) {
  if (n_tasks == 0) return BBML_OK;
  BBML_CHECK_PTR(tasks);
  BBML_CHECK_PTR(X);
  BBML_CHECK_PTR(y);
  BBML_CHECK_PTR(weights);
  BBML_CHECK_PTR(loss);
  BBML_CHECK_PTR(grads);
  return pnn_loss_grad_launch(tasks, n_tasks, X, y, x_stride, weights, nll_eps, loss, grads,
                              (cudaStream_t)stream);
}

bbml_status bbml_lm_jacobian(const bbml_pred_task* tasks, int32_t n_tasks, const double* X,
                             const double* y, int32_t x_stride, const double* weights,
                             const int64_t* jac_offset, double* jac, double* resid,
                             double* energies, void* stream) {
  if (n_tasks == 0) return BBML_OK;
  BBML_CHECK_PTR(tasks);
  BBML_CHECK_PTR(X);
  BBML_CHECK_PTR(y);
  BBML_CHECK_PTR(weights);
  BBML_CHECK_PTR(resid);
  if (jac != nullptr) BBML_CHECK_PTR(jac_offset);
  return lm_jacobian_launch(tasks, n_tasks, X, y, x_stride, weights, jac_offset, jac, resid,
                            energies, (cudaStream_t)stream);
}

bbml_status bbml_lm_gram(const int32_t* P, const int32_t* n, int32_t n_tasks,
                         const int64_t* j_offset, const int64_t* r_offset,
                         const int64_t* pp_offset, const int64_t* p_offset, const double* J,
                         const double* r, double* jtj, double* jtr, void* stream) {
  if (n_tasks == 0) return BBML_OK;
  BBML_CHECK_PTR(P);
  BBML_CHECK_PTR(n);
  BBML_CHECK_PTR(j_offset);
  BBML_CHECK_PTR(r_offset);
  BBML_CHECK_PTR(pp_offset);
  BBML_CHECK_PTR(p_offset);
  BBML_CHECK_PTR(J);
  BBML_CHECK_PTR(r);
  BBML_CHECK_PTR(jtj);
  BBML_CHECK_PTR(jtr);
  for (int i = 0; i < n_tasks; ++i)
    if (P[i] < 1 || n[i] < 0) {
      set_error("bbml_lm_gram: task %d P=%d n=%d", i, P[i], n[i]);
      return BBML_ERR_INVALID;
    }
  return gram_launch(P, n, n_tasks, j_offset, r_offset, pp_offset, p_offset, J, r, jtj, jtr,
                     (cudaStream_t)stream);
}

bbml_status bbml_adam_step(double* params, const double* grads, double* m, double* v,
                           int64_t n_params, const int64_t* block_begin, int32_t n_blocks,
                           double bc1, double bc2, double lr, double beta1, double beta2,
                           double eps, int32_t* bad_block, void* stream) {
  BBML_CHECK_PTR(params);
  BBML_CHECK_PTR(grads);
  BBML_CHECK_PTR(m);
  BBML_CHECK_PTR(v);
  BBML_CHECK_PTR(block_begin);
  BBML_CHECK_PTR(bad_block);
  if (n_params < 0 || n_blocks < 1) {
    set_error("bbml_adam_step: n_params=%lld n_blocks=%d", (long long)n_params, n_blocks);
    return BBML_ERR_INVALID;
  }
  return adam_launch(params, grads, m, v, n_params, block_begin, n_blocks, bc1, bc2, lr, beta1,
                     beta2, eps, bad_block, (cudaStream_t)stream);
}

bbml_status bbml_fma_peak(int32_t precision, int32_t blocks, int32_t iters, void* out,
                          void* stream) {
  BBML_CHECK_PTR(out);
  if ((precision != 32 && precision != 64) || blocks < 1 || iters < 1) {
    set_error("bbml_fma_peak: precision=%d blocks=%d iters=%d", precision, blocks, iters);
    return BBML_ERR_INVALID;
  }
  return fma_peak_launch(precision, blocks, iters, out, (cudaStream_t)stream);
}

bbml_status bbml_tansig(const double* x, double* y, int64_t n, void* stream) {
  if (n == 0) return BBML_OK;
  BBML_CHECK_PTR(x);
  BBML_CHECK_PTR(y);
  return tansig_launch(x, y, n, (cudaStream_t)stream);
}

bbml_status bbml_lm_solve(const int32_t* P, int32_t n_tasks, const int64_t* pp_offset,
                          const int64_t* p_offset, const double* jtj, const double* jtr,
                          const double* w, const double* abm, double* delta, int32_t* info,
                          void* stream) {
  if (n_tasks == 0) return BBML_OK;
  BBML_CHECK_PTR(P);
  BBML_CHECK_PTR(pp_offset);
  BBML_CHECK_PTR(p_offset);
  BBML_CHECK_PTR(jtj);
  BBML_CHECK_PTR(jtr);
  BBML_CHECK_PTR(w);
  BBML_CHECK_PTR(abm);
  BBML_CHECK_PTR(delta);
  BBML_CHECK_PTR(info);
  return lm_unit_launch(0, P, n_tasks, pp_offset, p_offset, jtj, jtr, w, abm, 3, delta, nullptr,
                        info, (cudaStream_t)stream);
}

bbml_status bbml_lm_evidence(const int32_t* P, int32_t n_tasks, const int64_t* pp_offset,
                             const int64_t* p_offset, const double* jtj, const double* in5,
                             double* eig, double* out5, void* stream) {
  if (n_tasks == 0) return BBML_OK;
  BBML_CHECK_PTR(P);
  BBML_CHECK_PTR(pp_offset);
  BBML_CHECK_PTR(p_offset);
  BBML_CHECK_PTR(jtj);
  BBML_CHECK_PTR(in5);
  BBML_CHECK_PTR(eig);
  BBML_CHECK_PTR(out5);
  return lm_unit_launch(1, P, n_tasks, pp_offset, p_offset, jtj, nullptr, nullptr, in5, 5, eig,
                        out5, nullptr, (cudaStream_t)stream);
}

}  // extern "C"
