/*
 * bbml.h — C-ABI of the B200-native BB-ML trainer / predictor (libbbml.so).
 *
 * The reference (bbcount, pure Python/NumPy) has no FFI; its drop-in
 * boundary is the Python API.  Each entry point below replaces one
 * reference routine, batched over many independent models:
 *
 *   bbml_pnn_train    <- bbcount/pnn.py:211-250      pnn.train (+ init_model 87-105,
 *                                                     loss_and_grads 121-147, adam_step 174-189)
 *   bbml_lm_train     <- bbcount/brbpnn.py:286-346   brbpnn.train (+ lm_trial/lm_step 174-211,
 *                                                     solve_damped 153-171, evidence_update 221-251)
 *   bbml_predict      <- bbcount/pnn.py:108-118      pnn.forward
 *   bbml_metrics      <- bbcount/metrics.py:33-76    mse / pearson / spearman
 *   bbml_pooled_metrics <- bbcount/experiment.py:180-206 pooled per-app correlations
 *   bbml_heatmaps     <- bbcount/metrics.py:145-156  heatmap_data (experiment.py:417-424)
 *   bbml_kde          <- bbcount/metrics.py:95-118   kde (experiment.py:425-430)
 *                        bbcount/brbpnn.py:85-91     brbpnn.forward
 *                        bbcount/persist.py:35-43    SavedModel.predict_normalized / predict_counts
 *   bbml_pnn_loss_grad<- bbcount/pnn.py:121-147      pnn.loss_and_grads (unit level)
 *   bbml_lm_jacobian  <- bbcount/brbpnn.py:109-130   objective + jacobian (unit level)
 *   bbml_lm_solve     <- bbcount/brbpnn.py:153-171   solve_damped (unit level)
 *   bbml_lm_evidence  <- bbcount/brbpnn.py:221-251   evidence_update (unit level)
 *   bbml_lm_gram      <- bbcount/brbpnn.py:166-167   J.T @ J, J.T @ r (unit level)
 *   bbml_adam_step    <- bbcount/pnn.py:174-189      adam_step (unit level)
 *   bbml_tansig       <- bbcount/brbpnn.py:33-38     tansig (unit level)
 *   bbml_seedseq_generate / bbml_pcg64_state
 *                     <- numpy SeedSequence / default_rng as called at
 *                        pnn.py:226, brbpnn.py:309, experiment.py:38-50
 *
 * Conventions
 *  - Task tables are HOST arrays (read during the call, not retained).
 *  - Every data pointer (X, y, weights, history, status, out) is DEVICE memory
 *    owned by the caller.  The library allocates only stream-ordered scratch
 *    that is released on the same stream before the call's work completes.
 *  - `stream` is a cudaStream_t (NULL = legacy default stream).  All work is
 *    enqueued on it; calls return without synchronising.  Re-entrant across
 *    streams; no global mutable state except the thread-local last error.
 *  - Parameters of one model are packed in the reference pack() order
 *    (brbpnn.py:94-99): W1 (h x d, row-major), b1 (h), W2 (h), b2.
 *  - Launch/config problems return a non-zero bbml_status; per-model
 *    numerical outcomes are reported in bbml_model_status.code.
 */
#ifndef BBML_H_
#define BBML_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BBML_ABI_VERSION 1
#define BBML_MAX_ENTROPY_WORDS 8
#define BBML_MAX_INPUTS 16
#define BBML_PNN_MAX_HIDDEN 64
#define BBML_LM_MAX_PARAMS 512

typedef enum {
  BBML_OK = 0,
  BBML_ERR_INVALID = 1,     /* bad argument / task field */
  BBML_ERR_CUDA = 2,        /* CUDA runtime error (see bbml_last_error) */
  BBML_ERR_UNSUPPORTED = 3  /* shape outside the supported envelope */
} bbml_status;

/* per-model outcome codes (bbml_model_status.code) */
enum {
  BBML_MODEL_OK = 0,
  BBML_MODEL_DIVERGED = 1,       /* pnn.TrainingError: non-finite batch loss (value = loss) */
  BBML_MODEL_NONFINITE_GRAD = 2, /* pnn.NumericError: detail = block 0..3 (W1,b1,W2,b2) */
  BBML_MODEL_SINGULAR = 3,       /* brbpnn.NumericError: damped system singular (value = mu) */
  BBML_MODEL_BAD_TASK = 4        /* task rejected by the device (shape) */
};

/* numpy.random.SeedSequence entropy for one model. */
typedef struct bbml_seed {
  uint32_t words[BBML_MAX_ENTROPY_WORDS]; /* little-endian 32-bit entropy words */
  int32_t n_words;                        /* 1..8 */
  int32_t mode; /* 0: default_rng(entropy)                        (pnn.train seed=...)
                   1: default_rng(SeedSequence(entropy).generate_state(1, u64)[0])
                      (experiment.series_seed -> train, experiment.py:38-50,117) */
} bbml_seed;

typedef struct bbml_pnn_task {
  int64_t row_begin;   /* first training row in X / y */
  int64_t w_offset;    /* doubles into weights */
  int64_t hist_offset; /* doubles into history (epochs entries) or -1 */
  int32_t n, d, h, epochs, batch, reserved;
  double lr, eps;
  bbml_seed seed;
} bbml_pnn_task;

typedef struct bbml_lm_task {
  int64_t row_begin;
  int64_t w_offset;
  int64_t hist_offset; /* doubles into history (max_epochs x 10 records) or -1 */
  int32_t n, d, h, max_epochs, estimate, reserved;
  double mu0, mu_inc, mu_dec, mu_max, alpha0, beta0;
  bbml_seed seed;
} bbml_lm_task;

typedef struct bbml_pred_task {
  int64_t row_begin;   /* first query row in Xq */
  int64_t w_offset;    /* doubles into weights */
  int64_t norm_offset; /* doubles into norm: x_min[d], x_max[d], y_min, y_max; -1 = none */
  int64_t out_offset;  /* doubles into out */
  int32_t n, d, h, kind; /* kind 0 = PNN (softplus rate), 1 = BR-BPNN (linear out) */
  double eps;
} bbml_pred_task;

typedef struct bbml_model_status {
  int32_t code;    /* BBML_MODEL_* */
  int32_t epochs;  /* epochs completed (BR: history length; PNN: failing epoch on error) */
  int32_t detail;  /* PNN: failing block; BR: any pinned hyper-parameter update (0/1) */
  int32_t trials;  /* BR: LM trials run */
  double value;    /* PNN: diverged loss; BR: mu when singular */
  double mu, gamma, alpha, beta; /* BR: final state (gamma NaN when not estimated) */
} bbml_model_status;

/* ---- library info ---- */
int32_t bbml_abi_version(void);
/* sizeof the ABI structs, for binding layout checks:
   0 bbml_seed, 1 bbml_pnn_task, 2 bbml_lm_task, 3 bbml_pred_task, 4 bbml_model_status */
int64_t bbml_struct_size(int32_t which);
const char* bbml_version(void);
const char* bbml_last_error(void);

/* ---- RNG (host functions, no GPU needed) ---- */
/* SeedSequence(words).generate_state(n_out, uint32) */
bbml_status bbml_seedseq_generate(const uint32_t* words, int32_t n_words, uint32_t* out,
                                  int32_t n_out);
/* PCG64 state after default_rng(seed): out = {state_hi, state_lo, inc_hi, inc_lo} */
bbml_status bbml_pcg64_state(const bbml_seed* seed, uint64_t* out4);

/* ---- training ---- */
/* precision: 64 = FP64 arithmetic (bit-faithful to the reference up to
   summation order), 32 = FP32 arithmetic (initial weights drawn in FP64). */
bbml_status bbml_pnn_train(const bbml_pnn_task* tasks, int32_t n_tasks, const double* X,
                           const double* y, int32_t x_stride, double* weights, double* history,
                           bbml_model_status* status, int32_t precision, void* stream);

bbml_status bbml_lm_train(const bbml_lm_task* tasks, int32_t n_tasks, const double* X,
                          const double* y, int32_t x_stride, double* weights, double* history,
                          bbml_model_status* status, void* stream);

/* ---- inference / extrapolation ---- */
bbml_status bbml_predict(const bbml_pred_task* tasks, int32_t n_tasks, const double* Xq,
                         int32_t x_stride, const double* weights, const double* norm,
                         double* out, void* stream);

/* ---- per-model test metrics ----
   Replaces the host loop over bbcount/metrics.py mse / pearson / spearman
   (metrics.py:33-76) as experiment.train_one applies them (experiment.py:128-152).
   Task i (bbml_pred_task reused): n test rows; actual_norm / actual_raw rows at
   row_begin; predictions (normalised) at w_offset of pred; norm_offset -> the
   series' [x_min(d), x_max(d), y_min, y_max] in norm.  Writes 4 doubles at
   out_offset: mse (normalised space), pearson and spearman of the de-normalised
   predictions vs actual_raw (NaN = undefined: constant vector or n < 2), and
   1.0 (Pearson / Spearman computed: always, any n -- test sets over 4096 rows
   take a counting-rank path in global memory). */
bbml_status bbml_metrics(const bbml_pred_task* tasks, int32_t n_tasks, const double* pred,
                         const double* actual_norm, const double* actual_raw,
                         const double* norm, double* out, void* stream);
/* Pooled correlations per group of models (experiment.summarize, experiment.py:
   180-206: Pearson / Spearman of the concatenated de-normalised predictions vs
   raw counts of every successful model of an (app, kind)).  seg_of: HOST, the
   group of each task (tasks of a group concatenate in task order).  out
   (device): 2 doubles per group {pearson, spearman}, NaN when undefined. */
bbml_status bbml_pooled_metrics(const bbml_pred_task* tasks, int32_t n_tasks,
                                const int32_t* seg_of, int32_t n_seg, const double* pred,
                                const double* actual_raw, const double* norm, double* out,
                                void* stream);
/* Per-model prediction-vs-actual heatmaps (metrics.heatmap_data, metrics.py:145-156):
   bins in [2, 200]; edges (device, bins+1 doubles per task) = linspace(0, max(pred, actual) or 1, bins+1),
   counts (device, bins*bins int32 per task, [pred_bin][actual_bin]) of histogram2d. */
bbml_status bbml_heatmaps(const bbml_pred_task* tasks, int32_t n_tasks, const double* pred,
                          const double* actual_raw, const double* norm, int32_t bins,
                          double* edges, int32_t* counts, void* stream);

/* Per-series count KDE (metrics.kde, metrics.py:95-118): series i = values[offsets[i] ..
   offsets[i+1]) (offsets: HOST, n_series + 1; values: device).  Out (device): grid and density
   (grid_points doubles per series) and the Scott bandwidth; bandwidth 0 = no curve (zero
   spread or n < 2, where the reference raises BandwidthError). */
bbml_status bbml_kde(const int64_t* offsets, int32_t n_series, const double* values,
                     int32_t grid_points, double* grid, double* density, double* bandwidth,
                     void* stream);

/* ---- unit-level kernels (one model per task; rows at row_begin, n rows) ---- */
/* loss[i] and grads (P doubles at w_offset of grads) of the batch NLL */
bbml_status bbml_pnn_loss_grad(const bbml_pred_task* tasks, int32_t n_tasks, const double* X,
                               const double* y, int32_t x_stride, const double* weights,
                               double nll_eps, double* loss, double* grads, void* stream);
/* J (n x P, row-major, at jac_offset[i] doubles; jac_offset is a HOST array; NULL jac =
   skip J) and the residual r = f(x) - y (n doubles at row_begin of resid) at weights
   w_offset; energies (device, optional) receives {E_D, E_W} per task (objective, 109-115) */
bbml_status bbml_lm_jacobian(const bbml_pred_task* tasks, int32_t n_tasks, const double* X,
                             const double* y, int32_t x_stride, const double* weights,
                             const int64_t* jac_offset, double* jac, double* resid,
                             double* energies, void* stream);
/* J'J (P*P at pp_offset[i]) and J'r (P at p_offset[i]) of J (n[i] x P[i] at j_offset[i])
   and r (n[i] at r_offset[i]).  P, n and the offsets are HOST tables. */
bbml_status bbml_lm_gram(const int32_t* P, const int32_t* n, int32_t n_tasks,
                         const int64_t* j_offset, const int64_t* r_offset,
                         const int64_t* pp_offset, const int64_t* p_offset, const double* J,
                         const double* r, double* jtj, double* jtr, void* stream);
/* pnn.adam_step on one flat vector of n_params split in blocks starting at block_begin
   (DEVICE, n_blocks entries).  bc1 = 1-beta1^t, bc2 = 1-beta2^t.  bad_block (device, 1 int)
   = first block with a non-finite gradient (blocks before it ARE updated, like the
   reference's dict loop) or -1. */
bbml_status bbml_adam_step(double* params, const double* grads, double* m, double* v,
                           int64_t n_params, const int64_t* block_begin, int32_t n_blocks,
                           double bc1, double bc2, double lr, double beta1, double beta2,
                           double eps, int32_t* bad_block, void* stream);
/* FMA-pipe peak microbenchmark: blocks x 256 threads x 8 chains x iters FMAs
   (FLOPs = 2 x that); precision 32 or 64.  out: device scratch (unused). */
bbml_status bbml_fma_peak(int32_t precision, int32_t blocks, int32_t iters, void* out,
                          void* stream);
/* y = 2/(1+exp(-2x)) - 1 elementwise (device arrays) */
bbml_status bbml_tansig(const double* x, double* y, int64_t n, void* stream);
/* delta = solve(beta J'J + (mu+alpha) I, -(beta J'r + alpha w)).
   P, pp_offset, p_offset: HOST task tables.  Device: jtj (P*P at pp_offset[i]),
   jtr / w / delta (P at p_offset[i]), abm (3 per task: alpha, beta, mu),
   info (1 per task: 0 ok, 1 singular -> brbpnn.NumericError). */
bbml_status bbml_lm_solve(const int32_t* P, int32_t n_tasks, const int64_t* pp_offset,
                          const int64_t* p_offset, const double* jtj, const double* jtr,
                          const double* w, const double* abm, double* delta, int32_t* info,
                          void* stream);
/* eigenvalues (unsorted, P at p_offset[i]) of jtj and the evidence update.
   Device: in5 = {e_d, e_w, alpha, beta, n}, out5 = {alpha, beta, gamma, pinned, 0} per task. */
bbml_status bbml_lm_evidence(const int32_t* P, int32_t n_tasks, const int64_t* pp_offset,
                             const int64_t* p_offset, const double* jtj, const double* in5,
                             double* eig, double* out5, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* BBML_H_ */
