// lm_train.cu — batched Bayesian-regularised Levenberg-Marquardt trainer
// (BR-BPNN), one model per CTA, all state FP64 in shared memory.
//
// Reference semantics (bbcount/brbpnn.py):
//   tansig 33-38, forward 85-91, pack/unpack 94-106, objective 109-115,
//   jacobian 118-130, solve_damped 153-171 (LAPACK dgesv: LU with partial
//   pivoting; exact zero pivot -> NumericError), lm_trial 174-196 (accept iff
//   F strictly decreases; mu*0.1 floored at 1e-20, else mu*10), lm_step
//   199-211 (stall when mu > mu_max), evidence_update 221-251 (eigenvalues of
//   J'J clipped at 0, gamma = sum beta*l/(beta*l+alpha) with the OLD alpha,beta,
//   pinned clamps), train 286-346 (records, early stop after 5 stable epochs).
//
// Per epoch the kernel forms J'J and J'r ONCE at the accepted weights and
// reuses them for (a) the evidence update and (b) every LM trial of the next
// epoch (the reference recomputes the identical J at the same w each trial).
// J rows are staged CH at a time in shared memory and contracted into the
// upper triangle; LU + triangular solves and a parallel cyclic Jacobi
// eigen-solver run in shared memory.
#include <algorithm>
#include <vector>

#include "common.cuh"
#include "launch.h"
#include "pcg64.cuh"

namespace bbml {

constexpr int LM_NT = 128;
constexpr int LM_WARPS = LM_NT / 32;

struct LmSmem {
  double* w;      // [P]
  double* wt;     // [P] trial weights
  double* delta;  // [P]
  double* jtr;    // [P]
  double* rhs;    // [P]
  double* jtj;    // [P*P] full symmetric
  double* A;      // [P*P] LU / Jacobi workspace
  double* Jc;     // [CH*P] staged Jacobian rows
  double* rc;     // [CH] staged residuals
  double* cs;     // [2*(P+1)] Jacobi rotations
  double* red;    // [LM_WARPS + 2] reductions
  int* piv;       // [P]
  int* flag;      // [4]
};

// block-wide deterministic sum (fixed tree); result broadcast to all threads
__device__ double block_sum(double v, double* red) {
  for (int m = 16; m >= 1; m >>= 1) v += __shfl_xor_sync(0xffffffffu, v, m);
  const int warp = threadIdx.x >> 5;
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[warp] = v;
  __syncthreads();
  double s = red[0];
  for (int i = 1; i < LM_WARPS; ++i) s += red[i];
  return s;
}

// brbpnn.forward for one sample; optionally the Jacobian row (pack order)
__device__ __forceinline__ double br_sample(const double* __restrict__ w, const double* x, int d,
                                            int h, double* jrow) {
  const int hd = h * d;
  double out = 0.0;
  for (int j = 0; j < h; ++j) {
    double pre = 0.0;
    for (int k = 0; k < d; ++k) pre = fma(x[k], w[j * d + k], pre);
    pre = __dadd_rn(pre, w[hd + j]);
    const double a = tansig(pre);
    const double w2 = w[hd + h + j];
    out = fma(a, w2, out);
    if (jrow) {
      const double da = __dmul_rn(__dsub_rn(1.0, __dmul_rn(a, a)), w2);
      for (int k = 0; k < d; ++k) jrow[j * d + k] = __dmul_rn(da, x[k]);
      jrow[hd + j] = da;
      jrow[hd + h + j] = a;
    }
  }
  if (jrow) jrow[hd + 2 * h] = 1.0;
  return __dadd_rn(out, w[hd + 2 * h]);
}

// E_D = sum r^2 at weights wv (objective, brbpnn.py:109-115)
__device__ double energy_pass(const double* wv, const double* X, const double* Y, int n, int d,
                              int h, int xs, double* red) {
  double acc = 0.0;
  double x[BBML_MAX_INPUTS];
  for (int i = threadIdx.x; i < n; i += LM_NT) {
    for (int k = 0; k < d; ++k) x[k] = __ldg(X + (int64_t)i * xs + k);
    const double r = __dsub_rn(br_sample(wv, x, d, h, nullptr), __ldg(Y + i));
    acc = fma(r, r, acc);
  }
  return block_sum(acc, red);
}

// J'J (full) and J'r at weights S.w
template <int CH>
__device__ void stats_pass(LmSmem& S, const double* X, const double* Y, int n, int d, int h, int P,
                           int xs) {
  const int npair = P * (P + 1) / 2;
  for (int e = threadIdx.x; e < P * P; e += LM_NT) S.jtj[e] = 0.0;
  for (int e = threadIdx.x; e < P; e += LM_NT) S.jtr[e] = 0.0;
  __syncthreads();
  double x[BBML_MAX_INPUTS];
  for (int base = 0; base < n; base += CH) {
    const int cnt = min(CH, n - base);
    for (int c = threadIdx.x; c < cnt; c += LM_NT) {
      const int i = base + c;
      for (int k = 0; k < d; ++k) x[k] = __ldg(X + (int64_t)i * xs + k);
      S.rc[c] = __dsub_rn(br_sample(S.w, x, d, h, S.Jc + c * P), __ldg(Y + i));
    }
    __syncthreads();
    for (int e = threadIdx.x; e < npair + P; e += LM_NT) {
      if (e < npair) {
        // e -> (a, b) with a <= b, row-major upper triangle
        int a = 0, rem = e;
        while (rem >= P - a) {
          rem -= P - a;
          ++a;
        }
        const int b = a + rem;
        double s = S.jtj[a * P + b];
        for (int c = 0; c < cnt; ++c) s = fma(S.Jc[c * P + a], S.Jc[c * P + b], s);
        S.jtj[a * P + b] = s;
      } else {
        const int a = e - npair;
        double s = S.jtr[a];
        for (int c = 0; c < cnt; ++c) s = fma(S.Jc[c * P + a], S.rc[c], s);
        S.jtr[a] = s;
      }
    }
    __syncthreads();
  }
  for (int e = threadIdx.x; e < P * P; e += LM_NT) {
    const int a = e / P, b = e % P;
    if (a > b) S.jtj[e] = S.jtj[b * P + a];
  }
  __syncthreads();
}

// delta = solve(beta J'J + (mu+alpha) I, -(beta J'r + alpha w)); returns false on a zero pivot
__device__ bool damped_solve(LmSmem& S, int P, double alpha, double beta, double mu) {
  const double damp = __dadd_rn(mu, alpha);
  for (int e = threadIdx.x; e < P * P; e += LM_NT) {
    const int a = e / P, b = e % P;
    const double v = __dmul_rn(beta, S.jtj[e]);
    S.A[e] = (a == b) ? __dadd_rn(v, damp) : v;
  }
  for (int a = threadIdx.x; a < P; a += LM_NT)
    S.rhs[a] = -__dadd_rn(__dmul_rn(beta, S.jtr[a]), __dmul_rn(alpha, S.w[a]));
  __syncthreads();
  // LU with partial pivoting (right-looking, dgetf2 order), row swaps applied to rhs
  for (int k = 0; k < P; ++k) {
    if (threadIdx.x < 32) {
      double best = -1.0;
      int bi = k;
      for (int i = k + threadIdx.x; i < P; i += 32) {
        const double v = fabs(S.A[i * P + k]);
        if (v > best) {
          best = v;
          bi = i;
        }
      }
      for (int m = 16; m >= 1; m >>= 1) {
        const double ob = __shfl_xor_sync(0xffffffffu, best, m);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, m);
        if (ob > best || (ob == best && oi < bi)) {
          best = ob;
          bi = oi;
        }
      }
      if (threadIdx.x == 0) S.piv[k] = bi;
    }
    __syncthreads();
    const int p = S.piv[k];
    if (S.A[p * P + k] == 0.0) return false;  // uniform across the block
    if (p != k) {
      for (int j = threadIdx.x; j < P; j += LM_NT) {
        const double t = S.A[k * P + j];
        S.A[k * P + j] = S.A[p * P + j];
        S.A[p * P + j] = t;
      }
      if (threadIdx.x == 0) {
        const double t = S.rhs[k];
        S.rhs[k] = S.rhs[p];
        S.rhs[p] = t;
      }
    }
    __syncthreads();
    const double piv = S.A[k * P + k];
    const int m = P - k - 1;
    for (int e = threadIdx.x; e < m; e += LM_NT) {
      const int i = k + 1 + e;
      S.A[i * P + k] = __ddiv_rn(S.A[i * P + k], piv);
    }
    __syncthreads();
    for (int e = threadIdx.x; e < m * m; e += LM_NT) {
      const int i = k + 1 + e / m, j = k + 1 + e % m;
      S.A[i * P + j] = fma(-S.A[i * P + k], S.A[k * P + j], S.A[i * P + j]);
    }
    __syncthreads();
  }
  // forward (unit L) then backward (U) substitution by warp 0
  if (threadIdx.x < 32) {
    for (int i = 0; i < P; ++i) {
      double s = 0.0;
      for (int j = threadIdx.x; j < i; j += 32) s = fma(S.A[i * P + j], S.rhs[j], s);
      for (int mm = 16; mm >= 1; mm >>= 1) s += __shfl_xor_sync(0xffffffffu, s, mm);
      if (threadIdx.x == 0) S.rhs[i] = __dsub_rn(S.rhs[i], s);
      __syncwarp();
    }
    for (int i = P - 1; i >= 0; --i) {
      double s = 0.0;
      for (int j = i + 1 + threadIdx.x; j < P; j += 32) s = fma(S.A[i * P + j], S.delta[j], s);
      for (int mm = 16; mm >= 1; mm >>= 1) s += __shfl_xor_sync(0xffffffffu, s, mm);
      if (threadIdx.x == 0) S.delta[i] = __ddiv_rn(__dsub_rn(S.rhs[i], s), S.A[i * P + i]);
      __syncwarp();
    }
  }
  __syncthreads();
  return true;
}

// eigenvalues of S.jtj (copied into S.A) by parallel cyclic Jacobi; returns
// gamma = sum beta*l/(beta*l+alpha) over eigenvalues clipped at 0
__device__ double jacobi_gamma(LmSmem& S, int P, double alpha, double beta, double* eig_out) {
  for (int e = threadIdx.x; e < P * P; e += LM_NT) S.A[e] = S.jtj[e];
  __syncthreads();
  const int Pp = (P + 1) & ~1;  // even player count; index P (if odd) is a bye
  const int npairs = Pp / 2;
  for (int sweep = 0; sweep < 40; ++sweep) {
    if (threadIdx.x == 0) S.flag[0] = 0;
    __syncthreads();
    for (int r = 0; r < Pp - 1; ++r) {
      for (int k = threadIdx.x; k < npairs; k += LM_NT) {
        const int pa = (k == 0) ? 0 : 1 + ((k - 1 + r) % (Pp - 1));
        const int qa = 1 + ((Pp - 2 - k + r) % (Pp - 1));
        int p = min(pa, qa), q = max(pa, qa);
        double c = 1.0, s = 0.0;
        if (q < P) {
          const double apq = S.A[p * P + q];
          const double app = S.A[p * P + p], aqq = S.A[q * P + q];
          if (fabs(apq) > 1e-300 && fabs(apq) > 1e-15 * sqrt(fabs(app * aqq))) {
            const double tau = (aqq - app) / (2.0 * apq);
            const double t = (tau >= 0.0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
            c = 1.0 / sqrt(1.0 + t * t);
            s = t * c;
            S.flag[0] = 1;
          }
        }
        S.cs[2 * k] = c;
        S.cs[2 * k + 1] = s;
      }
      __syncthreads();
      // columns: A <- A J
      for (int e = threadIdx.x; e < npairs * P; e += LM_NT) {
        const int k = e / P, i = e % P;
        const double s = S.cs[2 * k + 1];
        if (s == 0.0) continue;
        const int pa = (k == 0) ? 0 : 1 + ((k - 1 + r) % (Pp - 1));
        const int qa = 1 + ((Pp - 2 - k + r) % (Pp - 1));
        const int p = min(pa, qa), q = max(pa, qa);
        const double c = S.cs[2 * k];
        const double aip = S.A[i * P + p], aiq = S.A[i * P + q];
        S.A[i * P + p] = c * aip - s * aiq;
        S.A[i * P + q] = s * aip + c * aiq;
      }
      __syncthreads();
      // rows: A <- J' A
      for (int e = threadIdx.x; e < npairs * P; e += LM_NT) {
        const int k = e / P, j = e % P;
        const double s = S.cs[2 * k + 1];
        if (s == 0.0) continue;
        const int pa = (k == 0) ? 0 : 1 + ((k - 1 + r) % (Pp - 1));
        const int qa = 1 + ((Pp - 2 - k + r) % (Pp - 1));
        const int p = min(pa, qa), q = max(pa, qa);
        const double c = S.cs[2 * k];
        const double apj = S.A[p * P + j], aqj = S.A[q * P + j];
        // the rotation annihilates (p,q) exactly; store the zero so rounding
        // noise cannot keep the sweep alive
        S.A[p * P + j] = (j == q) ? 0.0 : c * apj - s * aqj;
        S.A[q * P + j] = (j == p) ? 0.0 : s * apj + c * aqj;
      }
      __syncthreads();
    }
    if (S.flag[0] == 0) break;
    __syncthreads();
  }
  double part = 0.0;
  for (int i = threadIdx.x; i < P; i += LM_NT) {
    const double lam = fmax(S.A[i * P + i], 0.0);
    if (eig_out) eig_out[i] = S.A[i * P + i];
    const double sc = __dmul_rn(beta, lam);
    const double den = __dadd_rn(sc, alpha);
    part += den > 0.0 ? __ddiv_rn(sc, den) : 0.0;
  }
  // deterministic: gather per-thread partials in thread order
  __syncthreads();
  if (threadIdx.x < P) S.rc[threadIdx.x] = part;
  __syncthreads();
  double g = 0.0;
  for (int i = 0; i < min(P, LM_NT); ++i) g += S.rc[i];
  __syncthreads();
  return g;
}

template <int PMAX, int CH>
__global__ void __launch_bounds__(LM_NT) lm_train_kernel(LmLaunch L) {
  const int task = blockIdx.x;
  if (task >= L.n_tasks) return;
  const bbml_lm_task tk = L.tasks[task];
  const int orig = L.orig_index[task];
  const int n = tk.n, d = tk.d, h = tk.h;
  const int P = h * (d + 2) + 1;
  const int xs = L.x_stride;
  const double* X = L.X + tk.row_begin * (int64_t)xs;
  const double* Y = L.y + tk.row_begin;

  extern __shared__ double sm[];
  LmSmem S;
  double* q = sm;
  S.w = q; q += PMAX;
  S.wt = q; q += PMAX;
  S.delta = q; q += PMAX;
  S.jtr = q; q += PMAX;
  S.rhs = q; q += PMAX;
  S.jtj = q; q += PMAX * PMAX;
  S.A = q; q += PMAX * PMAX;
  S.Jc = q; q += CH * PMAX;
  S.rc = q; q += (CH > LM_NT ? CH : LM_NT);
  S.cs = q; q += 2 * (PMAX + 2);
  S.red = q; q += LM_WARPS + 2;
  S.piv = (int*)q; q += (PMAX + 1) / 2 + 1;
  S.flag = (int*)q;

  // init (brbpnn.py:323-331): thread 0 draws P uniforms in pack order
  if (threadIdx.x == 0) {
    Pcg64 rng;
    rng.seed(tk.seed);
    const double s1 = __ddiv_rn(1.0, __dsqrt_rn((double)d));
    const double s2 = __ddiv_rn(1.0, __dsqrt_rn((double)h));
    const int hd = h * d;
    for (int i = 0; i < hd + h; ++i) S.w[i] = rng.uniform(-s1, s1);
    for (int i = hd + h; i < P; ++i) S.w[i] = rng.uniform(-s2, s2);
  }
  __syncthreads();

  double alpha = tk.alpha0, beta = tk.beta0, mu = tk.mu0;
  const bool est = tk.estimate != 0;
  double* hist = (tk.hist_offset >= 0) ? L.history + tk.hist_offset : nullptr;

  double e_d = energy_pass(S.w, X, Y, n, d, h, xs, S.red);
  double e_w = 0.0;
  for (int i = 0; i < P; ++i) e_w = fma(S.w[i], S.w[i], e_w);
  bool have_stats = false;
  int code = BBML_MODEL_OK, trials = 0, epochs = 0, any_pinned = 0;
  double fail_mu = 0.0, last_mu = NAN, last_gamma = NAN;
  double prev_g = 0.0, prev_d = 0.0, prev_w = 0.0;
  bool have_prev = false;
  int stable = 0;

  for (int ep = 0; ep < tk.max_epochs; ++ep) {
    if (!have_stats) stats_pass<CH>(S, X, Y, n, d, h, P, xs);
    const double f0 = __dadd_rn(__dmul_rn(beta, e_d), __dmul_rn(alpha, e_w));
    bool accepted = false;
    double td = 0.0, tw = 0.0;
    while (true) {
      ++trials;
      if (!damped_solve(S, P, alpha, beta, mu)) {
        code = BBML_MODEL_SINGULAR;
        fail_mu = mu;
        break;
      }
      for (int i = threadIdx.x; i < P; i += LM_NT) S.wt[i] = __dadd_rn(S.w[i], S.delta[i]);
      __syncthreads();
      td = energy_pass(S.wt, X, Y, n, d, h, xs, S.red);
      tw = 0.0;
      for (int i = 0; i < P; ++i) tw = fma(S.wt[i], S.wt[i], tw);
      const double f1 = __dadd_rn(__dmul_rn(beta, td), __dmul_rn(alpha, tw));
      if (f1 < f0) {
        mu = fmax(__dmul_rn(mu, tk.mu_dec), 1e-20);
        accepted = true;
        break;
      }
      mu = __dmul_rn(mu, tk.mu_inc);
      if (mu > tk.mu_max) break;
    }
    if (code != BBML_MODEL_OK || !accepted) break;
    __syncthreads();
    for (int i = threadIdx.x; i < P; i += LM_NT) S.w[i] = S.wt[i];
    __syncthreads();
    e_d = td;
    e_w = tw;
    const double f1 = __dadd_rn(__dmul_rn(beta, e_d), __dmul_rn(alpha, e_w));
    double gamma = NAN;
    int pinned = 0;
    if (est) {
      stats_pass<CH>(S, X, Y, n, d, h, P, xs);
      have_stats = true;
      gamma = jacobi_gamma(S, P, alpha, beta, nullptr);
      double na, nb;
      if (e_w > 0.0) {
        na = __ddiv_rn(gamma, __dmul_rn(2.0, e_w));
      } else {
        na = 1e12;
        pinned = 1;
      }
      if (e_d > 0.0) {
        nb = __ddiv_rn(__dsub_rn((double)n, gamma), __dmul_rn(2.0, e_d));
      } else {
        nb = 1e12;
        pinned = 1;
      }
      alpha = fmin(fmax(na, 1e-12), 1e12);
      beta = fmin(fmax(nb, 1e-12), 1e12);
    } else {
      have_stats = false;
    }
    any_pinned |= pinned;
    last_mu = mu;
    last_gamma = gamma;
    epochs = ep + 1;
    if (hist && threadIdx.x == 0) {
      double* r = hist + (int64_t)ep * 10;
      r[0] = ep; r[1] = f0; r[2] = f1; r[3] = e_d; r[4] = e_w;
      r[5] = alpha; r[6] = beta; r[7] = gamma; r[8] = mu; r[9] = pinned;
    }
    if (have_prev && est) {
      const bool ok = fabs(gamma - prev_g) <= 1e-7 * fmax(fabs(prev_g), 1e-300) &&
                      fabs(e_d - prev_d) <= 1e-7 * fmax(fabs(prev_d), 1e-300) &&
                      fabs(e_w - prev_w) <= 1e-7 * fmax(fabs(prev_w), 1e-300);
      if (ok) {
        if (++stable >= 5) break;
      } else {
        stable = 0;
      }
    }
    prev_g = gamma;
    prev_d = e_d;
    prev_w = e_w;
    have_prev = true;
  }

  __syncthreads();
  double* W = L.weights + tk.w_offset;
  for (int i = threadIdx.x; i < P; i += LM_NT) W[i] = S.w[i];
  if (threadIdx.x == 0) {
    bbml_model_status st{};
    st.code = code;
    st.epochs = epochs;
    st.detail = any_pinned;
    st.trials = trials;
    st.value = fail_mu;
    st.mu = last_mu;
    st.gamma = last_gamma;
    st.alpha = alpha;
    st.beta = beta;
    L.status[orig] = st;
  }
}

template <int PMAX, int CH>
static size_t lm_smem_bytes() {
  size_t dbl = 5 * PMAX + 2 * PMAX * PMAX + CH * PMAX + (CH > LM_NT ? CH : LM_NT) +
               2 * (PMAX + 2) + LM_WARPS + 2 + (PMAX + 1) / 2 + 1 + 4;
  return dbl * sizeof(double);
}

template <int PMAX, int CH>
static cudaError_t lm_launch_bucket(const LmLaunch& L, cudaStream_t s) {
  const size_t smem = lm_smem_bytes<PMAX, CH>();
  auto k = lm_train_kernel<PMAX, CH>;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  k<<<L.n_tasks, LM_NT, smem, s>>>(L);
  return cudaGetLastError();
}

static int lm_bucket(int P) { return P <= 8 ? 8 : P <= 32 ? 32 : P <= 64 ? 64 : 96; }

bbml_status lm_train_launch(const bbml_lm_task* tasks, int32_t n_tasks, const double* X,
                            const double* y, int32_t x_stride, double* weights, double* history,
                            bbml_model_status* status, cudaStream_t stream) {
  std::vector<int> idx(n_tasks);
  for (int i = 0; i < n_tasks; ++i) {
    const bbml_lm_task& t = tasks[i];
    if (t.n < 1 || t.d < 1 || t.h < 1 || t.max_epochs < 0 || t.row_begin < 0 || t.w_offset < 0 ||
        t.seed.n_words < 1 || t.seed.n_words > BBML_MAX_ENTROPY_WORDS) {
      set_error("lm task %d: invalid field", i);
      return BBML_ERR_INVALID;
    }
    const int P = t.h * (t.d + 2) + 1;
    if (t.d > BBML_MAX_INPUTS || P > 96) {
      set_error("lm task %d: d=%d h=%d (P=%d) outside the supported envelope", i, t.d, t.h, P);
      return BBML_ERR_UNSUPPORTED;
    }
    if (t.hist_offset >= 0 && history == nullptr) {
      set_error("lm task %d: history requested but history == NULL", i);
      return BBML_ERR_INVALID;
    }
    idx[i] = i;
  }
  auto P_of = [&](int i) { return tasks[i].h * (tasks[i].d + 2) + 1; };
  std::stable_sort(idx.begin(), idx.end(), [&](int a, int b) {
    const int ka = lm_bucket(P_of(a)), kb = lm_bucket(P_of(b));
    if (ka != kb) return ka > kb;
    const double ca = (double)tasks[a].n * P_of(a) * P_of(a);
    const double cb = (double)tasks[b].n * P_of(b) * P_of(b);
    return ca > cb;
  });
  std::vector<bbml_lm_task> sorted(n_tasks);
  std::vector<int32_t> orig(n_tasks);
  for (int i = 0; i < n_tasks; ++i) {
    sorted[i] = tasks[idx[i]];
    orig[i] = idx[i];
  }
  ScratchBuffer scratch(stream);
  bbml_lm_task* d_tasks = nullptr;
  int32_t* d_orig = nullptr;
  bbml_status st;
  if ((st = scratch.alloc(&d_tasks, n_tasks)) != BBML_OK) return st;
  if ((st = scratch.alloc(&d_orig, n_tasks)) != BBML_OK) return st;
  if ((st = scratch.upload(d_tasks, sorted.data(), n_tasks)) != BBML_OK) return st;
  if ((st = scratch.upload(d_orig, orig.data(), n_tasks)) != BBML_OK) return st;
  int begin = 0;
  while (begin < n_tasks) {
    const int b = lm_bucket(P_of(idx[begin]));
    int end = begin;
    while (end < n_tasks && lm_bucket(P_of(idx[end])) == b) ++end;
    LmLaunch L{};
    L.tasks = d_tasks + begin;
    L.orig_index = d_orig + begin;
    L.n_tasks = end - begin;
    L.x_stride = x_stride;
    L.pmax = b;
    L.X = X;
    L.y = y;
    L.weights = weights;
    L.history = history;
    L.status = status;
    cudaError_t e;
    if (b == 8) e = lm_launch_bucket<8, 128>(L, stream);
    else if (b == 32) e = lm_launch_bucket<32, 64>(L, stream);
    else if (b == 64) e = lm_launch_bucket<64, 32>(L, stream);
    else e = lm_launch_bucket<96, 16>(L, stream);
    if (e != cudaSuccess) return cuda_status(e, "lm_train launch");
    begin = end;
  }
  return scratch.release();
}

}  // namespace bbml

// ------------------------------------------------------------------------
// unit-level kernels (brbpnn.jacobian/objective, solve_damped, evidence_update)
// ------------------------------------------------------------------------
namespace bbml {

__global__ void __launch_bounds__(LM_NT)
    lm_jacobian_kernel(const bbml_pred_task* __restrict__ tasks, const int64_t* __restrict__ joff,
                       const double* __restrict__ X, const double* __restrict__ Y, int xs,
                       const double* __restrict__ weights, double* __restrict__ jac,
                       double* __restrict__ resid, double* __restrict__ energies) {
  __shared__ double red[LM_WARPS + 2];
  const bbml_pred_task tk = tasks[blockIdx.x];
  const int P = tk.h * (tk.d + 2) + 1;
  const double* w = weights + tk.w_offset;
  double x[BBML_MAX_INPUTS];
  double acc = 0.0;
  for (int i = threadIdx.x; i < tk.n; i += LM_NT) {
    const int64_t row = tk.row_begin + i;
    for (int k = 0; k < tk.d; ++k) x[k] = X[row * xs + k];
    double* jrow = jac ? jac + joff[blockIdx.x] + (int64_t)i * P : nullptr;
    const double r = __dsub_rn(br_sample(w, x, tk.d, tk.h, jrow), Y[row]);
    resid[row] = r;
    acc = fma(r, r, acc);
  }
  const double e_d = block_sum(acc, red);
  if (energies && threadIdx.x == 0) {
    double e_w = 0.0;
    for (int i = 0; i < P; ++i) e_w = fma(w[i], w[i], e_w);
    energies[2 * blockIdx.x] = e_d;
    energies[2 * blockIdx.x + 1] = e_w;
  }
}

template <int PMAX>
__global__ void lm_unit_kernel(int mode, const int32_t* __restrict__ Ps,
                               const int64_t* __restrict__ pp_off, const int64_t* __restrict__ p_off,
                               const double* __restrict__ jtj, const double* __restrict__ jtr,
                               const double* __restrict__ w, const double* __restrict__ params,
                               double* __restrict__ out_vec, double* __restrict__ out5,
                               int32_t* __restrict__ info) {
  const int t = blockIdx.x;
  const int P = Ps[t];
  extern __shared__ double sm[];
  LmSmem S;
  double* q = sm;
  S.w = q; q += PMAX;
  S.wt = q; q += PMAX;
  S.delta = q; q += PMAX;
  S.jtr = q; q += PMAX;
  S.rhs = q; q += PMAX;
  S.jtj = q; q += PMAX * PMAX;
  S.A = q; q += PMAX * PMAX;
  S.Jc = nullptr;
  S.rc = q; q += LM_NT;
  S.cs = q; q += 2 * (PMAX + 2);
  S.red = q; q += LM_WARPS + 2;
  S.piv = (int*)q; q += (PMAX + 1) / 2 + 1;
  S.flag = (int*)q;
  for (int e = threadIdx.x; e < P * P; e += LM_NT) S.jtj[e] = jtj[pp_off[t] + e];
  if (mode == 0)
    for (int e = threadIdx.x; e < P; e += LM_NT) {
      S.jtr[e] = jtr[p_off[t] + e];
      S.w[e] = w[p_off[t] + e];
    }
  __syncthreads();
  if (mode == 0) {
    const double* abm = params + 3 * t;  // alpha, beta, mu
    const bool ok = damped_solve(S, P, abm[0], abm[1], abm[2]);
    for (int e = threadIdx.x; e < P; e += LM_NT) out_vec[p_off[t] + e] = ok ? S.delta[e] : NAN;
    if (threadIdx.x == 0) info[t] = ok ? 0 : 1;
  } else {
    const double* in5 = params + 5 * t;  // e_d, e_w, alpha, beta, n
    const double e_d = in5[0], e_w = in5[1], alpha = in5[2], beta = in5[3], n = in5[4];
    const double gamma = jacobi_gamma(S, P, alpha, beta, out_vec + p_off[t]);
    if (threadIdx.x == 0) {
      int pinned = 0;
      double na, nb;
      if (e_w > 0.0) na = gamma / (2.0 * e_w); else { na = 1e12; pinned = 1; }
      if (e_d > 0.0) nb = (n - gamma) / (2.0 * e_d); else { nb = 1e12; pinned = 1; }
      double* o = out5 + 5 * t;
      o[0] = fmin(fmax(na, 1e-12), 1e12);
      o[1] = fmin(fmax(nb, 1e-12), 1e12);
      o[2] = gamma;
      o[3] = pinned;
      o[4] = 0.0;
    }
  }
}

bbml_status lm_jacobian_launch(const bbml_pred_task* tasks, int32_t n_tasks, const double* X,
                               const double* y, int32_t xs, const double* weights,
                               const int64_t* jac_offset, double* jac, double* resid,
                               double* energies, cudaStream_t s) {
  if (n_tasks == 0) return BBML_OK;
  for (int i = 0; i < n_tasks; ++i)
    if (tasks[i].d < 1 || tasks[i].h < 1 || tasks[i].n < 0 || tasks[i].d > BBML_MAX_INPUTS) {
      set_error("jacobian task %d: invalid field", i);
      return BBML_ERR_INVALID;
    }
  ScratchBuffer scratch(s);
  bbml_pred_task* d_tasks = nullptr;
  int64_t* d_off = nullptr;
  bbml_status st;
  if ((st = scratch.alloc(&d_tasks, n_tasks)) != BBML_OK) return st;
  if ((st = scratch.alloc(&d_off, n_tasks)) != BBML_OK) return st;
  if ((st = scratch.upload(d_tasks, tasks, n_tasks)) != BBML_OK) return st;
  if (jac && (st = scratch.upload(d_off, jac_offset, n_tasks)) != BBML_OK) return st;
  lm_jacobian_kernel<<<n_tasks, LM_NT, 0, s>>>(d_tasks, d_off, X, y, xs, weights, jac, resid,
                                               energies);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_status(e, "jacobian launch");
  return scratch.release();
}

bbml_status lm_unit_launch(int mode, const int32_t* P, int32_t n_tasks, const int64_t* pp_offset,
                           const int64_t* p_offset, const double* jtj, const double* jtr,
                           const double* w, const double* params, int n_params_per_task,
                           double* out_vec, double* out5, int32_t* info, cudaStream_t s) {
  if (n_tasks == 0) return BBML_OK;
  int pmax = 0;
  for (int i = 0; i < n_tasks; ++i) {
    if (P[i] < 1 || P[i] > 96) {
      set_error("lm unit task %d: P=%d outside 1..96", i, P[i]);
      return BBML_ERR_UNSUPPORTED;
    }
    pmax = std::max(pmax, P[i]);
  }
  ScratchBuffer scratch(s);
  int32_t* dP = nullptr;
  int64_t *dpp = nullptr, *dp = nullptr;
  bbml_status st;
  if ((st = scratch.alloc(&dP, n_tasks)) != BBML_OK) return st;
  if ((st = scratch.alloc(&dpp, n_tasks)) != BBML_OK) return st;
  if ((st = scratch.alloc(&dp, n_tasks)) != BBML_OK) return st;
  if ((st = scratch.upload(dP, P, n_tasks)) != BBML_OK) return st;
  if ((st = scratch.upload(dpp, pp_offset, n_tasks)) != BBML_OK) return st;
  if ((st = scratch.upload(dp, p_offset, n_tasks)) != BBML_OK) return st;
  const int PM = 96;
  const size_t smem = (5 * PM + 2 * PM * PM + LM_NT + 2 * (PM + 2) + LM_WARPS + 2 + (PM + 1) / 2 + 1 + 4) *
                      sizeof(double);
  auto k = lm_unit_kernel<96>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k<<<n_tasks, LM_NT, smem, s>>>(mode, dP, dpp, dp, jtj, jtr, w, params, out_vec, out5, info);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_status(e, "lm unit launch");
  (void)n_params_per_task;
  return scratch.release();
}

}  // namespace bbml
