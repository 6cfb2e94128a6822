// lm_train.cu — batched Bayesian-regularised Levenberg-Marquardt trainer
// (BR-BPNN), all state FP64.  Training kernels: one model per warp
// (`lm_warp_kernel<PM, D>`, P <= 8 / P <= 32, workspace in shared memory),
// one model per CTA of 4 warps for hidden-1 series with n >= 2048, and the
// wide CTA-per-model kernel in lm_wide.cu (P <= 512).  The CTA helpers at the
// top (LmSmem, damped_solve, jacobi_gamma) serve the unit-level entry points.
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
// Per epoch a model forms J'J and J'r ONCE at the accepted weights and reuses
// them for (a) the evidence update and (b) every LM trial of the next epoch
// (the reference recomputes the identical J at the same w each trial).
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "common.cuh"
#include "sturm.cuh"
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


// ===========================================================================
// Warp-per-model LM trainer for P <= 32 (all hidden-1 models, and hidden 10
// at d = 1, e.g. gramschmit): no block barriers at all.  Lanes stride over
// samples for the energy / Jacobian passes.  Hidden-1 models (the paper's
// default) use a compile-time-shaped path: weights, the
// Jacobian row and the 1/2 P(P+1) + P accumulators of J'J | J'r live in
// registers.  Other shapes stage 32 Jacobian rows in shared memory and
// contract them lane-parallel.  LU with partial pivoting and the cyclic
// Jacobi eigen-solver run lane-parallel on a per-warp shared-memory copy
// (odd row stride: conflict-free column access), synchronised with
// __syncwarp only.
// ===========================================================================
template <int PM>
struct alignas(16) WarpLm {
  static constexpr int LD = PM + 1;
  static constexpr int NE = PM * (PM + 1) / 2 + PM;
  double w[PM], wt[PM], delta[PM], jtr[PM], rhs[PM];
  double jtj[PM * LD];
  double A[PM * LD];
  // PM = 32 (statistics staged in A, Householder + bisection gamma) only needs
  // the tridiagonal (dd, e2, ee) here; the per-entry statistics tables and the
  // Jacobi schedule exist for PM = 8 only (smaller footprint -> more warps/SM)
  static constexpr bool kWide = PM > 8;
  static constexpr int JCH = kWide ? 5 : 32;  // staged Jacobian rows per chunk (PM = 8);
                                              // PM = 32: dd, e2, ee, {d, e^2} rows
  double Jc[JCH * PM];
  double rc[kWide ? 2 : JCH];
  double cs[kWide ? 2 : 2 * 16];
  int pq[kWide ? 2 : 16];
  unsigned short ent[kWide ? 4 : NE];  // (a << 8 | b) for the upper triangle, b == P -> J'r
  unsigned short rr[kWide ? 4 : (PM - 1) * (PM / 2)];  // round-robin pair schedule (p | q << 8)
};

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int m = 16; m >= 1; m >>= 1) v += __shfl_xor_sync(0xffffffffu, v, m);
  return v;
}

// hidden-1 model with D inputs, pack order [W1 (D), b1, W2, b2]
template <int D>
struct H1 {
  double w1[D], b1, w2, b2;
  __device__ __forceinline__ void load(const double* w) {
#pragma unroll
    for (int k = 0; k < D; ++k) w1[k] = w[k];
    b1 = w[D];
    w2 = w[D + 1];
    b2 = w[D + 2];
  }
  // forward exactly as br_sample: dot, + b1, tansig, a*w2 (+0), + b2
  __device__ __forceinline__ double out(const double (&x)[D], double& a) const {
    double pre = 0.0;
#pragma unroll
    for (int k = 0; k < D; ++k) pre = fma(x[k], w1[k], pre);
    a = tansig(__dadd_rn(pre, b1));
    return __dadd_rn(fma(a, w2, 0.0), b2);
  }
};

template <int D>
__device__ __forceinline__ void load_x(double (&x)[D], const double* X, int64_t i, int xs) {
#pragma unroll
  for (int k = 0; k < D; ++k) x[k] = __ldg(X + i * xs + k);
}

// Per-sample passes take a sample split (sw of NW warps sharing one model;
// NW = 1: the warp owns the model and the lane's sample order is i = lane,
// lane + 32, ...).  They return / store warp-level sums; NW > 1 callers
// reduce across warps.
template <int PM, int D, int NW = 1>
__device__ double w_energy(const WarpLm<PM>& S, const double* wv, const double* X, const double* Y,
                           int n, int d, int h, int xs, int lane, int sw = 0) {
  double acc = 0.0;
  constexpr int ST = 32 * NW;
  if constexpr (D > 0) {
    H1<D> m;
    m.load(wv);
    // 8 samples per lane per iteration, all loads issued first (L2 latency)
    // then independent exp/div chains (ILP); the accumulation order stays the
    // sample order of the lane
    constexpr int U8 = 8;
    int i = sw * 32 + lane;
    for (; i + ST * (U8 - 1) < n; i += ST * U8) {
      double xv[U8][D], yv[U8], r[U8];
#pragma unroll
      for (int u = 0; u < U8; ++u) {
        load_x<D>(xv[u], X, i + ST * u, xs);
        yv[u] = __ldg(Y + i + ST * u);
      }
#pragma unroll
      for (int u = 0; u < U8; ++u) {
        double a;
        r[u] = __dsub_rn(m.out(xv[u], a), yv[u]);
      }
#pragma unroll
      for (int u = 0; u < U8; ++u) acc = fma(r[u], r[u], acc);
    }
    for (; i < n; i += ST) {
      double x[D];
      load_x<D>(x, X, i, xs);
      double a;
      const double r = __dsub_rn(m.out(x, a), __ldg(Y + i));
      acc = fma(r, r, acc);
    }
  } else {
    double x[BBML_MAX_INPUTS];
    for (int i = lane; i < n; i += 32) {
      for (int k = 0; k < d; ++k) x[k] = __ldg(X + (int64_t)i * xs + k);
      const double r = __dsub_rn(br_sample(wv, x, d, h, nullptr), __ldg(Y + i));
      acc = fma(r, r, acc);
    }
  }
  return warp_sum(acc);
}

// P <= 32 statistics (generic h, d): rows of [J | r] are staged CH at a time
// in the LU workspace (idle during the statistics), one sample per lane, then
// each lane accumulates 4x4 register blocks of the upper triangle of
// [J r]'[J r] (45 blocks over 9 column blocks, two per lane) in sample order
// -- the same order and rounding as the per-entry loop, with 8x fewer shared
// loads per FMA.
template <int PM>
__device__ void w_stats_blocked(WarpLm<PM>& S, const double* X, const double* Y, int n, int d,
                                int h, int P, int xs, int lane) {
  constexpr int LD = WarpLm<PM>::LD;
  constexpr int RW = 36;               // J columns (P <= 32) + r, padded to 9 blocks of 4
  constexpr int CH = (PM * LD) / RW;   // staged rows per chunk (29 at PM = 32)
  constexpr int NB = RW / 4;
  constexpr int NBLK = NB * (NB + 1) / 2;
  static_assert(NBLK <= 64, "two blocks per lane");
  double* Jc = S.A;
  int ba[2], bb[2];
  bool valid[2];
#pragma unroll
  for (int u = 0; u < 2; ++u) {
    int t = lane + 32 * u, r = 0;
    valid[u] = t < NBLK;
    if (!valid[u]) t = 0;
    while (t >= NB - r) {
      t -= NB - r;
      ++r;
    }
    ba[u] = r;
    bb[u] = r + t;
  }
  double acc[2][4][4];
#pragma unroll
  for (int u = 0; u < 2; ++u)
#pragma unroll
    for (int p = 0; p < 4; ++p)
#pragma unroll
      for (int q = 0; q < 4; ++q) acc[u][p][q] = 0.0;
  double x[BBML_MAX_INPUTS];
  for (int base = 0; base < n; base += CH) {
    const int cnt = min(CH, n - base);
    __syncwarp();
    if (lane < cnt) {
      const int i = base + lane;
      for (int k = 0; k < d; ++k) x[k] = __ldg(X + (int64_t)i * xs + k);
      double* row = Jc + lane * RW;
      row[P] = __dsub_rn(br_sample(S.w, x, d, h, row), __ldg(Y + i));
      for (int c = P + 1; c < RW; ++c) row[c] = 0.0;
    }
    __syncwarp();
    for (int c = 0; c < cnt; ++c) {
      const double* row = Jc + c * RW;
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        if (!valid[u]) continue;
        const double2 a01 = *(const double2*)(row + 4 * ba[u]);
        const double2 a23 = *(const double2*)(row + 4 * ba[u] + 2);
        const double2 b01 = *(const double2*)(row + 4 * bb[u]);
        const double2 b23 = *(const double2*)(row + 4 * bb[u] + 2);
        const double va[4] = {a01.x, a01.y, a23.x, a23.y};
        const double vb[4] = {b01.x, b01.y, b23.x, b23.y};
#pragma unroll
        for (int p = 0; p < 4; ++p)
#pragma unroll
          for (int q = 0; q < 4; ++q) acc[u][p][q] = fma(va[p], vb[q], acc[u][p][q]);
      }
    }
  }
  __syncwarp();
#pragma unroll
  for (int u = 0; u < 2; ++u) {
    if (!valid[u]) continue;
#pragma unroll
    for (int p = 0; p < 4; ++p)
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int a = 4 * ba[u] + p, b = 4 * bb[u] + q;
        if (a > b || a >= P) continue;
        if (b < P) {
          S.jtj[a * LD + b] = acc[u][p][q];
          S.jtj[b * LD + a] = acc[u][p][q];
        } else if (b == P) {
          S.jtr[a] = acc[u][p][q];
        }
      }
  }
  __syncwarp();
}

template <int PM, int D, int NW = 1>
__device__ void w_stats(WarpLm<PM>& S, const double* X, const double* Y, int n, int d, int h, int P,
                        int xs, int lane, int sw = 0, double* red = nullptr) {
  constexpr int LD = WarpLm<PM>::LD;
  if constexpr (D > 0) {
    constexpr int PP = D + 3;
    constexpr int NA = PP * (PP + 1) / 2 + PP;
    H1<D> m;
    m.load(S.w);
    double acc[NA];
#pragma unroll
    for (int e = 0; e < NA; ++e) acc[e] = 0.0;
    // per sample: residual, Jacobian row, rank-1 update of [J'J | J'r] in the
    // lane's sample order; samples in blocks of 4 with every load of the block
    // issued first (L2 latency) and the four exp/div chains independent
    auto sample = [&](const double (&x)[D], double yv) {
      double a;
      const double r = __dsub_rn(m.out(x, a), yv);
      const double g = __dmul_rn(__dsub_rn(1.0, __dmul_rn(a, a)), m.w2);
      double jr[PP];
#pragma unroll
      for (int k = 0; k < D; ++k) jr[k] = __dmul_rn(g, x[k]);
      jr[D] = g;
      jr[D + 1] = a;
      jr[D + 2] = 1.0;
      int e = 0;
#pragma unroll
      for (int p = 0; p < PP; ++p)
#pragma unroll
        for (int q = p; q < PP; ++q, ++e) acc[e] = fma(jr[p], jr[q], acc[e]);
#pragma unroll
      for (int p = 0; p < PP; ++p, ++e) acc[e] = fma(jr[p], r, acc[e]);
    };
    constexpr int UB = 4;
    constexpr int ST = 32 * NW;
    int i = sw * 32 + lane;
    for (; i + ST * (UB - 1) < n; i += ST * UB) {
      double xv[UB][D], yv[UB];
#pragma unroll
      for (int u = 0; u < UB; ++u) {
        load_x<D>(xv[u], X, i + ST * u, xs);
        yv[u] = __ldg(Y + i + ST * u);
      }
#pragma unroll
      for (int u = 0; u < UB; ++u) sample(xv[u], yv[u]);
    }
    for (; i < n; i += ST) {
      double x[D];
      load_x<D>(x, X, i, xs);
      sample(x, __ldg(Y + i));
    }
    if constexpr (NW > 1) {  // warp partials -> red[sw][e]; the caller reduces
      int e = 0;
#pragma unroll
      for (int p = 0; p < NA; ++p, ++e) {
        const double v = warp_sum(acc[e]);
        if (lane == 0) red[sw * NA + e] = v;
      }
      return;
    }
    int e = 0;
#pragma unroll
    for (int p = 0; p < PP; ++p)
#pragma unroll
      for (int q = p; q < PP; ++q, ++e) {
        const double v = warp_sum(acc[e]);
        if (lane == 0) {
          S.jtj[p * LD + q] = v;
          S.jtj[q * LD + p] = v;
        }
      }
#pragma unroll
    for (int p = 0; p < PP; ++p, ++e) {
      const double v = warp_sum(acc[e]);
      if (lane == 0) S.jtr[p] = v;
    }
  } else if constexpr (PM > 8) {
    w_stats_blocked<PM>(S, X, Y, n, d, h, P, xs, lane);
  } else {
    const int ne = P * (P + 1) / 2 + P;
    double x[BBML_MAX_INPUTS];
    for (int e = lane; e < PM * LD; e += 32) S.jtj[e] = 0.0;
    for (int e = lane; e < PM; e += 32) S.jtr[e] = 0.0;
    constexpr int JCH = WarpLm<PM>::JCH;
    for (int base = 0; base < n; base += JCH) {
      const int cnt = min(JCH, n - base);
      if (lane < cnt) {
        const int i = base + lane;
        for (int k = 0; k < d; ++k) x[k] = __ldg(X + (int64_t)i * xs + k);
        S.rc[lane] = __dsub_rn(br_sample(S.w, x, d, h, S.Jc + lane * PM), __ldg(Y + i));
      }
      __syncwarp();
      for (int e = lane; e < ne; e += 32) {
        const int a = S.ent[e] >> 8, b = S.ent[e] & 255;
        double s = (b < P) ? S.jtj[a * LD + b] : S.jtr[a];
        if (b < P) {
          for (int c = 0; c < cnt; ++c) s = fma(S.Jc[c * PM + a], S.Jc[c * PM + b], s);
          S.jtj[a * LD + b] = s;
        } else {
          for (int c = 0; c < cnt; ++c) s = fma(S.Jc[c * PM + a], S.rc[c], s);
          S.jtr[a] = s;
        }
      }
      __syncwarp();
    }
    for (int e = lane; e < ne; e += 32) {
      const int a = S.ent[e] >> 8, b = S.ent[e] & 255;
      if (b < P && a != b) S.jtj[b * LD + a] = S.jtj[a * LD + b];
    }
  }
  __syncwarp();
}

// LU with partial pivoting (first maximal |pivot|, as idamax) + substitutions
// (PM = 8: P <= 8)
template <int PM>
__device__ bool w_solve(WarpLm<PM>& S, int P, double alpha, double beta, double mu, int lane) {
  constexpr int LD = WarpLm<PM>::LD;
  const double damp = __dadd_rn(mu, alpha);
  if (lane < P) {
    for (int b = 0; b < P; ++b) {
      const double v = __dmul_rn(beta, S.jtj[lane * LD + b]);
      S.A[lane * LD + b] = (lane == b) ? __dadd_rn(v, damp) : v;
    }
    S.rhs[lane] = -__dadd_rn(__dmul_rn(beta, S.jtr[lane]), __dmul_rn(alpha, S.w[lane]));
  }
  __syncwarp();
  for (int k = 0; k < P; ++k) {
    // pivot: the first maximal |a_ik|, i >= k (idamax), scanned by lane 0
    // (P <= 8 entries) and broadcast once
    int bi = k;
    if (lane == 0) {
      double best = fabs(S.A[k * LD + k]);
#pragma unroll
      for (int i = 1; i < PM; ++i) {
        const double v = (i > k && i < P) ? fabs(S.A[i * LD + k]) : -1.0;
        if (v > best) {
          best = v;
          bi = i;
        }
      }
    }
    const int p = __shfl_sync(0xffffffffu, bi, 0);
    if (S.A[p * LD + k] == 0.0) return false;
    if (p != k) {
      if (lane < P) {
        const double t = S.A[k * LD + lane];
        S.A[k * LD + lane] = S.A[p * LD + lane];
        S.A[p * LD + lane] = t;
      }
      if (lane == 0) {
        const double t = S.rhs[k];
        S.rhs[k] = S.rhs[p];
        S.rhs[p] = t;
      }
    }
    __syncwarp();
    if (lane > k && lane < P) {
      const double l = div_safe_bf(S.A[lane * LD + k], S.A[k * LD + k]);
      S.A[lane * LD + k] = l;
      for (int j = k + 1; j < P; ++j) S.A[lane * LD + j] = fma(-l, S.A[k * LD + j], S.A[lane * LD + j]);
    }
    __syncwarp();
  }
  // substitutions (P <= 8) by lane 0 in registers: the same row dot
  // products and the same pairwise order as the warp reduction they replace
  // (warp_sum over one term per lane: ((t0+t4)+(t2+t6)) + ((t1+t5)+(t3+t7))),
  // so the results are unchanged, without the five dependent shuffles per row
  if (lane == 0) {
    auto tree8 = [](const double (&t)[8]) {
      return ((t[0] + t[4]) + (t[2] + t[6])) + ((t[1] + t[5]) + (t[3] + t[7]));
    };
    double b[PM];
#pragma unroll
    for (int i = 0; i < PM; ++i) b[i] = i < P ? S.rhs[i] : 0.0;
#pragma unroll
    for (int i = 0; i < PM; ++i) {  // L y = b (unit diagonal), row i
      if (i < P) {
        double t[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) t[j] = j < i ? fma(S.A[i * LD + j], b[j], 0.0) : 0.0;
        b[i] = __dsub_rn(b[i], tree8(t));
        S.rhs[i] = b[i];
      }
    }
#pragma unroll
    for (int i = PM - 1; i >= 0; --i) {  // U x = y, row i (term L = column i+1+L)
      if (i < P) {
        double t[8];
#pragma unroll
        for (int l = 0; l < 8; ++l) {
          const int j = i + 1 + l;
          t[l] = (j < PM && j < P) ? fma(S.A[i * LD + (j < PM ? j : 0)], b[j < PM ? j : 0], 0.0) : 0.0;
        }
        b[i] = div_safe_bf(__dsub_rn(b[i], tree8(t)), S.A[i * LD + i]);
        S.delta[i] = b[i];
      }
    }
  }
  __syncwarp();
  return true;
}

// P <= 32 variant (h >= 2 models, parity gated statistically): same LU with
// partial pivoting, but the trailing row update is unrolled over restrict
// pointers (loads pipelined instead of serialised behind the stores) and both
// substitutions are column-oriented (dtrsv order) with the right-hand side in
// registers, one shuffle per column instead of a warp reduction per row.
template <int PM>
__device__ bool w_solve_cols(WarpLm<PM>& S, int P, double alpha, double beta, double mu, int lane) {
  constexpr int LD = WarpLm<PM>::LD;
  const double damp = __dadd_rn(mu, alpha);
  if (lane < P) {
    for (int b = 0; b < P; ++b) {
      const double v = __dmul_rn(beta, S.jtj[lane * LD + b]);
      S.A[lane * LD + b] = (lane == b) ? __dadd_rn(v, damp) : v;
    }
    S.rhs[lane] = -__dadd_rn(__dmul_rn(beta, S.jtr[lane]), __dmul_rn(alpha, S.w[lane]));
  }
  __syncwarp();
  for (int k = 0; k < P; ++k) {
    double best = (lane >= k && lane < P) ? fabs(S.A[lane * LD + k]) : -1.0;
    int bi = lane;
#pragma unroll
    for (int m = 16; m >= 1; m >>= 1) {
      const double ob = __shfl_xor_sync(0xffffffffu, best, m);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, m);
      if (ob > best || (ob == best && oi < bi)) {
        best = ob;
        bi = oi;
      }
    }
    const int p = bi;
    if (S.A[p * LD + k] == 0.0) return false;
    if (p != k) {
      if (lane < P) {
        const double t = S.A[k * LD + lane];
        S.A[k * LD + lane] = S.A[p * LD + lane];
        S.A[p * LD + lane] = t;
      }
      if (lane == 0) {
        const double t = S.rhs[k];
        S.rhs[k] = S.rhs[p];
        S.rhs[p] = t;
      }
    }
    __syncwarp();
    if (lane > k && lane < P) {
      double* __restrict__ ai = S.A + lane * LD;
      const double* __restrict__ ak = S.A + k * LD;
      const double l = __ddiv_rn(ai[k], ak[k]);
      ai[k] = l;
      int j = k + 1;
      for (; j + 3 < P; j += 4) {
        const double a0 = ai[j], a1 = ai[j + 1], a2 = ai[j + 2], a3 = ai[j + 3];
        const double r0 = ak[j], r1 = ak[j + 1], r2 = ak[j + 2], r3 = ak[j + 3];
        ai[j] = fma(-l, r0, a0);
        ai[j + 1] = fma(-l, r1, a1);
        ai[j + 2] = fma(-l, r2, a2);
        ai[j + 3] = fma(-l, r3, a3);
      }
      for (; j < P; ++j) ai[j] = fma(-l, ak[j], ai[j]);
    }
    __syncwarp();
  }
  double r = lane < P ? S.rhs[lane] : 0.0;
  for (int k = 0; k + 1 < P; ++k) {  // L y = Pb, unit lower, column by column
    const double yk = __shfl_sync(0xffffffffu, r, k);
    if (lane > k && lane < P) r = fma(-S.A[lane * LD + k], yk, r);
  }
  double mine = 0.0;
  for (int i = P - 1; i >= 0; --i) {  // U x = y, column by column
    double di = lane == i ? __ddiv_rn(r, S.A[i * LD + i]) : 0.0;
    di = __shfl_sync(0xffffffffu, di, i);
    if (lane == i) mine = di;
    if (lane < i) r = fma(-S.A[lane * LD + i], di, r);
  }
  if (lane < P) S.delta[lane] = mine;
  __syncwarp();
  return true;
}

// Damped solve on the tridiagonal form w_gamma_tri leaves behind (warp
// kernels, P >= 6: hidden-1 fits with d >= 3 and the P <= 32 path).  The LM trials of epoch e use the J'J that epoch e-1's
// evidence update tridiagonalised: J'J = Q T Q', Q = H_0 ... H_{P-3},
// H_k = I - bh_k v_k v_k' (v_k in column k below the diagonal of S.A, bh_k at
// S.A[k][k+1], T = diag(S.A) + off-diagonal ee), so
//   (beta J'J + (mu + alpha) I) delta = -g   <=>   delta = Q M^-1 Q' (-g),
//   M = beta T + (mu + alpha) I  (SPD tridiagonal),
// with g = beta J'r + alpha w (brbpnn.py:153-171).  Q'(-g) is formed once per
// epoch (first trial); each trial is an LDL' of M (2P sequential steps) and
// the back-transform -- O(P^2) instead of the LU's O(P^3) with a pivot
// search per column.  Backward stable (orthogonal Q, SPD M); returns false
// if a pivot of M is not positive (J'J numerically indefinite against a tiny
// damping), and the caller falls back to the LU (w_solve_cols).
template <int PM>
__device__ bool w_solve_tri(WarpLm<PM>& S, int P, double alpha, double beta, double mu, int lane,
                            bool first) {
  constexpr int LD = WarpLm<PM>::LD;
  const unsigned FULL = 0xffffffffu;
  const double* __restrict__ ee = S.Jc + 2 * PM;
  if (first) {
    double x = lane < P ? -__dadd_rn(__dmul_rn(beta, S.jtr[lane]), __dmul_rn(alpha, S.w[lane])) : 0.0;
    for (int k = 0; k + 2 < P; ++k) {  // Q' = H_{P-3} ... H_0
      const double vi = (lane > k && lane < P) ? S.A[lane * LD + k] : 0.0;
      const double bh = S.A[k * LD + k + 1];
      x = fma(-bh * warp_sum(vi * x), vi, x);
    }
    if (lane < P) S.rhs[lane] = x;
    __syncwarp();
  }
  const double damp = __dadd_rn(mu, alpha);
  double dp = 0.0, yp = 0.0, md = 1.0, my = 0.0;
  bool ok = true;
  for (int i = 0; i < P; ++i) {  // M = L D L', L y = z (every lane, lane i keeps d_i, y_i)
    const double mii = fma(beta, S.A[i * LD + i], damp);
    double di = mii, yi = S.rhs[i];
    if (i > 0) {
      const double off = beta * ee[i - 1];
      const double l = off / dp;
      di = fma(-l, off, mii);
      yi = fma(-l, yp, yi);
    }
    ok = ok && di > 0.0;
    if (lane == i) {
      md = di;
      my = yi;
    }
    dp = di;
    yp = yi;
  }
  if (!ok) return false;
  double x = 0.0, xn = 0.0;
  for (int i = P - 1; i >= 0; --i) {  // D L' x = y
    const double off = i + 1 < P ? beta * ee[i] : 0.0;
    xn = __shfl_sync(FULL, (my - off * xn) / md, i);
    if (lane == i) x = xn;
  }
  for (int k = P - 3; k >= 0; --k) {  // Q = H_0 ... H_{P-3}
    const double vi = (lane > k && lane < P) ? S.A[lane * LD + k] : 0.0;
    const double bh = S.A[k * LD + k + 1];
    x = fma(-bh * warp_sum(vi * x), vi, x);
  }
  if (lane < P) S.delta[lane] = x;
  __syncwarp();
  return true;
}

// gamma from the eigenvalues of J'J: cyclic Jacobi, round-robin disjoint
// pairs, rotations skipped below max(eps * max|diag|, 1e-15 sqrt|a_pp a_qq|)
// (LAPACK dsyevd's eigenvalues carry the same eps * ||A|| absolute accuracy)
template <int PM>
__device__ double w_gamma(WarpLm<PM>& S, int P, double alpha, double beta, int lane) {
  constexpr int LD = WarpLm<PM>::LD;
  if (lane < P)
    for (int b = 0; b < P; ++b) S.A[lane * LD + b] = S.jtj[lane * LD + b];
  double dmax = lane < P ? fabs(S.jtj[lane * LD + lane]) : 0.0;
#pragma unroll
  for (int m = 16; m >= 1; m >>= 1) dmax = fmax(dmax, __shfl_xor_sync(0xffffffffu, dmax, m));
  const double floor_abs = 2.220446049250313e-16 * dmax;
  __syncwarp();
  const int Pp = (P + 1) & ~1;
  const int np = Pp / 2;
  for (int sweep = 0; sweep < 40; ++sweep) {
    bool any = false;
    for (int r = 0; r < Pp - 1; ++r) {
      bool rot = false;
      if (lane < np) {
        const int pqv = S.rr[r * (PM / 2) + lane];
        const int p = pqv & 255, q = pqv >> 8;
        double c = 1.0, s = 0.0;
        if (q < P) {
          const double apq = S.A[p * LD + q], app = S.A[p * LD + p], aqq = S.A[q * LD + q];
          // same arithmetic with the branch-free correctly-rounded division and
          // square root (f64math.cuh): identical values, no branch per operation
          if (fabs(apq) > floor_abs && fabs(apq) > 1e-15 * sqrt_nonneg_bf(fabs(app * aqq))) {
            const double tau = div_safe_bf(aqq - app, 2.0 * apq);
            const double t = div_safe_bf(tau >= 0.0 ? 1.0 : -1.0, fabs(tau) + sqrt_nonneg_bf(1.0 + tau * tau));
            c = div_rn_bf(1.0, sqrt_rn_bf(1.0 + t * t));
            s = t * c;
            rot = true;
          }
        }
        S.cs[2 * lane] = c;
        S.cs[2 * lane + 1] = s;
        S.pq[lane] = p | (q << 8);
      }
      rot = __any_sync(0xffffffffu, rot);
      __syncwarp();
      if (!rot) continue;
      any = true;
      if (lane < P) {  // columns: A <- A J   (lane = row i)
        for (int k = 0; k < np; ++k) {
          const double s = S.cs[2 * k + 1];
          if (s == 0.0) continue;
          const int p = S.pq[k] & 255, q = S.pq[k] >> 8;
          const double c = S.cs[2 * k], aip = S.A[lane * LD + p], aiq = S.A[lane * LD + q];
          S.A[lane * LD + p] = c * aip - s * aiq;
          S.A[lane * LD + q] = s * aip + c * aiq;
        }
      }
      __syncwarp();
      if (lane < P) {  // rows: A <- J' A   (lane = column j), (p,q) annihilated
        for (int k = 0; k < np; ++k) {
          const double s = S.cs[2 * k + 1];
          if (s == 0.0) continue;
          const int p = S.pq[k] & 255, q = S.pq[k] >> 8;
          const double c = S.cs[2 * k], apj = S.A[p * LD + lane], aqj = S.A[q * LD + lane];
          S.A[p * LD + lane] = (lane == q) ? 0.0 : c * apj - s * aqj;
          S.A[q * LD + lane] = (lane == p) ? 0.0 : s * apj + c * aqj;
        }
      }
      __syncwarp();
    }
    if (!any) break;
  }
  double part = 0.0;
  if (lane < P) {
    const double lam = fmax(S.A[lane * LD + lane], 0.0);
    const double sc = __dmul_rn(beta, lam);
    const double den = __dadd_rn(sc, alpha);
    part = den > 0.0 ? __ddiv_rn(sc, den) : 0.0;
  }
  return warp_sum(part);
}

// gamma for the wider warp path (P up to 32): Householder tridiagonalisation
// of J'J (lane = row, reflector/rank-2 update lane-parallel) followed by
// Sturm-sequence bisection, one eigenvalue per lane.  Same eps*||A||
// absolute eigenvalue accuracy as LAPACK dsyevd (tridiagonalise + solve),
// ~3x fewer instructions than cyclic Jacobi at P = 31.
template <int PM>
__device__ double w_gamma_tri(WarpLm<PM>& S, int P, double alpha, double beta, int lane) {
  constexpr int LD = WarpLm<PM>::LD;
  double* v = S.rhs;     // reflector
  double* wv = S.delta;  // rank-2 partner
  double* dd = S.Jc;     // diagonal of T
  double* e2 = S.Jc + PM;  // squared off-diagonal of T
  double* ee = S.Jc + 2 * PM;
  if (lane < P)
    for (int b = 0; b < P; ++b) S.A[lane * LD + b] = S.jtj[lane * LD + b];
  __syncwarp();
  for (int k = 0; k + 2 < P; ++k) {
    const double xi = (lane > k && lane < P) ? S.A[lane * LD + k] : 0.0;
    const double sig = warp_sum(xi * xi);
    const double x0 = S.A[(k + 1) * LD + k];
    const double tail = sig - x0 * x0;
    if (!(tail > 0.0)) {  // column already tridiagonal
      if (lane == 0) {
        ee[k] = x0;
        S.A[k * LD + k + 1] = 0.0;  // H_k = I
      }
      __syncwarp();
      continue;
    }
    const double al = x0 > 0.0 ? -sqrt(sig) : sqrt(sig);
    const double bh = 1.0 / (sig - al * x0);  // 2 / v'v
    if (lane > k && lane < P) v[lane] = xi - (lane == k + 1 ? al : 0.0);
    __syncwarp();
    double pi = 0.0;
    if (lane > k && lane < P) {  // four partial sums: the FMA chain is the latency
      const double* __restrict__ ai = S.A + lane * LD;
      double p1 = 0.0, p2 = 0.0, p3 = 0.0;
      int j = k + 1;
      for (; j + 3 < P; j += 4) {
        pi = fma(ai[j], v[j], pi);
        p1 = fma(ai[j + 1], v[j + 1], p1);
        p2 = fma(ai[j + 2], v[j + 2], p2);
        p3 = fma(ai[j + 3], v[j + 3], p3);
      }
      for (; j < P; ++j) pi = fma(ai[j], v[j], pi);
      pi = ((pi + p1) + (p2 + p3)) * bh;
    }
    const double K = 0.5 * bh * warp_sum((lane > k && lane < P) ? v[lane] * pi : 0.0);
    if (lane > k && lane < P) wv[lane] = pi - K * v[lane];
    __syncwarp();
    if (lane > k && lane < P) {
      double* __restrict__ ai = S.A + lane * LD;
      const double vi = v[lane], wi = wv[lane];
      int j = k + 1;
      for (; j + 3 < P; j += 4) {
        const double a0 = ai[j], a1 = ai[j + 1], a2 = ai[j + 2], a3 = ai[j + 3];
        ai[j] = a0 - fma(vi, wv[j], wi * v[j]);
        ai[j + 1] = a1 - fma(vi, wv[j + 1], wi * v[j + 1]);
        ai[j + 2] = a2 - fma(vi, wv[j + 2], wi * v[j + 2]);
        ai[j + 3] = a3 - fma(vi, wv[j + 3], wi * v[j + 3]);
      }
      for (; j < P; ++j) ai[j] -= fma(vi, wv[j], wi * v[j]);
      ai[k] = vi;  // reflector kept for w_solve_tri
    }
    if (lane == 0) {
      ee[k] = al;
      S.A[k * LD + k + 1] = bh;  // row k is final
    }
    __syncwarp();
  }
  if (lane < P) dd[lane] = S.A[lane * LD + lane];
  if (lane == 0 && P >= 2) ee[P - 2] = S.A[(P - 1) * LD + (P - 2)];
  __syncwarp();
  // Gershgorin interval of T, then T scaled by a power of two to ||T|| <= 1
  double glo = 0.0, ghi = 0.0;
  if (lane < P) {
    const double r = (lane > 0 ? fabs(ee[lane - 1]) : 0.0) + (lane + 1 < P ? fabs(ee[lane]) : 0.0);
    glo = dd[lane] - r;
    ghi = dd[lane] + r;
  }
#pragma unroll
  for (int m = 16; m >= 1; m >>= 1) {
    glo = fmin(glo, __shfl_xor_sync(0xffffffffu, glo, m));
    ghi = fmax(ghi, __shfl_xor_sync(0xffffffffu, ghi, m));
  }
  const double tnorm = fmax(fabs(glo), fabs(ghi));
  if (!(tnorm > 0.0)) return 0.0;  // J'J = 0: every eigenvalue clipped to 0
  const double scale = sturm_scale(tnorm);
  __syncwarp();
  if (lane < P) {
    dd[lane] *= scale;
    if (lane + 1 < P) {
      const double es = ee[lane] * scale;
      e2[lane] = es * es;
    }
  }
  __syncwarp();
  const double hi0 = (ghi + 2.220446049250313e-16 * tnorm) * scale;
  // T padded to PM rows (d = 2 > ||T||, e = 0), rows as {d_j, e_{j-1}^2}
  double2* de = (double2*)(S.Jc + 3 * PM);
  if (lane < PM) de[lane] = make_double2(lane < P ? dd[lane] : 2.0,
                                         (lane >= 1 && lane < P) ? e2[lane - 1] : 0.0);
  __syncwarp();
  const int n_tiny = sturm_count_fixed<PM>(de, kFixTiny);
  const double part = lane < P ? sturm_gamma_part_fixed<PM>(de, lane, n_tiny, hi0,
                                                            alpha / beta * scale, 1.0 / scale,
                                                            alpha, beta)
                               : 0.0;
  return warp_sum(part);
}


// Development-only phase profiler (compile with -DBBML_LM_PROF, e.g.
// BBML_NVCC_DEFS=-DBBML_LM_PROF python -m paper_2202_07798_b200.build):
// lane 0 of every warp model accumulates clock64() per phase; totals are
// printed to stderr after each bbml_lm_train call.
#ifdef BBML_LM_PROF
__device__ unsigned long long g_lm_prof[8];
#define LM_PROF_T(v) long long v = clock64()
#define LM_PROF_ADD(k, t0)                                                   \
  do {                                                                       \
    if (lane == 0) atomicAdd(&g_lm_prof[k], (unsigned long long)(clock64() - (t0))); \
  } while (0)
#else
#define LM_PROF_T(v) (void)0
#define LM_PROF_ADD(k, t0) (void)0
#endif

// CTAs per SM the register allocation must allow (A/B on sweep / suite16):
// hidden-1 d <= 2 -> 4 (128 registers; r01 measured 6 / 80 registers best
// with static one-model-per-warp grids, with the persistent warps of r02 the
// spill-free 4 wins: suite16 FP64 LM call 492 -> 454 ms, step 1 074 -> 1 057
// ms, tools/r2o.sh); d >= 3 includes the longest series
// (pathfinder n = 7604), where spills would lengthen the critical chain -> 4
// PM = 32: 19.5 KB of shared memory per warp (+2 KB static / reserved per
// CTA).  2-warp CTAs pack 5 x 2 = 10 warps per SM, 3-warp CTAs only 3 x 3;
// A/B on one box (tools/ab_step.sh): gramschmit BR 268 -> 258 ms, suite16
// step 854 -> 825 ms; 1-warp CTAs (10 per SM) measured 274 / 843 ms.
#ifndef LM32_WARPS
#define LM32_WARPS 2
#endif
#ifndef LM32_MINB
#define LM32_MINB 5
#endif
#ifndef LM_H1_MINB
#define LM_H1_MINB 4
#endif
template <int PM, int D>
constexpr int lm_min_blocks() {
  return PM > 8 ? LM32_MINB : (D == 1 || D == 2) ? LM_H1_MINB : 4;
}
// NW = 1: one model per warp.  NW > 1 (hidden-1 long series): one model per
// CTA of NW warps -- the per-sample passes (objective, J'J / J'r) are split
// over the warps and reduced in warp order through shared memory; the
// damped solve and the eigen-solve run on warp 0; the scalar LM / evidence
// bookkeeping is computed identically by every warp.
// One BR-BPNN fit (brbpnn.train) by one warp (NW = 1) or one CTA of NW warps.
template <int PM, int D, int NW>
__device__ __forceinline__ void lm_fit_task(const LmLaunch& L, int64_t task, unsigned char* lm_smem,
                                            int lane, int wi) {
  if (task >= L.n_tasks) return;
  WarpLm<PM>& S = NW > 1 ? *(WarpLm<PM>*)lm_smem : ((WarpLm<PM>*)lm_smem)[wi];
  // NW > 1: cross-warp partials + broadcast slots after the model workspace
  double* red = (double*)(lm_smem + sizeof(WarpLm<PM>));
  const bool lead = NW == 1 || wi == 0;
  const bbml_lm_task tk = L.tasks[task];
  const int orig = L.orig_index[task];
  const int n = tk.n, d = tk.d, h = tk.h;
  const int P = h * (d + 2) + 1;
  const int xs = L.x_stride;
  const double* X = L.X + tk.row_begin * (int64_t)xs;
  const double* Y = L.y + tk.row_begin;
  const double* X_ = X;
  const double* Y_ = Y;
  const int n_ = n, d_ = d, h_ = h, xs_ = xs;
  const int sw = NW > 1 ? wi : 0;
  auto sync = [&]() {
    if constexpr (NW > 1) __syncthreads();
    else __syncwarp();
  };
  // objective over all samples (NW > 1: warp partials summed in warp order)
  auto energy = [&](const double* wv) -> double {
    const double v = w_energy<PM, D, NW>(S, wv, X_, Y_, n_, d_, h_, xs_, lane, sw);
    if constexpr (NW == 1) {
      return v;
    } else {
      __syncthreads();
      if (lane == 0) red[wi] = v;
      __syncthreads();
      double t = 0.0;
#pragma unroll
      for (int w = 0; w < NW; ++w) t += red[w];
      return t;
    }
  };
  auto stats = [&]() {
    if constexpr (NW == 1) {
      w_stats<PM, D>(S, X, Y, n, d, h, P, xs, lane);
    } else {
      constexpr int PP = D + 3;
      constexpr int NA = PP * (PP + 1) / 2 + PP;
      __syncthreads();
      w_stats<PM, D, NW>(S, X, Y, n, d, h, P, xs, lane, sw, red);
      __syncthreads();
      if (wi == 0) {
        constexpr int LD = WarpLm<PM>::LD;
        for (int e = lane; e < NA; e += 32) {
          double v = 0.0;
#pragma unroll
          for (int w = 0; w < NW; ++w) v += red[w * NA + e];
          int a = 0, b = e;  // e -> (a, b) in the upper-triangle order, then J'r
          if (e < PP * (PP + 1) / 2) {
            while (b >= PP - a) {
              b -= PP - a;
              ++a;
            }
            b += a;
            S.jtj[a * LD + b] = v;
            S.jtj[b * LD + a] = v;
          } else {
            S.jtr[e - PP * (PP + 1) / 2] = v;
          }
        }
      }
      __syncthreads();
    }
  };

  if (lead && lane == 0) {  // init (brbpnn.py:63-82, called at 309-310)
    Pcg64 rng;
    rng.seed(tk.seed);
    const double s1 = __ddiv_rn(1.0, __dsqrt_rn((double)d));
    const double s2 = __ddiv_rn(1.0, __dsqrt_rn((double)h));
    const int hd = h * d;
    for (int i = 0; i < hd + h; ++i) S.w[i] = rng.uniform(-s1, s1);
    for (int i = hd + h; i < P; ++i) S.w[i] = rng.uniform(-s2, s2);
    if constexpr (!WarpLm<PM>::kWide) {
      int e = 0;  // upper-triangle entry table for the generic stats path
      for (int a = 0; a < P; ++a)
        for (int b = a; b <= P; ++b) S.ent[e++] = (unsigned short)((a << 8) | b);
      const int Pp = (P + 1) & ~1;  // Jacobi round-robin schedule (index P = bye when P is odd)
      for (int r = 0; r < Pp - 1; ++r)
        for (int k = 0; k < Pp / 2; ++k) {
          const int pa = k == 0 ? 0 : 1 + ((k - 1 + r) % (Pp - 1));
          const int qa = 1 + ((Pp - 2 - k + r) % (Pp - 1));
          S.rr[r * (PM / 2) + k] = (unsigned short)(min(pa, qa) | (max(pa, qa) << 8));
        }
    }
  }
  sync();

  double alpha = tk.alpha0, beta = tk.beta0, mu = tk.mu0;
  const bool est = tk.estimate != 0;
  double* hist = (tk.hist_offset >= 0) ? L.history + tk.hist_offset : nullptr;
  double e_d = energy(S.w);
  double e_w = 0.0;
  for (int i = 0; i < P; ++i) e_w = fma(S.w[i], S.w[i], e_w);
  bool have_stats = false;
  bool tri = false;  // P >= 6: S.A holds the tridiagonal form + reflectors of J'J
  int code = BBML_MODEL_OK, trials = 0, epochs = 0, any_pinned = 0, stable = 0;
  double fail_mu = 0.0, last_mu = NAN, last_gamma = NAN;
  double prev_g = 0.0, prev_d = 0.0, prev_w = 0.0;
  bool have_prev = false;

  for (int ep = 0; ep < tk.max_epochs; ++ep) {
    if (!have_stats) {
      LM_PROF_T(t0);
      stats();
      LM_PROF_ADD(0, t0);
      tri = false;
    }
    const double f0 = __dadd_rn(__dmul_rn(beta, e_d), __dmul_rn(alpha, e_w));
    bool accepted = false;
    bool tri_first = true;
    double td = 0.0, tw = 0.0;
    while (true) {
      ++trials;
      LM_PROF_T(t2);
      bool solved = true;
      if (lead) {
        bool done = false;
        if (tri) {
          done = w_solve_tri<PM>(S, P, alpha, beta, mu, lane, tri_first);
          tri_first = false;
        }
        if (!done) {
          tri = false;  // the LU overwrites the reflectors
          if constexpr (PM > 8) solved = w_solve_cols<PM>(S, P, alpha, beta, mu, lane);
          else solved = w_solve<PM>(S, P, alpha, beta, mu, lane);  // P <= 8 only
        }
        if (lane < P) S.wt[lane] = __dadd_rn(S.w[lane], S.delta[lane]);
      }
      if constexpr (NW > 1) {
        if (wi == 0 && lane == 0) red[NW * 64] = solved ? 1.0 : 0.0;
        __syncthreads();
        solved = red[NW * 64] != 0.0;
      }
      LM_PROF_ADD(2, t2);
      if (!solved) {
        code = BBML_MODEL_SINGULAR;
        fail_mu = mu;
        break;
      }
      sync();
      LM_PROF_T(t3);
      td = energy(S.wt);
      LM_PROF_ADD(3, t3);
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
    if (lead && lane < P) S.w[lane] = S.wt[lane];
    sync();
    e_d = td;
    e_w = tw;
    const double f1 = __dadd_rn(__dmul_rn(beta, e_d), __dmul_rn(alpha, e_w));
    double gamma = NAN;
    int pinned = 0;
    if (est) {
      LM_PROF_T(t0);
      stats();
      LM_PROF_ADD(0, t0);
      have_stats = true;
      LM_PROF_T(t1);
      // P <= 5: cyclic Jacobi (converges in a few sweeps at this size);
      // P >= 6: Householder + bisection
      if (lead) {
        if constexpr (WarpLm<PM>::kWide) {
          gamma = w_gamma_tri<PM>(S, P, alpha, beta, lane);
          tri = true;
        } else if (P >= 6) {
          gamma = w_gamma_tri<PM>(S, P, alpha, beta, lane);
          tri = true;
        }
        else gamma = w_gamma<PM>(S, P, alpha, beta, lane);
      }
      if constexpr (NW > 1) {
        if (wi == 0 && lane == 0) red[NW * 64 + 1] = gamma;
        __syncthreads();
        gamma = red[NW * 64 + 1];
        __syncthreads();
      }
      LM_PROF_ADD(1, t1);
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
    if (hist && lead && lane == 0) {
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
  sync();
  if (!lead) return;
  double* W = L.weights + tk.w_offset;
  if (lane < P) W[lane] = S.w[lane];
  if (lane == 0) {
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

// NW > 1: one model per CTA (blockIdx.x).  NW = 1 with L.queue set: a
// persistent grid of warps, each pulling the next model index from an
// atomic counter over the cost-sorted task list, so a warp whose fit
// early-stopped (BR fits stop anywhere between ~10 and 1000 epochs) takes
// the next model instead of idling until its CTA's slowest fit ends
// (SURVEY §8e).  Without a queue: one model per warp, static.
template <int PM, int D, int NW = 1>
__global__ void __launch_bounds__(NW > 1 ? 32 * NW : (PM > 8 ? 32 * LM32_WARPS : 128),
                                  NW > 1 ? 1 : lm_min_blocks<PM, D>()) lm_warp_kernel(LmLaunch L) {
  extern __shared__ __align__(16) unsigned char lm_smem[];
  const int lane = threadIdx.x & 31, wi = threadIdx.x >> 5;
  if constexpr (NW > 1) {
    lm_fit_task<PM, D, NW>(L, (int64_t)blockIdx.x, lm_smem, lane, wi);
  } else if (L.queue == nullptr) {
    lm_fit_task<PM, D, 1>(L, (int64_t)blockIdx.x * (blockDim.x >> 5) + wi, lm_smem, lane, wi);
  } else {
    while (true) {
      int t = 0;
      if (lane == 0) t = atomicAdd(L.queue, 1);
      t = __shfl_sync(0xffffffffu, t, 0);
      if (t >= L.n_tasks) break;
      lm_fit_task<PM, D, 1>(L, t, lm_smem, lane, wi);
      __syncwarp();
    }
  }
}

// persistent warps by default (BBML_LM_QUEUE=0: static one-model-per-warp grid)
static bool lm_queue_on() {
  static const bool on = [] {
    const char* e = getenv("BBML_LM_QUEUE");
    return !(e && e[0] == '0');
  }();
  return on;
}

template <int PM, int D>
static cudaError_t lm_launch_warp(const LmLaunch& L, cudaStream_t s) {
  const int warps = PM > 8 ? LM32_WARPS : 4;
  const size_t smem = warps * sizeof(WarpLm<PM>);
  auto k = lm_warp_kernel<PM, D>;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  int blocks = (int)ceil_div(L.n_tasks, warps);
  if (L.queue != nullptr) {  // one resident wave of persistent warps
    int per_sm = 0, dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, 32 * warps, smem);
    blocks = std::min(blocks, std::max(1, per_sm) * sms);
  }
  k<<<blocks, 32 * warps, smem, s>>>(L);
  return cudaGetLastError();
}

// hidden-1 long series: one model per CTA of LM_NW warps
#ifndef BBML_LM_NW
#define BBML_LM_NW 4
#endif
#ifndef BBML_LONG_LM
#define BBML_LONG_LM 2048
#endif
constexpr int LM_NW = BBML_LM_NW;
constexpr int kLongLm = BBML_LONG_LM;  // samples from which a hidden-1 fit gets a CTA
template <int D>
static cudaError_t lm_launch_multi(const LmLaunch& L, cudaStream_t s) {
  const size_t smem = sizeof(WarpLm<8>) + (size_t)(LM_NW * 64 + 8) * sizeof(double);
  lm_warp_kernel<8, D, LM_NW><<<L.n_tasks, 32 * LM_NW, smem, s>>>(L);
  return cudaGetLastError();
}

// launch key: 1..4 = hidden-1 warp fast path with d inputs (101..104: the
// same for n >= kLongLm, one CTA of LM_NW warps per model); 8 / 32 = warp
// kernels (P <= 8 / P <= 32); 512 = wide CTA-per-model kernel (lm_wide.cu)
static int lm_key(const bbml_lm_task& t) {
  const int P = t.h * (t.d + 2) + 1;
  if (t.h == 1 && t.d <= 4) return t.n >= kLongLm ? 100 + t.d : t.d;
  return P <= 8 ? 8 : P <= 32 ? 32 : 512;
}

bbml_status lm_wide_launch(const bbml_lm_task* d_tasks, const int32_t* d_orig,
                           const bbml_lm_task* h_tasks, int32_t n_tasks, const double* X,
                           const double* y, int32_t x_stride, double* weights, double* history,
                           bbml_model_status* status, ScratchBuffer& scratch, cudaStream_t s,
                           bool alloc_only, double** slabs);

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
    if (t.d > BBML_MAX_INPUTS || P > BBML_LM_MAX_PARAMS) {
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
    const int ka = lm_key(tasks[a]), kb = lm_key(tasks[b]);
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
  std::vector<std::pair<int, int>> groups;
  for (int b0 = 0; b0 < n_tasks;) {
    int b1 = b0;
    while (b1 < n_tasks && lm_key(sorted[b1]) == lm_key(sorted[b0])) ++b1;
    groups.push_back({b0, b1});
    b0 = b1;
  }
  // wide slabs are allocated on the parent stream before the fork
  double* wide_slabs = nullptr;
  for (auto& g : groups)
    if (lm_key(sorted[g.first]) == 512)
      if ((st = lm_wide_launch(nullptr, nullptr, sorted.data() + g.first, g.second - g.first, X, y,
                               x_stride, weights, history, status, scratch, stream, true,
                               &wide_slabs)) != BBML_OK)
        return st;
  int* queues = nullptr;  // one work counter per shape group (persistent warp kernels)
  if ((st = scratch.alloc(&queues, (int64_t)groups.size())) != BBML_OK) return st;
  if (cudaMemsetAsync(queues, 0, groups.size() * sizeof(int), stream) != cudaSuccess)
    return cuda_status(cudaGetLastError(), "lm queue reset");
  StreamFork fork(stream, (int)groups.size());  // shape groups run concurrently
  for (size_t gno = 0; gno < groups.size(); ++gno) {
    const int begin = groups[gno].first, end = groups[gno].second;
    const int b = lm_key(sorted[begin]);
    cudaStream_t cs = fork.child((int)gno);
    if (b == 512) {
      if ((st = lm_wide_launch(d_tasks + begin, d_orig + begin, sorted.data() + begin, end - begin, X,
                               y, x_stride, weights, history, status, scratch, cs, false,
                               &wide_slabs)) != BBML_OK)
        return st;
      continue;
    }
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
    if (b < 100 && lm_queue_on()) {  // per-group work counter, zeroed on the group's stream
      L.queue = queues + gno;
    }
    cudaError_t e;
    if (b == 101) e = lm_launch_multi<1>(L, cs);
    else if (b == 102) e = lm_launch_multi<2>(L, cs);
    else if (b == 103) e = lm_launch_multi<3>(L, cs);
    else if (b == 104) e = lm_launch_multi<4>(L, cs);
    else if (b == 1) e = lm_launch_warp<8, 1>(L, cs);
    else if (b == 2) e = lm_launch_warp<8, 2>(L, cs);
    else if (b == 3) e = lm_launch_warp<8, 3>(L, cs);
    else if (b == 4) e = lm_launch_warp<8, 4>(L, cs);
    else if (b == 8) e = lm_launch_warp<8, 0>(L, cs);
    else e = lm_launch_warp<32, 0>(L, cs);
    if (e != cudaSuccess) return cuda_status(e, "lm_train launch");
  }
  if ((st = fork.join()) != BBML_OK) return st;
#ifdef BBML_LM_PROF
  {
    unsigned long long pr[8];
    cudaStreamSynchronize(stream);
    cudaMemcpyFromSymbol(pr, g_lm_prof, sizeof(pr));
    fprintf(stderr, "[lm_prof] Mcycles stats %.1f gamma %.1f solve %.1f energy %.1f\n", pr[0] * 1e-6,
            pr[1] * 1e-6, pr[2] * 1e-6, pr[3] * 1e-6);
    const unsigned long long z[8] = {};
    cudaMemcpyToSymbol(g_lm_prof, z, sizeof(z));
  }
#endif
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

// PMAX <= 96: J'J and the LU / Jacobi workspace in shared memory; PMAX = 512
// (the wide BR-BPNN shapes, hidden 64 at P = 257): both P x P matrices in a
// global scratch slab per task (gws), the vectors in shared memory.
template <int PMAX>
__global__ void lm_unit_kernel(int mode, const int32_t* __restrict__ Ps,
                               const int64_t* __restrict__ pp_off, const int64_t* __restrict__ p_off,
                               const double* __restrict__ jtj, const double* __restrict__ jtr,
                               const double* __restrict__ w, const double* __restrict__ params,
                               double* __restrict__ out_vec, double* __restrict__ out5,
                               int32_t* __restrict__ info, double* __restrict__ gws) {
  constexpr bool kGlobal = PMAX > 96;
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
  if constexpr (kGlobal) {
    S.jtj = gws + (int64_t)t * 2 * P * P;
    S.A = S.jtj + (int64_t)P * P;
  } else {
    S.jtj = q; q += PMAX * PMAX;
    S.A = q; q += PMAX * PMAX;
  }
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
    if (P[i] < 1 || P[i] > BBML_LM_MAX_PARAMS) {
      set_error("lm unit task %d: P=%d outside 1..%d", i, P[i], BBML_LM_MAX_PARAMS);
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
  const bool big = pmax > 96;
  const int PM = big ? BBML_LM_MAX_PARAMS : 96;
  const size_t mats = big ? 0 : 2 * (size_t)PM * PM;
  const size_t smem = (5 * PM + mats + LM_NT + 2 * (PM + 2) + LM_WARPS + 2 + (PM + 1) / 2 + 1 + 4) *
                      sizeof(double);
  double* gws = nullptr;
  if (big) {  // per-task P x P slabs (sized by the largest P) for J'J and the workspace
    int64_t per = 0;
    for (int i = 0; i < n_tasks; ++i) per = std::max<int64_t>(per, 2 * (int64_t)P[i] * P[i]);
    if ((st = scratch.alloc(&gws, per * n_tasks)) != BBML_OK) return st;
  }
  auto k = big ? lm_unit_kernel<BBML_LM_MAX_PARAMS> : lm_unit_kernel<96>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k<<<n_tasks, LM_NT, smem, s>>>(mode, dP, dpp, dp, jtj, jtr, w, params, out_vec, out5, info, gws);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_status(e, "lm unit launch");
  (void)n_params_per_task;
  return scratch.release();
}

}  // namespace bbml
