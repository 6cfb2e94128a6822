// lm_wide.cu — BR-BPNN Levenberg-Marquardt trainer for wide networks
// (33 <= P <= 512, e.g. hidden 64 at d = 2 -> P = 257; BASELINE config 5).
//
// Same semantics as lm_train.cu (brbpnn.py:286-346, see there for line refs),
// one model per CTA of 256 threads.  The P x P matrices (J'J and the
// factorisation / tridiagonalisation workspace) live in a per-model global
// scratch slab (L2-resident for ~100 models); vectors, the staged [J r] rows
// and the Cholesky panel live in shared memory.  No Jacobian is materialised.
//   J'J, J'r   : [J r] rows generated 32 at a time into shared memory, 4x4
//                register blocks of the upper triangle (wide_stats_chunked)
//   solve      : blocked Cholesky (32-column panels, panel in shared memory,
//                register-blocked trailing update) + blocked substitutions;
//                LU with partial pivoting (dgetf2 order) if a pivot is not
//                positive (wide_chol / wide_solve)
//   gamma      : Householder tridiagonalisation + Sturm bisection (one or two
//                eigenvalues per thread), like LAPACK dsytrd + dstebz
#include <algorithm>
#include <cstdio>
#include <vector>

#include "common.cuh"
#include "sturm.cuh"
#include "launch.h"
#include "pcg64.cuh"

namespace bbml {

#ifdef BBML_LM_PROF
__device__ unsigned long long g_wide_prof[16];
#define WP_T(v) long long v = clock64()
#define WP_ADD(k, t0)                                                                     \
  do {                                                                                    \
    if (threadIdx.x == 0) atomicAdd(&g_wide_prof[k], (unsigned long long)(clock64() - (t0))); \
  } while (0)
#else
#define WP_T(v) (void)0
#define WP_ADD(k, t0) (void)0
#endif

constexpr int WNT = 512;
constexpr int WWARPS = WNT / 32;
constexpr int WPMAX = 512;

struct WideLaunch {
  const bbml_lm_task* tasks;
  const int32_t* orig_index;
  int32_t n_tasks;
  int32_t x_stride;
  const double* X;
  const double* y;
  double* weights;
  double* history;
  bbml_model_status* status;
  double* scratch;        // one slab per resident CTA
  int64_t slab_doubles;   // doubles per slab
  int32_t ld;             // leading dimension of the P x P matrices (>= P, multiple of 4)
  int* queue;             // next-task counter of the persistent grid
  int32_t dyn_doubles;    // dynamic shared memory per CTA (doubles)
};

struct WideSmem {
  double w[WPMAX], wt[WPMAX], delta[WPMAX], jtr[WPMAX], rhs[WPMAX];
  double v[WPMAX], pv[WPMAX], dd[WPMAX], ee[WPMAX], e2[WPMAX];
  double red[WWARPS * 2];
  int ired[WWARPS];
  int piv;
};

__device__ __forceinline__ double bsum(double x, WideSmem& S) {
#pragma unroll
  for (int m = 16; m >= 1; m >>= 1) x += __shfl_xor_sync(0xffffffffu, x, m);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) S.red[threadIdx.x >> 5] = x;
  __syncthreads();
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < WWARPS; ++i) s += S.red[i];
  return s;
}

__device__ __forceinline__ double bmax(double x, WideSmem& S) {
#pragma unroll
  for (int m = 16; m >= 1; m >>= 1) x = fmax(x, __shfl_xor_sync(0xffffffffu, x, m));
  __syncthreads();
  if ((threadIdx.x & 31) == 0) S.red[threadIdx.x >> 5] = x;
  __syncthreads();
  double s = S.red[0];
#pragma unroll
  for (int i = 1; i < WWARPS; ++i) s = fmax(s, S.red[i]);
  return s;
}

// forward of one sample (brbpnn.forward) and optionally its Jacobian row
__device__ __forceinline__ double wide_sample(const double* __restrict__ w, const double* x, int d,
                                              int h, double* jrow) {
  const int hd = h * d;
  double out = 0.0;
  for (int j = 0; j < h; ++j) {
    double pre = 0.0;
    for (int k = 0; k < d; ++k) pre = fma(x[k], w[j * d + k], pre);
    const double a = tansig(__dadd_rn(pre, w[hd + j]));
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

__device__ double wide_energy(const double* wv, const double* X, const double* Y, int n, int d, int h,
                              int xs, WideSmem& S) {
  double acc = 0.0, x[BBML_MAX_INPUTS];
  for (int i = threadIdx.x; i < n; i += WNT) {
    for (int k = 0; k < d; ++k) x[k] = __ldg(X + (int64_t)i * xs + k);
    const double r = __dsub_rn(wide_sample(wv, x, d, h, nullptr), __ldg(Y + i));
    acc = fma(r, r, acc);
  }
  return bsum(acc, S);
}

// [J r] rows are generated 32 at a time into shared memory (no Jacobian in
// HBM): one (row, hidden unit) item per thread, then the residual per row in
// the reference's summation order.
constexpr int WCH = 32;  // staged rows per chunk

// staged row width: P J columns + r, padded to 8-column tiles and to 8 (mod
// 16) doubles so that the DMMA fragment loads (4 rows x 8 columns per warp)
// take the minimum two shared-memory wavefronts
__device__ __host__ __forceinline__ int wide_rw(int P) {
  const int w = (P + 1 + 7) & ~7;
  return (w & 15) ? w : w + 8;
}

// J'J and J'r on the FP64 tensor cores (BASELINE cfg 5): the same staged
// [J r] chunks, the upper triangle of [J r]'[J r] in 8x8 tiles, one
// mma.sync.m8n8k4.f64 per tile and 4 staged rows (A fragment = tile row block,
// B fragment = tile column block of the same 4 rows).  Each warp owns a run
// of up to WCAP consecutive tiles of the row-major upper-triangle list (so
// the A fragment is reused along the run); accumulators stay in registers
// across all chunks.
constexpr int WCAP = 18;

// Packed J'J: the strict upper triangle lives in the upper half of the P x P
// slab (row a < column b) and the diagonal in ld doubles after it; the lower
// half and the diagonal of the slab hold the Cholesky / tridiagonalisation
// workspace.  One ld x ld array per model instead of two: 140 cfg-5 models
// take 74 MB of L2 instead of 148 MB (B200 L2: 126 MB).
__device__ __forceinline__ double jtj_at(const double* jtj, int ld, int a, int b) {
  return a == b ? jtj[(int64_t)ld * ld + a]
                : jtj[a < b ? (int64_t)a * ld + b : (int64_t)b * ld + a];
}

__device__ __forceinline__ void dmma884(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

__device__ void wide_stats_dmma(double* jtj, int ld, const double* X, const double* Y, int n, int d,
                                int h, int P, int xs, WideSmem& S, double* Jc) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int rw = wide_rw(P);
  const int nt = (P + 1 + 7) / 8;
  const int npair = nt * (nt + 1) / 2;
  const int hd = h * d;
  for (int p0 = 0; p0 < npair; p0 += WWARPS * WCAP) {
    const int first = p0 + warp * WCAP;
    const int cnt = max(0, min(WCAP, npair - first));
    int ta0 = 0, tb0 = 0;
    {
      int t = cnt > 0 ? first : 0;
      while (t >= nt - ta0) {
        t -= nt - ta0;
        ++ta0;
      }
      tb0 = ta0 + t;
    }
    double acc[WCAP][2];
#pragma unroll
    for (int q = 0; q < WCAP; ++q) acc[q][0] = acc[q][1] = 0.0;
    for (int base = 0; base < n; base += WCH) {
      const int rows = min(WCH, n - base);
      const int rows4 = (rows + 3) & ~3;
      __syncthreads();
      for (int it = threadIdx.x; it < rows * h; it += WNT) {  // (row, hidden unit) items
        const int c = it / h, j = it - c * h;
        const double* x = X + (int64_t)(base + c) * xs;
        double pre = 0.0;
        for (int k = 0; k < d; ++k) pre = fma(__ldg(x + k), S.w[j * d + k], pre);
        const double a = tansig(__dadd_rn(pre, S.w[hd + j]));
        const double da = __dmul_rn(__dsub_rn(1.0, __dmul_rn(a, a)), S.w[hd + h + j]);
        double* row = Jc + c * rw;
        for (int k = 0; k < d; ++k) row[j * d + k] = __dmul_rn(da, __ldg(x + k));
        row[hd + j] = da;
        row[hd + h + j] = a;
      }
      for (int e = rows * rw + threadIdx.x; e < rows4 * rw; e += WNT) Jc[e] = 0.0;  // pad rows
      __syncthreads();
      for (int c = threadIdx.x; c < rows; c += WNT) {  // residual, wide_sample's order
        double* row = Jc + c * rw;
        double out = 0.0;
        for (int j = 0; j < h; ++j) out = fma(row[hd + h + j], S.w[hd + h + j], out);
        row[hd + 2 * h] = 1.0;
        row[P] = __dsub_rn(__dadd_rn(out, S.w[hd + 2 * h]), __ldg(Y + base + c));
        for (int q = P + 1; q < rw; ++q) row[q] = 0.0;
      }
      __syncthreads();
      if (cnt > 0) {
        for (int ks = 0; ks < rows4; ks += 4) {
          const double* fr = Jc + (ks + (lane & 3)) * rw + (lane >> 2);
          int ta = ta0, tb = tb0;
          double fa = fr[8 * ta];
#pragma unroll
          for (int q = 0; q < WCAP; ++q) {
            if (q < cnt) {
              dmma884(acc[q], fa, fr[8 * tb]);
              if (++tb == nt) {
                ++ta;
                tb = ta;
                if (ta < nt) fa = fr[8 * ta];
              }
            }
          }
        }
      }
    }
    int ta = ta0, tb = tb0;
#pragma unroll
    for (int q = 0; q < WCAP; ++q) {
      if (q < cnt) {
        const int a = 8 * ta + (lane >> 2);
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          const int b = 8 * tb + 2 * (lane & 3) + i;
          if (a <= b && a < P) {
            if (b < P) {  // packed: strict upper triangle in place, diagonal after the matrix
              if (a < b) jtj[(int64_t)a * ld + b] = acc[q][i];
              else jtj[(int64_t)ld * ld + a] = acc[q][i];
            } else if (b == P) {
              S.jtr[a] = acc[q][i];
            }
          }
        }
        if (++tb == nt) {
          ++ta;
          tb = ta;
        }
      }
    }
  }
  __syncthreads();
}

// Damped system by blocked Cholesky (A = beta J'J + (mu+alpha) I is SPD; the
// north star's "in-shared-memory Cholesky"): 32-column panels -- the diagonal
// block factored by one warp in shared memory, the panel below solved one row
// per thread and kept transposed in shared memory, the trailing lower
// triangle updated with 4x4 register blocks from the panel (one L2 pass per
// panel).  Blocked forward / backward substitution.  Returns false when a
// pivot is not positive (numerically indefinite); the caller then runs the
// LU of the reference (wide_solve).
constexpr int WNB = 32;

__device__ bool wide_chol(double* A, const double* jtj, int ld, int P, double alpha, double beta,
                          double mu, WideSmem& S, double* dyn) {
  const double damp = __dadd_rn(mu, alpha);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int rw = wide_rw(P);
  double* PT = dyn;               // panel, transposed: PT[t * rw + i]
  double* D = dyn + WNB * rw;     // diagonal block, 32 x 33
  WP_T(tc0);
  for (int a = warp; a < P; a += WWARPS)
    for (int b = lane; b <= a; b += 32) {
      const double v = __dmul_rn(beta, jtj_at(jtj, ld, a, b));
      A[(int64_t)a * ld + b] = (a == b) ? __dadd_rn(v, damp) : v;
    }
  for (int a = threadIdx.x; a < P; a += WNT)
    S.rhs[a] = -__dadd_rn(__dmul_rn(beta, S.jtr[a]), __dmul_rn(alpha, S.w[a]));
  __syncthreads();
  WP_ADD(8, tc0);
  for (int kb = 0; kb < P; kb += WNB) {
    const int nb = min(WNB, P - kb), r0 = kb + nb, m = P - r0;
    WP_T(tc1);
    for (int e = threadIdx.x; e < nb * nb; e += WNT) {
      const int i = e / nb, j = e - i * nb;
      D[i * 33 + j] = j <= i ? A[(int64_t)(kb + i) * ld + kb + j] : 0.0;
    }
    __syncthreads();
    if (warp == 0) {  // unblocked right-looking Cholesky of the diagonal block
      bool bad = false;
      for (int k = 0; k < nb; ++k) {
        const double dkk = D[k * 33 + k];
        if (!(dkk > 0.0)) {
          bad = true;
          break;
        }
        const double sk = sqrt(dkk);
        __syncwarp();
        if (lane == k) D[k * 33 + k] = sk;
        if (lane > k && lane < nb) D[lane * 33 + k] = D[lane * 33 + k] / sk;
        __syncwarp();
        if (lane > k && lane < nb) {
          const double lk = D[lane * 33 + k];
          for (int j = k + 1; j <= lane; ++j) D[lane * 33 + j] = fma(-lk, D[j * 33 + k], D[lane * 33 + j]);
        }
        __syncwarp();
      }
      if (lane == 0) S.piv = bad ? 1 : 0;
    }
    __syncthreads();
    WP_ADD(9, tc1);
    WP_T(tc2);
    if (S.piv) return false;
    for (int e = threadIdx.x; e < nb * nb; e += WNT) {
      const int i = e / nb, j = e - i * nb;
      if (j <= i) A[(int64_t)(kb + i) * ld + kb + j] = D[i * 33 + j];
    }
    // panel rows below: x = a * L11^-T, one row per thread
    for (int i = threadIdx.x; i < m; i += WNT) {
      const double* ai = A + (int64_t)(r0 + i) * ld + kb;
      double xv[WNB];
#pragma unroll
      for (int j = 0; j < WNB; ++j) xv[j] = j < nb ? ai[j] : 0.0;
#pragma unroll
      for (int j = 0; j < WNB; ++j) {
        if (j < nb) {
          double sacc = xv[j];
#pragma unroll
          for (int t = 0; t < j; ++t) sacc = fma(-xv[t], D[j * 33 + t], sacc);
          xv[j] = sacc / D[j * 33 + j];
        }
      }
      double* ao = A + (int64_t)(r0 + i) * ld + kb;
#pragma unroll
      for (int j = 0; j < WNB; ++j)
        if (j < nb) {
          ao[j] = xv[j];
          PT[j * rw + i] = xv[j];
        }
    }
    __syncthreads();
    WP_ADD(10, tc2);
    WP_T(tc3);
    // trailing update of the lower triangle: A22 -= X X'
    const int mb = (m + 3) >> 2;
    const int nt = mb * (mb + 1) / 2;
    for (int t = threadIdx.x; t < nt; t += WNT) {
      int ti = 0, rem = t;  // lower triangle, row-major: (ti >= tj)
      while (rem > ti) {
        rem -= ti + 1;
        ++ti;
      }
      const int tj = rem;
      double acc[4][4];
#pragma unroll
      for (int p = 0; p < 4; ++p)
#pragma unroll
        for (int q = 0; q < 4; ++q) acc[p][q] = 0.0;
      for (int k = 0; k < nb; ++k) {
        const double* pk = PT + k * rw;
        double va[4], vb[4];
#pragma unroll
        for (int p = 0; p < 4; ++p) {
          va[p] = 4 * ti + p < m ? pk[4 * ti + p] : 0.0;
          vb[p] = 4 * tj + p < m ? pk[4 * tj + p] : 0.0;
        }
#pragma unroll
        for (int p = 0; p < 4; ++p)
#pragma unroll
          for (int q = 0; q < 4; ++q) acc[p][q] = fma(va[p], vb[q], acc[p][q]);
      }
#pragma unroll
      for (int p = 0; p < 4; ++p)
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int i = 4 * ti + p, j = 4 * tj + q;
          if (i < m && j <= i) {
            double* a = A + (int64_t)(r0 + i) * ld + r0 + j;
            *a = *a - acc[p][q];
          }
        }
    }
    __syncthreads();
    WP_ADD(11, tc3);
  }
  WP_T(tc4);
  auto load_diag = [&](int kb, int nb) {  // factored diagonal block -> D (shared)
    for (int e = threadIdx.x; e < nb * nb; e += WNT) {
      const int i = e / nb, j = e - i * nb;
      D[i * 33 + j] = j <= i ? A[(int64_t)(kb + i) * ld + kb + j] : 0.0;
    }
  };
  // forward: L y = b
  for (int kb = 0; kb < P; kb += WNB) {
    const int nb = min(WNB, P - kb), r0 = kb + nb;
    load_diag(kb, nb);
    __syncthreads();
    if (warp == 0) {
      double b = lane < nb ? S.rhs[kb + lane] : 0.0;
      for (int k = 0; k < nb; ++k) {
        double yk = lane == k ? b / D[k * 33 + k] : 0.0;
        yk = __shfl_sync(0xffffffffu, yk, k);
        if (lane == k) b = yk;
        if (lane > k && lane < nb) b = fma(-D[lane * 33 + k], yk, b);
      }
      if (lane < nb) S.rhs[kb + lane] = b;
    }
    __syncthreads();
    for (int i = r0 + threadIdx.x; i < P; i += WNT) {
      const double* li = A + (int64_t)i * ld + kb;
      double sacc = S.rhs[i];
      for (int t = 0; t < nb; ++t) sacc = fma(-li[t], S.rhs[kb + t], sacc);
      S.rhs[i] = sacc;
    }
    __syncthreads();
  }
  // backward: L' x = y
  const int nblk = (P + WNB - 1) / WNB;
  for (int bi = nblk - 1; bi >= 0; --bi) {
    const int kb = bi * WNB, nb = min(WNB, P - kb), r0 = kb + nb;
    {  // y_block -= L(r0:, block)' x(r0:): column c = lane, rows split over warps
      double part = 0.0;
      if (lane < nb)
        for (int i = r0 + warp; i < P; i += WWARPS) part = fma(A[(int64_t)i * ld + kb + lane], S.delta[i], part);
      S.v[warp * 32 + lane] = part;
    }
    load_diag(kb, nb);
    __syncthreads();
    if (warp == 0) {
      double b = 0.0;
      if (lane < nb) {
        b = S.rhs[kb + lane];
        double tot = 0.0;
        for (int w = 0; w < WWARPS; ++w) tot += S.v[w * 32 + lane];
        b -= tot;
      }
      for (int k = nb - 1; k >= 0; --k) {
        double xk = lane == k ? b / D[k * 33 + k] : 0.0;
        xk = __shfl_sync(0xffffffffu, xk, k);
        if (lane == k) b = xk;
        if (lane < k) b = fma(-D[k * 33 + lane], xk, b);
      }
      if (lane < nb) S.delta[kb + lane] = b;
    }
    __syncthreads();
  }
  WP_ADD(12, tc4);
  return true;
}

// LU with partial pivoting on A = beta J'J + (mu+alpha) I; false on a zero pivot
__device__ bool wide_solve(double* A, const double* jtj, int ld, int P, double alpha, double beta,
                           double mu, WideSmem& S) {
  const double damp = __dadd_rn(mu, alpha);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  (void)warp;
  (void)lane;
  // A and the packed J'J share storage: each (a <= b) pair is read once and
  // both (a, b) and (b, a) written by the same thread (the LU consumes the
  // upper triangle: the caller recomputes J'J before its next use)
  for (int e = threadIdx.x; e < P * P; e += WNT) {
    const int a = e / P, b = e - a * P;
    if (a > b) continue;
    const double v = __dmul_rn(beta, jtj_at(jtj, ld, a, b));
    A[(int64_t)a * ld + b] = (a == b) ? __dadd_rn(v, damp) : v;
    A[(int64_t)b * ld + a] = v;
  }
  for (int a = threadIdx.x; a < P; a += WNT)
    S.rhs[a] = -__dadd_rn(__dmul_rn(beta, S.jtr[a]), __dmul_rn(alpha, S.w[a]));
  __syncthreads();
  for (int k = 0; k < P; ++k) {
    double best = -1.0;
    int bi = k;
    for (int i = k + threadIdx.x; i < P; i += WNT) {
      const double v = fabs(A[(int64_t)i * ld + k]);
      if (v > best) {
        best = v;
        bi = i;
      }
    }
#pragma unroll
    for (int m = 16; m >= 1; m >>= 1) {
      const double ob = __shfl_xor_sync(0xffffffffu, best, m);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, m);
      if (ob > best || (ob == best && oi < bi)) {
        best = ob;
        bi = oi;
      }
    }
    if ((threadIdx.x & 31) == 0) {
      S.red[threadIdx.x >> 5] = best;
      S.ired[threadIdx.x >> 5] = bi;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      double b = S.red[0];
      int p = S.ired[0];
      for (int i = 1; i < WWARPS; ++i)
        if (S.red[i] > b || (S.red[i] == b && S.ired[i] < p)) {
          b = S.red[i];
          p = S.ired[i];
        }
      S.piv = p;
    }
    __syncthreads();
    const int p = S.piv;
    if (A[(int64_t)p * ld + k] == 0.0) return false;
    if (p != k) {
      for (int j = threadIdx.x; j < P; j += WNT) {
        const double t = A[(int64_t)k * ld + j];
        A[(int64_t)k * ld + j] = A[(int64_t)p * ld + j];
        A[(int64_t)p * ld + j] = t;
      }
      if (threadIdx.x == 0) {
        const double t = S.rhs[k];
        S.rhs[k] = S.rhs[p];
        S.rhs[p] = t;
      }
      __syncthreads();
    }
    const double pk = A[(int64_t)k * ld + k];
    const int m = P - k - 1;
    for (int i = threadIdx.x; i < m; i += WNT) {
      double* ai = A + (int64_t)(k + 1 + i) * ld;
      ai[k] = __ddiv_rn(ai[k], pk);
    }
    __syncthreads();
    // rank-1 update of the trailing block: warp = row, lanes = columns; four
    // independent L2 loads in flight per lane (the update is L2-latency bound)
    const double* __restrict__ rk = A + (int64_t)k * ld;
    for (int i = k + 1 + warp; i < P; i += WWARPS) {
      double* __restrict__ ai = A + (int64_t)i * ld;
      const double l = ai[k];
      int j = k + 1 + lane;
      for (; j + 96 < P; j += 128) {
        const double a0 = ai[j], a1 = ai[j + 32], a2 = ai[j + 64], a3 = ai[j + 96];
        const double r0 = rk[j], r1 = rk[j + 32], r2 = rk[j + 64], r3 = rk[j + 96];
        ai[j] = fma(-l, r0, a0);
        ai[j + 32] = fma(-l, r1, a1);
        ai[j + 64] = fma(-l, r2, a2);
        ai[j + 96] = fma(-l, r3, a3);
      }
      for (; j < P; j += 32) ai[j] = fma(-l, rk[j], ai[j]);
    }
    __syncthreads();
  }
  for (int i = 0; i < P; ++i) {  // L y = Pb (unit lower)
    double s = 0.0;
    for (int j = threadIdx.x; j < i; j += WNT) s = fma(A[(int64_t)i * ld + j], S.rhs[j], s);
    s = bsum(s, S);
    if (threadIdx.x == 0) S.rhs[i] = __dsub_rn(S.rhs[i], s);
    __syncthreads();
  }
  for (int i = P - 1; i >= 0; --i) {  // U x = y
    double s = 0.0;
    for (int j = i + 1 + threadIdx.x; j < P; j += WNT) s = fma(A[(int64_t)i * ld + j], S.delta[j], s);
    s = bsum(s, S);
    if (threadIdx.x == 0) S.delta[i] = __ddiv_rn(__dsub_rn(S.rhs[i], s), A[(int64_t)i * ld + i]);
    __syncthreads();
  }
  return true;
}

// gamma = sum beta*l/(beta*l+alpha) over the eigenvalues of J'J (clipped at 0)
// Householder tridiagonalisation (dsytrd, lower) of the symmetric J'J, one
// pass over the trailing lower triangle per step: the rank-2 update of step
// k-1 (A -= v w' + w v') is applied in the same sweep that forms p = A v of
// step k (row dot products by warp reductions, the transposed half by
// per-lane column partials reduced across warps), so each element is read
// and written once per step instead of read twice and written once, and only
// the lower triangle is touched.  Leaves diag / off-diag in S.dd / S.ee.
// Where the trailing triangle lives: the slab's lower triangle in global
// memory (row i at A + i*ld) while it is larger than the shared-memory
// budget, then (from step ks on) packed in shared memory, row i >= ks holding
// columns ks..i at T + tri(i - ks).  A step reads every trailing element once,
// so the global phase is bound by the L2 round trip per row and the
// shared-memory phase by issue; at P = 257 the triangle fits after ~50 steps.
struct TriGlobal {
  double* A;
  int ld;
  __device__ __forceinline__ double* row(int i) const { return A + (int64_t)i * ld; }
};
struct TriShared {
  double* T;
  int ks;
  __device__ __forceinline__ double* row(int i) const {
    const int m = i - ks;
    return T + (m * (m + 1) / 2 - ks);
  }
};

__device__ __forceinline__ int tri_count(int m) { return m * (m + 1) / 2; }

// step k of the reduction (column k brought up to date and reflected, then
// the fused sweep over rows/cols > k); WC column partials per lane (32 WC >= P)
template <int WC, class Rows>
__device__ __forceinline__ void tri_step(int k, int P, bool& pend, const Rows& R, WideSmem& S,
                                         double* colp) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* vp = S.v;    // pending reflector (step k-1)
  double* wp = S.pv;   // pending rank-2 partner
  double* vn = S.e2;   // reflector of step k (e2 is free until the Sturm stage)
  double* rowp = S.wt; // row dot products (wt is free during the evidence update)
  double part = 0.0;
  for (int i = k + threadIdx.x; i < P; i += WNT) {
    double* a = R.row(i) + k;
    double x = *a;
    if (pend) {
      x -= fma(vp[i], wp[k], wp[i] * vp[k]);
      *a = x;
    }
    if (i > k) part = fma(x, x, part);
  }
  const double sig = bsum(part, S);
  const double x0 = R.row(k + 1)[k];
  const double akk = R.row(k)[k];
  const bool refl = sig - x0 * x0 > 0.0;
  const double al = x0 > 0.0 ? -sqrt(sig) : sqrt(sig);
  const double bh = refl ? 1.0 / (sig - al * x0) : 0.0;
  for (int i = k + 1 + threadIdx.x; i < P; i += WNT)
    vn[i] = refl ? R.row(i)[k] - (i == k + 1 ? al : 0.0) : 0.0;
  if (threadIdx.x == 0) {
    S.dd[k] = akk;
    S.ee[k] = refl ? al : x0;
  }
  __syncthreads();
  double cacc[WC];
#pragma unroll
  for (int t = 0; t < WC; ++t) cacc[t] = 0.0;
  for (int i = k + 1 + warp; i < P; i += WWARPS) {
    double* ai = R.row(i);
    const double vpi = pend ? vp[i] : 0.0, wpi = pend ? wp[i] : 0.0, vni = vn[i];
    double racc = 0.0, av[WC];
#pragma unroll
    for (int t = 0; t < WC; ++t) {  // all loads of the row segment in flight first
      const int j = k + 1 + lane + 32 * t;
      av[t] = j <= i ? ai[j] : 0.0;
    }
#pragma unroll
    for (int t = 0; t < WC; ++t) {
      const int j = k + 1 + lane + 32 * t;
      if (j <= i) {
        double a = av[t];
        if (pend) {
          a -= fma(vpi, wp[j], wpi * vp[j]);
          ai[j] = a;
        }
        racc = fma(a, vn[j], racc);
        if (j < i) cacc[t] = fma(a, vni, cacc[t]);
      }
    }
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) racc += __shfl_xor_sync(0xffffffffu, racc, o);
    if (lane == 0) rowp[i] = racc;
  }
#pragma unroll
  for (int t = 0; t < WC; ++t) {
    const int j = k + 1 + lane + 32 * t;
    if (j < P) colp[warp * P + j] = cacc[t];
  }
  __syncthreads();
  double kp = 0.0;
  for (int i = k + 1 + threadIdx.x; i < P; i += WNT) {
    double pi = rowp[i];
#pragma unroll
    for (int w = 0; w < WWARPS; ++w) pi += colp[w * P + i];
    pi *= bh;
    rowp[i] = pi;
    kp = fma(vn[i], pi, kp);
  }
  const double K = 0.5 * bh * bsum(kp, S);
  for (int i = k + 1 + threadIdx.x; i < P; i += WNT) {
    wp[i] = rowp[i] - K * vn[i];
    vp[i] = vn[i];
  }
  if (threadIdx.x == 0) {  // entries <= k of the new pending vectors are unused
    vp[k] = 0.0;
    wp[k] = 0.0;
  }
  pend = refl;
  __syncthreads();
}

// Householder reduction of J'J to tridiagonal form (the eigenvalue problem of
// brbpnn.py:221-236), one block-wide step per column.  The whole CTA makes one
// pass over the trailing lower triangle per step: the rank-2 update of step
// k-1 (A -= v w' + w v') is applied in the same sweep that forms p = A v of
// step k (row dot products by warp reductions, the transposed half by
// per-lane column partials reduced across warps), so each element is read
// and written once per step instead of read twice and written once, and only
// the lower triangle is touched.  dyn holds the WWARPS x P column partials
// and, after them, the shared-memory copy of the trailing triangle
// (dyn_doubles in all).  Leaves diag / off-diag in S.dd / S.ee.
template <int WC>
__device__ void wide_tridiag(double* A, const double* jtj, int ld, int P, WideSmem& S, double* dyn,
                             int dyn_doubles) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* colp = dyn;
  double* T = dyn + ((WWARPS * P + 1) & ~1);
  const int cap = dyn_doubles - ((WWARPS * P + 1) & ~1);
  int ks = 0;
  while (ks + 2 < P && tri_count(P - ks) > cap) ++ks;
  const TriGlobal G{A, ld};
  const TriShared SH{T, ks};
  if (ks == 0) {
    for (int a = warp; a < P; a += WWARPS)
      for (int b = lane; b <= a; b += 32) SH.row(a)[b] = jtj_at(jtj, ld, a, b);
  } else {
    for (int a = warp; a < P; a += WWARPS)
      for (int b = lane; b <= a; b += 32) G.row(a)[b] = jtj_at(jtj, ld, a, b);
  }
  bool pend = false;
  __syncthreads();
  int k = 0;
  WP_T(tg);
  for (; k < ks && k + 2 < P; ++k) tri_step<WC>(k, P, pend, G, S, colp);
  WP_ADD(5, tg);
  if (ks > 0 && ks + 2 < P) {  // trailing rows/cols >= ks into shared memory
    for (int a = ks + warp; a < P; a += WWARPS)
      for (int b = ks + lane; b <= a; b += 32) SH.row(a)[b] = G.row(a)[b];
    __syncthreads();
  }
  const bool sh = ks + 2 < P || ks == 0;
  for (; k + 2 < P; ++k) tri_step<WC>(k, P, pend, SH, S, colp);
  // last 2x2 block
  if (threadIdx.x < 3) {
    const int i = threadIdx.x == 1 ? P - 1 : P - 2 + (threadIdx.x > 0);
    const int j = threadIdx.x == 1 ? P - 2 : P - 2 + (threadIdx.x > 1);
    double x = sh ? SH.row(i)[j] : G.row(i)[j];
    if (pend) x -= fma(S.v[i], S.pv[j], S.pv[i] * S.v[j]);
    if (threadIdx.x == 0) S.dd[P - 2] = x;
    else if (threadIdx.x == 1) S.ee[P - 2] = x;
    else S.dd[P - 1] = x;
  }
  __syncthreads();
}

__device__ double wide_gamma(double* A, const double* jtj, int ld, int P, double alpha, double beta,
                             WideSmem& S, double* dyn, int dyn_doubles) {
  if (P <= 9 * 32) wide_tridiag<9>(A, jtj, ld, P, S, dyn, dyn_doubles);
  else wide_tridiag<WPMAX / 32>(A, jtj, ld, P, S, dyn, dyn_doubles);
  WP_T(tb);
  double glo = 1e308, ghi = -1e308;
  for (int i = threadIdx.x; i < P; i += WNT) {
    const double r = (i > 0 ? fabs(S.ee[i - 1]) : 0.0) + (i + 1 < P ? fabs(S.ee[i]) : 0.0);
    glo = fmin(glo, S.dd[i] - r);
    ghi = fmax(ghi, S.dd[i] + r);
  }
  glo = -bmax(-glo, S);
  ghi = bmax(ghi, S);
  const double tnorm = fmax(fabs(glo), fabs(ghi));
  if (!(tnorm > 0.0)) return 0.0;  // J'J = 0: every eigenvalue clipped to 0
  // T scaled by a power of two to ||T|| <= 1 for the division-free Sturm count
  const double scale = sturm_scale(tnorm);
  for (int i = threadIdx.x; i < P; i += WNT) {
    S.dd[i] *= scale;
    if (i + 1 < P) {
      const double es = S.ee[i] * scale;
      S.e2[i] = es * es;
    }
  }
  __syncthreads();
  const double hi0 = (ghi + 2.220446049250313e-16 * tnorm) * scale;
  // rows {d_j, e_{j-1}^2} padded to a multiple of 4 (d = 2 > ||T||, e = 0)
  // in the dynamic buffer (free after the reduction)
  const int n4 = (P + 3) & ~3;
  double2* de = reinterpret_cast<double2*>(dyn);
  for (int i = threadIdx.x; i < n4; i += WNT)
    de[i] = make_double2(i < P ? S.dd[i] : 2.0, (i >= 1 && i < P) ? S.e2[i - 1] : 0.0);
  __syncthreads();
  const int n_tiny = sturm_count_rt(de, kFixTiny, n4);
  const double r = alpha / beta * scale;
  double part = 0.0;
  for (int idx = threadIdx.x; idx < P; idx += WNT)
    part += sturm_gamma_part_rt(de, n4, idx, n_tiny, hi0, r, 1.0 / scale, alpha, beta);
  const double g = bsum(part, S);
  WP_ADD(4, tb);
  return g;
}

// One wide BR-BPNN fit (brbpnn.train) by the whole CTA; `slab` = this CTA's
// P x P workspace (J'J + factorisation), reused by every fit the CTA runs.
__device__ __forceinline__ void lm_wide_fit(const WideLaunch& L, int task, double* slab, WideSmem& S,
                                         double* wdyn) {
  const bbml_lm_task tk = L.tasks[task];
  const int orig = L.orig_index[task];
  const int n = tk.n, d = tk.d, h = tk.h;
  const int P = h * (d + 2) + 1;
  const int ld = L.ld, xs = L.x_stride;
  const double* X = L.X + tk.row_begin * (int64_t)xs;
  const double* Y = L.y + tk.row_begin;
  double* jtj = slab;  // packed J'J (upper triangle + diagonal vector)
  double* A = slab;    // workspace: lower triangle + diagonal of the same array
  bool jtj_ok = false; // the LU fallback consumes the packed J'J

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
  double e_d = wide_energy(S.w, X, Y, n, d, h, xs, S);
  double e_w = 0.0;
  for (int i = 0; i < P; ++i) e_w = fma(S.w[i], S.w[i], e_w);
  bool have_stats = false;
  int code = BBML_MODEL_OK, trials = 0, epochs = 0, any_pinned = 0, stable = 0;
  double fail_mu = 0.0, last_mu = NAN, last_gamma = NAN, prev_g = 0.0, prev_d = 0.0, prev_w = 0.0;
  bool have_prev = false;

  for (int ep = 0; ep < tk.max_epochs; ++ep) {
    if (!have_stats || !jtj_ok) {
      WP_T(t0);
      wide_stats_dmma(jtj, ld, X, Y, n, d, h, P, xs, S, wdyn);
      WP_ADD(0, t0);
#ifdef BBML_LM_PROF
      if (threadIdx.x == 0) atomicAdd(&g_wide_prof[6], 1ull);
#endif
      jtj_ok = true;
    }
    const double f0 = __dadd_rn(__dmul_rn(beta, e_d), __dmul_rn(alpha, e_w));
    bool accepted = false;
    double td = 0.0, tw = 0.0;
    while (true) {
      ++trials;
      WP_T(t2);
      if (!jtj_ok) {  // a previous trial's LU consumed it: same statistics at the same w
        wide_stats_dmma(jtj, ld, X, Y, n, d, h, P, xs, S, wdyn);
        jtj_ok = true;
      }
      bool solved = wide_chol(A, jtj, ld, P, alpha, beta, mu, S, wdyn);
      if (!solved) {  // indefinite: LU (dgesv order)
        solved = wide_solve(A, jtj, ld, P, alpha, beta, mu, S);
        jtj_ok = false;
      }
      WP_ADD(2, t2);
      if (!solved) {
        code = BBML_MODEL_SINGULAR;
        fail_mu = mu;
        break;
      }
      for (int i = threadIdx.x; i < P; i += WNT) S.wt[i] = __dadd_rn(S.w[i], S.delta[i]);
      __syncthreads();
      WP_T(t3);
      td = wide_energy(S.wt, X, Y, n, d, h, xs, S);
      WP_ADD(3, t3);
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
    for (int i = threadIdx.x; i < P; i += WNT) S.w[i] = S.wt[i];
    __syncthreads();
    e_d = td;
    e_w = tw;
    const double f1 = __dadd_rn(__dmul_rn(beta, e_d), __dmul_rn(alpha, e_w));
    double gamma = NAN;
    int pinned = 0;
    if (est) {
      WP_T(t0);
      wide_stats_dmma(jtj, ld, X, Y, n, d, h, P, xs, S, wdyn);
      WP_ADD(0, t0);
#ifdef BBML_LM_PROF
      if (threadIdx.x == 0) atomicAdd(&g_wide_prof[6], 1ull);
#endif
      have_stats = true;
      jtj_ok = true;
      WP_T(t1);
      gamma = wide_gamma(A, jtj, ld, P, alpha, beta, S, wdyn, L.dyn_doubles);
      WP_ADD(1, t1);
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
  for (int i = threadIdx.x; i < P; i += WNT) W[i] = S.w[i];
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

// Persistent grid (one wave of resident CTAs): each CTA pulls the next fit
// from an atomic counter over the cost-sorted task list and reuses its own
// slab, so workspace memory is (resident CTAs x slab), not (fits x slab):
// 160k hidden-64 fits need 148 slabs (~160 MB), not 173 GB, and the fits
// that early-stop hand their SM to the next one.
__global__ void __launch_bounds__(WNT) lm_wide_kernel(WideLaunch L) {
  __shared__ WideSmem S;
  __shared__ int next;
  extern __shared__ __align__(16) double wdyn[];  // [J r] chunk / Cholesky panel + block
  double* slab = L.scratch + (int64_t)blockIdx.x * L.slab_doubles;
  while (true) {
    if (threadIdx.x == 0) next = atomicAdd(L.queue, 1);
    __syncthreads();
    const int task = next;
    __syncthreads();
    if (task >= L.n_tasks) break;
    lm_wide_fit(L, task, slab, S, wdyn);
    __syncthreads();
  }
}

// One fit per CTA (a single resident wave: n_tasks <= resident CTAs); the
// loop form above costs ~7% on cfg 5's 140 fits (different register schedule)
__global__ void __launch_bounds__(WNT) lm_wide_kernel_once(WideLaunch L) {
  __shared__ WideSmem S;
  extern __shared__ __align__(16) double wdyn[];
  if ((int)blockIdx.x < L.n_tasks)
    lm_wide_fit(L, blockIdx.x, L.scratch + (int64_t)blockIdx.x * L.slab_doubles, S, wdyn);
}

// Launch all wide tasks (P > 32) of one lm_train call on `s`; tasks/orig are
// device arrays (already sorted); scratch slabs are stream-ordered.
bbml_status lm_wide_launch(const bbml_lm_task* d_tasks, const int32_t* d_orig,
                           const bbml_lm_task* h_tasks, int32_t n_tasks, const double* X,
                           const double* y, int32_t x_stride, double* weights, double* history,
                           bbml_model_status* status, ScratchBuffer& scratch, cudaStream_t s,
                           bool alloc_only, double** slabs) {
  if (n_tasks == 0) return BBML_OK;
  int pmax = 0, nmax = 0;
  for (int i = 0; i < n_tasks; ++i) {
    pmax = std::max(pmax, h_tasks[i].h * (h_tasks[i].d + 2) + 1);
    nmax = std::max(nmax, h_tasks[i].n);
  }
  const int ld = (pmax + 3) & ~3;
  const int64_t slab = (int64_t)ld * ld + ld;  // packed J'J + workspace, one array
  const int rw = wide_rw(pmax);
  // dynamic shared memory: the [J r] chunk / Cholesky panel, or during the
  // tridiagonalisation the column partials + the trailing triangle; the
  // latter takes everything the opt-in limit leaves (one CTA per SM anyway:
  // 512 threads x 128 registers)
  int dev = 0, optin = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  cudaFuncAttributes fa{}, fb{};
  cudaFuncGetAttributes(&fa, lm_wide_kernel);
  cudaFuncGetAttributes(&fb, lm_wide_kernel_once);
  const size_t stat = std::max(fa.sharedSizeBytes, fb.sharedSizeBytes);
  const size_t need = (size_t)(WNB * rw + 32 * 33) * sizeof(double);
  const size_t dyn = std::max(need, ((size_t)optin > stat ? (size_t)optin - stat : 0) & ~(size_t)15);
  (void)nmax;
  static_assert(WCH == WNB, "chunk rows and panel width share the dynamic buffer");
  cudaError_t ea = cudaFuncSetAttribute(lm_wide_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)dyn);
  if (ea == cudaSuccess)
    ea = cudaFuncSetAttribute(lm_wide_kernel_once, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
  if (ea != cudaSuccess) return cuda_status(ea, "lm_wide smem");
  int sms = 0, per_sm = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, lm_wide_kernel, WNT, dyn);
  const int grid = std::min(n_tasks, std::max(1, per_sm) * sms);
  // slabs for the resident CTAs, then one double holding the work counter
  if (alloc_only) {
    bbml_status st = scratch.alloc(slabs, slab * grid + 1);
    if (st != BBML_OK) return st;
    if (cudaMemsetAsync(*slabs + slab * grid, 0, sizeof(double), s) != cudaSuccess)
      return cuda_status(cudaGetLastError(), "lm_wide queue reset");
    return BBML_OK;
  }
  double* d_scratch = *slabs;
  WideLaunch L{};
  L.tasks = d_tasks;
  L.orig_index = d_orig;
  L.n_tasks = n_tasks;
  L.x_stride = x_stride;
  L.X = X;
  L.y = y;
  L.weights = weights;
  L.history = history;
  L.status = status;
  L.scratch = d_scratch;
  L.slab_doubles = slab;
  L.ld = ld;
  L.queue = (int*)(d_scratch + slab * grid);
  L.dyn_doubles = (int32_t)(dyn / sizeof(double));
  if (grid == n_tasks) lm_wide_kernel_once<<<grid, WNT, dyn, s>>>(L);
  else lm_wide_kernel<<<grid, WNT, dyn, s>>>(L);
  cudaError_t e = cudaGetLastError();
#ifdef BBML_LM_PROF
  {
    unsigned long long pr[16];
    cudaStreamSynchronize(s);
    cudaMemcpyFromSymbol(pr, g_wide_prof, sizeof(pr));
    fprintf(stderr, "[wide_prof] stats calls %llu; chol Mcycles fill %.1f diag %.1f panel %.1f trailing %.1f subst %.1f\n", pr[6],
            pr[8] * 1e-6, pr[9] * 1e-6, pr[10] * 1e-6, pr[11] * 1e-6, pr[12] * 1e-6);
    fprintf(stderr, "[wide_prof] Mcycles stats %.1f gamma %.1f (bisect %.1f, tridiag global phase %.1f) solve %.1f energy %.1f\n",
            pr[0] * 1e-6, pr[1] * 1e-6, pr[4] * 1e-6, pr[5] * 1e-6, pr[2] * 1e-6, pr[3] * 1e-6);
    const unsigned long long z[16] = {};
    cudaMemcpyToSymbol(g_wide_prof, z, sizeof(z));
  }
#endif
  return e == cudaSuccess ? BBML_OK : cuda_status(e, "lm_wide launch");
}

}  // namespace bbml
