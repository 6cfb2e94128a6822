// units.cu — small elementwise / contraction kernels behind the unit-level
// drop-in functions (used directly by the reference's own tests):
//   bbml_adam_step <- pnn.adam_step    (pnn.py:174-189)
//   bbml_tansig    <- brbpnn.tansig    (brbpnn.py:33-38)
//   bbml_lm_gram   <- J.T @ J, J.T @ r (brbpnn.py:166-167, 260)
#include "common.cuh"
#include "launch.h"

namespace bbml {

// one flat parameter vector split into blocks [block_begin[b], block_begin[b+1]);
// bad_block[0] = first block index with a non-finite gradient or -1.
__global__ void adam_kernel(double* __restrict__ p, const double* __restrict__ g,
                            double* __restrict__ m, double* __restrict__ v, int64_t n,
                            const int64_t* __restrict__ block_begin, int n_blocks, double bc1,
                            double bc2, double lr, double b1, double b2, double eps,
                            int32_t* __restrict__ bad_block) {
  // pass 1 (single CTA): the reference raises before touching a bad block but
  // after updating the blocks before it (dict order)
  __shared__ int first_bad;
  if (threadIdx.x == 0) first_bad = n_blocks;
  __syncthreads();
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    if (!isfinite(g[i])) {
      int b = 0;
      while (b + 1 < n_blocks && i >= block_begin[b + 1]) ++b;
      atomicMin(&first_bad, b);
    }
  }
  __syncthreads();
  const int64_t limit = first_bad < n_blocks ? block_begin[first_bad] : n;
  const double c1 = __dsub_rn(1.0, b1), c2 = __dsub_rn(1.0, b2);
  for (int64_t i = threadIdx.x; i < limit; i += blockDim.x) {
    const double gi = g[i];
    const double mi = __dadd_rn(__dmul_rn(b1, m[i]), __dmul_rn(c1, gi));
    const double vi = __dadd_rn(__dmul_rn(b2, v[i]), __dmul_rn(c2, __dmul_rn(gi, gi)));
    m[i] = mi;
    v[i] = vi;
    const double mh = __ddiv_rn(mi, bc1), vh = __ddiv_rn(vi, bc2);
    p[i] = __dsub_rn(p[i], __ddiv_rn(__dmul_rn(lr, mh), __dadd_rn(sqrt(vh), eps)));
  }
  if (threadIdx.x == 0) bad_block[0] = first_bad < n_blocks ? first_bad : -1;
}

__global__ void tansig_kernel(const double* __restrict__ x, double* __restrict__ y, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    y[i] = tansig(x[i]);
}

// one CTA per task: jtj[a][b] = sum_i J[i][a] J[i][b], jtr[a] = sum_i J[i][a] r[i]
__global__ void gram_kernel(const int32_t* __restrict__ Ps, const int32_t* __restrict__ ns,
                            const int64_t* __restrict__ j_off, const int64_t* __restrict__ r_off,
                            const int64_t* __restrict__ pp_off, const int64_t* __restrict__ p_off,
                            const double* __restrict__ J, const double* __restrict__ r,
                            double* __restrict__ jtj, double* __restrict__ jtr) {
  const int t = blockIdx.x;
  const int P = Ps[t], n = ns[t];
  const double* Jt = J + j_off[t];
  for (int e = threadIdx.x; e < P * P + P; e += blockDim.x) {
    double s = 0.0;
    if (e < P * P) {
      const int a = e / P, b = e % P;
      for (int i = 0; i < n; ++i) s = fma(Jt[(int64_t)i * P + a], Jt[(int64_t)i * P + b], s);
      jtj[pp_off[t] + e] = s;
    } else {
      const int a = e - P * P;
      for (int i = 0; i < n; ++i) s = fma(Jt[(int64_t)i * P + a], r[r_off[t] + i], s);
      jtr[p_off[t] + a] = s;
    }
  }
}

bbml_status adam_launch(double* p, const double* g, double* m, double* v, int64_t n,
                        const int64_t* block_begin_dev, int n_blocks, double bc1, double bc2,
                        double lr, double b1, double b2, double eps, int32_t* bad, cudaStream_t s) {
  adam_kernel<<<1, 256, 0, s>>>(p, g, m, v, n, block_begin_dev, n_blocks, bc1, bc2, lr, b1, b2,
                                eps, bad);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? BBML_OK : cuda_status(e, "adam launch");
}

bbml_status tansig_launch(const double* x, double* y, int64_t n, cudaStream_t s) {
  if (n <= 0) return BBML_OK;
  const int blocks = (int)std::min<int64_t>((n + 255) / 256, 4096);
  tansig_kernel<<<blocks, 256, 0, s>>>(x, y, n);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? BBML_OK : cuda_status(e, "tansig launch");
}

bbml_status gram_launch(const int32_t* P, const int32_t* n, int32_t n_tasks, const int64_t* j_off,
                        const int64_t* r_off, const int64_t* pp_off, const int64_t* p_off,
                        const double* J, const double* r, double* jtj, double* jtr,
                        cudaStream_t s) {
  if (n_tasks == 0) return BBML_OK;
  ScratchBuffer scratch(s);
  int32_t *dP, *dn;
  int64_t *dj, *dr, *dpp, *dp;
  bbml_status st;
  if ((st = scratch.alloc(&dP, n_tasks)) || (st = scratch.alloc(&dn, n_tasks)) ||
      (st = scratch.alloc(&dj, n_tasks)) || (st = scratch.alloc(&dr, n_tasks)) ||
      (st = scratch.alloc(&dpp, n_tasks)) || (st = scratch.alloc(&dp, n_tasks)))
    return st;
  if ((st = scratch.upload(dP, P, n_tasks)) || (st = scratch.upload(dn, n, n_tasks)) ||
      (st = scratch.upload(dj, j_off, n_tasks)) || (st = scratch.upload(dr, r_off, n_tasks)) ||
      (st = scratch.upload(dpp, pp_off, n_tasks)) || (st = scratch.upload(dp, p_off, n_tasks)))
    return st;
  gram_kernel<<<n_tasks, 128, 0, s>>>(dP, dn, dj, dr, dpp, dp, J, r, jtj, jtr);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_status(e, "gram launch");
  return scratch.release();
}

}  // namespace bbml

// ------------------------------------------------------------------------
// FMA-pipe peak microbenchmark (the roofline denominator for the FP32/FP64
// training kernels; MEASURED_PEAKS.json only carries HBM and bf16 GEMM).
// ------------------------------------------------------------------------
namespace bbml {

template <typename T>
__global__ void __launch_bounds__(256) fma_peak_kernel(T* out, int iters, T b, T c) {
  T a[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) a[k] = T(threadIdx.x + k) * T(1e-3);
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = fma(a[k], b, c);
  }
  T s = a[0] + a[1] + a[2] + a[3] + a[4] + a[5] + a[6] + a[7];
  if (s == T(-12345.678)) out[0] = s;  // never true; keeps the chains live
}

bbml_status fma_peak_launch(int precision, int blocks, int iters, void* out, cudaStream_t s) {
  if (precision == 32)
    fma_peak_kernel<float><<<blocks, 256, 0, s>>>((float*)out, iters, 0.999999f, 1e-6f);
  else
    fma_peak_kernel<double><<<blocks, 256, 0, s>>>((double*)out, iters, 0.999999, 1e-6);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? BBML_OK : cuda_status(e, "fma_peak launch");
}

}  // namespace bbml
