// FP64 op latency microbenchmark (one warp, dependent chains), development tool
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_2202_07798_b200/csrc/f64math.cuh"
using namespace bbml;
__device__ double sink;
template <int OP>
__global__ void k(double x0, int iters, long long* cyc) {
  double x = x0 + threadIdx.x * 1e-9;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    if (OP == 0) x = tanh(x) + 0.3;
    if (OP == 1) x = exp(-x) + 0.2;
    if (OP == 2) x = log(x + 1.5);
    if (OP == 3) x = log1p(x) + 0.1;
    if (OP == 4) x = __ddiv_rn(1.7, x + 1.0);
    if (OP == 5) x = __dsqrt_rn(x + 1.0);
    if (OP == 6) x = __dadd_rn(__dmul_rn(x, 0.999), 1e-3);
    if (OP == 7) x = fma(x, 0.999, 1e-3);
    if (OP == 8) x = __shfl_xor_sync(0xffffffffu, x, 1) * 0.5 + 0.5;
    if (OP == 9) x = pow(0.999, x * 1000.0 + 5);
    if (OP == 10) { float f = (float)x; f = tanhf(f) + 0.3f; x = f; }
    if (OP == 11) x = tanh_bf(x) + 0.3;
    if (OP == 12) x = div_rn_bf(1.7, x + 1.0);
    if (OP == 13) x = sqrt_rn_bf(x + 1.0);
    if (OP == 16) x = exp_neg_bf(-x) + 0.2;
    if (OP == 17) x = log_bf(x + 1.5);
    if (OP == 18) x = log1p_bf(x) + 0.1;
    if (OP == 14) { double a0 = tanh(x), a1 = tanh(x + 0.1), a2 = tanh(x + 0.2), a3 = tanh(x + 0.3), a4 = tanh(x + 0.4); x = (a0 + a1 + a2 + a3 + a4) * 0.2; }
    if (OP == 15) { double a0 = tanh_bf(x), a1 = tanh_bf(x + 0.1), a2 = tanh_bf(x + 0.2), a3 = tanh_bf(x + 0.3), a4 = tanh_bf(x + 0.4); x = (a0 + a1 + a2 + a3 + a4) * 0.2; }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) *cyc = t1 - t0;
  if (x == 12345.0) sink = x;
}
int main() {
  long long* d; cudaMalloc(&d, 8); long long h;
  const char* names[] = {"tanh", "exp", "log", "log1p", "div_rn", "sqrt_rn", "mul+add", "dfma", "shfl+fma", "pow", "tanhf(cvt)", "tanh_bf", "div_rn_bf", "sqrt_rn_bf", "5x tanh", "5x tanh_bf", "exp_neg_bf", "log_bf", "log1p_bf"};
  int iters = 1000;
#define RUN(OP) k<OP><<<1, 32>>>(0.5, iters, d); cudaDeviceSynchronize(); k<OP><<<1, 32>>>(0.5, iters, d); cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost); printf("%-12s %8.1f cycles/iter\n", names[OP], (double)h / iters);
  RUN(0) RUN(1) RUN(2) RUN(3) RUN(4) RUN(5) RUN(6) RUN(7) RUN(8) RUN(9) RUN(10) RUN(11) RUN(12) RUN(13) RUN(14) RUN(15) RUN(16) RUN(17) RUN(18)
  return 0;
}
