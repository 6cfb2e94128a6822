// accuracy of the branch-free FP64 helpers vs libdevice (development tool)
#include <cstdio>
#include <cstdint>
#include <cmath>
#include "../../paper_2202_07798_b200/csrc/f64math.cuh"
using namespace bbml;
__device__ unsigned long long rng(unsigned long long& s) { s = s * 6364136223846793005ULL + 1442695040888963407ULL; return s; }
__device__ double u01(unsigned long long& s) { return (rng(s) >> 11) * 0x1p-53; }
__global__ void k(unsigned long long* out) {
  unsigned long long s = 1234567ULL + 7919ULL * (blockIdx.x * blockDim.x + threadIdx.x);
  unsigned long long ndiv = 0, nsqrt = 0, tanh_ulp_max = 0, tanh1 = 0, nsqrt_tiny = 0;
  for (int i = 0; i < 4000; ++i) {
    double a = (u01(s) - 0.5) * exp2(floor(u01(s) * 120 - 60));
    double b = (u01(s) + 0.05) * exp2(floor(u01(s) * 60 - 30));
    if (div_rn_bf(a, b) != __ddiv_rn(a, b)) ++ndiv;
    double x = u01(s) * exp2(floor(u01(s) * 200 - 100));
    if (sqrt_rn_bf(x) != __dsqrt_rn(x)) ++nsqrt;
    double xt = u01(s) * 1e-310;
    const bool tiny = xt < 0x1p-968;
    double st = sqrt_rn_bf(tiny ? xt * 0x1p1000 : xt); st = tiny ? st * 0x1p-500 : st;
    if (st != __dsqrt_rn(xt)) ++nsqrt_tiny;
    double t = (u01(s) - 0.5) * exp2(floor(u01(s) * 30 - 25)) * 8;
    double r1 = tanh_bf(t), r2 = tanh(t);
    long long d = llabs((long long)__double_as_longlong(r1) - (long long)__double_as_longlong(r2));
    if ((unsigned long long)d > tanh_ulp_max) tanh_ulp_max = d;
    if (d > 1) ++tanh1;
  }
  atomicAdd(out + 0, ndiv); atomicAdd(out + 1, nsqrt); atomicMax(out + 2, tanh_ulp_max); atomicAdd(out + 3, tanh1);
  atomicAdd(out + 4, nsqrt_tiny);
  unsigned long long ul[3] = {0, 0, 0}, nbig[3] = {0, 0, 0};
  for (int i = 0; i < 4000; ++i) {
    double y = -u01(s) * exp2(floor(u01(s) * 14 - 12)) * 8;  // exp arg <= 0
    double u = u01(s) * exp2(-floor(u01(s) * 60));            // log1p arg in (0,1]
    double x = (u01(s) + 0.01) * exp2(floor(u01(s) * 120 - 60)); // log arg
    double r[3][2] = {{exp_neg_bf(y), exp(y)}, {log1p_bf(u), log1p(u)}, {log_bf(x), log(x)}};
    for (int q = 0; q < 3; ++q) {
      unsigned long long d = llabs((long long)__double_as_longlong(r[q][0]) - (long long)__double_as_longlong(r[q][1]));
      if (d > ul[q]) ul[q] = d;
      if (d > 1) ++nbig[q];
    }
  }
  for (int q = 0; q < 3; ++q) { atomicMax(out + 5 + q, ul[q]); atomicAdd(out + 8 + q, nbig[q]); }
}
int main() {
  unsigned long long* d; cudaMalloc(&d, 128); cudaMemset(d, 0, 128);
  k<<<148, 256>>>(d); unsigned long long h[11]; cudaMemcpy(h, d, 88, cudaMemcpyDeviceToHost);
  printf("samples %d: div mismatches %llu, sqrt mismatches %llu, sqrt(denormal) mismatches %llu, tanh max ulp vs libdevice %llu, tanh >1ulp %llu\n",
         148 * 256 * 4000, h[0], h[1], h[4], h[2], h[3]);
  printf("max ulp vs libdevice: exp %llu (>1: %llu), log1p %llu (>1: %llu), log %llu (>1: %llu)\n", h[5], h[8], h[6], h[9], h[7], h[10]);
  return 0;
}
