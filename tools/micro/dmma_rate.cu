// DMMA.884 (mma.sync m8n8k4 f64) vs DFMA issue rate on one SM: 16 warps, each
// with 8 independent accumulator tiles (or 16 independent FMA chains).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dmma_rate dmma_rate.cu
#include <cstdio>
__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c[0]), "+d"(c[1]) : "d"(a), "d"(b));
}
__global__ void k_dmma(double* out, int iters, double a, double b) {
  double acc[8][2] = {};
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int q = 0; q < 8; ++q) dmma(acc[q], a + q, b);
  }
  double s = 0;
  for (int q = 0; q < 8; ++q) s += acc[q][0] + acc[q][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_dfma(double* out, int iters, double a, double b) {
  double acc[16] = {};
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int q = 0; q < 16; ++q) acc[q] = fma(acc[q], a, b + q);
  }
  double s = 0;
  for (int q = 0; q < 16; ++q) s += acc[q];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, sizeof(double) * sms * 1024);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 20000;
  for (int threads : {128, 256, 512, 1024}) {
    for (int rep = 0; rep < 2; ++rep) {
      float ms;
      cudaEventRecord(e0);
      k_dmma<<<sms, threads>>>(out, iters, 1.0, 1e-9);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      const double fl_d = 2.0 * 512.0 / 2 * 8 * iters * (threads / 32) * (double)sms;  // m8n8k4: 256 FMA = 512 flop
      cudaEventRecord(e0);
      k_dfma<<<sms, threads>>>(out, iters, 1.0, 1e-9);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms2;
      cudaEventElapsedTime(&ms2, e0, e1);
      const double fl_f = 2.0 * 16 * iters * (double)threads * sms;
      if (rep) printf("threads %4d: DMMA %.1f TFLOP/s   DFMA %.1f TFLOP/s\n", threads, fl_d / ms * 1e-9, fl_f / ms2 * 1e-9);
    }
  }
  return 0;
}
