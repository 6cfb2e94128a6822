// Fisher-Yates accept/swap scan cost on a shared-memory uint16 permutation (development tool)
#include <cstdio>
#include <cstdint>
__device__ uint32_t sink;
template <int MODE>
__global__ void k(int n, int reps, long long* cyc) {
  __shared__ uint16_t perm[8192];
  __shared__ uint32_t ring[64];
  for (int x = threadIdx.x; x < n; x += 32) perm[x] = x;
  uint64_t s = 0x9E3779B97F4A7C15ull * (threadIdx.x + 1);
  __syncwarp();
  long long t0 = clock64();
  int i = n - 1;
  long long draws = 0;
  for (int r = 0; r < reps && i > 0; ++r) {
    s = s * 6364136223846793005ull + 1442695040888963407ull;
    ring[2 * threadIdx.x] = (uint32_t)(s >> 32);
    ring[2 * threadIdx.x + 1] = (uint32_t)s;
    __syncwarp();
    if (threadIdx.x == 0) {
      if (MODE == 0) {
        int q = 0;
        while (q < 64 && i > 0) {
          const uint32_t v = ring[q++] & (0xffffffffu >> __clz(i));
          if ((int)v <= i) { uint16_t t = perm[i]; perm[i] = perm[v]; perm[v] = t; --i; }
        }
        draws += q;
      } else if (MODE == 1) {  // no swap: accept test only
        int q = 0;
        while (q < 64 && i > 0) {
          const uint32_t v = ring[q++] & (0xffffffffu >> __clz(i));
          if ((int)v <= i) --i;
        }
        draws += q;
      } else {  // swap with the top element kept in a register
        int q = 0;
        uint16_t top = perm[i];
        while (q < 64 && i > 0) {
          const uint32_t v = ring[q++] & (0xffffffffu >> __clz(i));
          if ((int)v <= i) {
            const uint16_t pv = (int)v == i ? top : perm[v];
            perm[i] = pv;
            if ((int)v != i) perm[v] = top;
            --i;
            top = perm[i];
          }
        }
        draws += q;
      }
    }
    i = __shfl_sync(0xffffffffu, i, 0);
    __syncwarp();
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = draws; sink = perm[0]; }
}
int main() {
  long long* d; cudaMalloc(&d, 16); long long h[2];
  for (int mode = 0; mode < 3; ++mode) {
    for (int rep = 0; rep < 2; ++rep) {
      if (mode == 0) k<0><<<1, 32>>>(7604, 100000, d);
      if (mode == 1) k<1><<<1, 32>>>(7604, 100000, d);
      if (mode == 2) k<2><<<1, 32>>>(7604, 100000, d);
      cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    }
    printf("mode %d: %.1f cycles per element, %.1f per draw\n", mode, (double)h[0] / 7603, (double)h[0] / h[1]);
  }
  return 0;
}
