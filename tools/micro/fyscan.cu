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
      } else if (MODE == 3 || MODE == 4) {  // 8-draw groups loaded ahead
        int q = 0;
        const uint4* r4 = (const uint4*)ring;
        uint4 c0 = r4[0], c1 = r4[1];
#pragma unroll 1
        for (int g = 0; g < 8 && i > 0; ++g) {
          uint4 n0 = c0, n1 = c1;
          if (g < 7) { n0 = r4[2 * g + 2]; n1 = r4[2 * g + 3]; }
          const uint32_t d8[8] = {c0.x, c0.y, c0.z, c0.w, c1.x, c1.y, c1.z, c1.w};
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) {
            if (i > 0) {
              ++q;
              const uint32_t v = d8[kk] & (0xffffffffu >> __clz(i));
              if ((int)v <= i) {
                if (MODE == 3) { uint16_t t = perm[i]; perm[i] = perm[v]; perm[v] = t; }
                --i;
              }
            }
          }
          c0 = n0; c1 = n1;
        }
        draws += q;
      } else if (MODE == 5) {  // 8-draw groups, branch-free accept, predicated swap
        int q = 0;
        const uint4* r4 = (const uint4*)ring;
        uint4 c0 = r4[0], c1 = r4[1];
#pragma unroll 1
        for (int g = 0; g < 8 && i > 0; ++g) {
          uint4 n0 = c0, n1 = c1;
          if (g < 7) { n0 = r4[2 * g + 2]; n1 = r4[2 * g + 3]; }
          const uint32_t d8[8] = {c0.x, c0.y, c0.z, c0.w, c1.x, c1.y, c1.z, c1.w};
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) {
            const bool live = i > 0;
            q += live;
            const uint32_t v = d8[kk] & (0xffffffffu >> __clz(i | 1));
            const bool acc = live && (int)v <= i;
            const int ii = acc ? i : 0, vv = acc ? (int)v : 0;   // dummy swap of slot 0 with itself
            const uint16_t a = perm[ii], b = perm[vv];
            perm[ii] = b; perm[vv] = a;
            i -= acc;
          }
          c0 = n0; c1 = n1;
        }
        draws += q;
      } else if (MODE == 6) {  // mode 5 + incremental mask (no FLO per draw)
        int q = 0;
        uint32_t mask = 0xffffffffu >> __clz(i | 1);
        const uint4* r4 = (const uint4*)ring;
        uint4 c0 = r4[0], c1 = r4[1];
#pragma unroll 1
        for (int g = 0; g < 8 && i > 0; ++g) {
          uint4 n0 = c0, n1 = c1;
          if (g < 7) { n0 = r4[2 * g + 2]; n1 = r4[2 * g + 3]; }
          const uint32_t d8[8] = {c0.x, c0.y, c0.z, c0.w, c1.x, c1.y, c1.z, c1.w};
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) {
            const bool live = i > 0;
            q += live;
            const uint32_t v = d8[kk] & mask;
            const bool acc = live && (int)v <= i;
            const int ii = acc ? i : 0, vv = acc ? (int)v : 0;
            const uint16_t a = perm[ii], b = perm[vv];
            perm[ii] = b; perm[vv] = a;
            i -= acc;
            mask = ((uint32_t)i <= (mask >> 1)) ? (mask >> 1) : mask;
          }
          c0 = n0; c1 = n1;
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
  for (int mode = 0; mode < 7; ++mode) {
    for (int rep = 0; rep < 2; ++rep) {
      if (mode == 0) k<0><<<1, 32>>>(7604, 100000, d);
      if (mode == 1) k<1><<<1, 32>>>(7604, 100000, d);
      if (mode == 2) k<2><<<1, 32>>>(7604, 100000, d);
      if (mode == 3) k<3><<<1, 32>>>(7604, 100000, d);
      if (mode == 4) k<4><<<1, 32>>>(7604, 100000, d);
      if (mode == 5) k<5><<<1, 32>>>(7604, 100000, d);
      if (mode == 6) k<6><<<1, 32>>>(7604, 100000, d);
      cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    }
    printf("mode %d: %.1f cycles per element, %.1f per draw\n", mode, (double)h[0] / 7603, (double)h[0] / h[1]);
  }
  return 0;
}
