// pnn_train.cu — fused batched Poisson-NN trainer (forward, Poisson-NLL
// backward, bias-corrected Adam) for many independent models.
//
// Reference semantics (bbcount/pnn.py):
//   init_model      87-105  U(+-1/sqrt(d)) W1 (row-major), b1; U(+-1/sqrt(h)) W2, b2
//   forward         108-118 rate = logaddexp(0, tanh(x W1' + b1) . W2 + b2) + eps
//   loss_and_grads  121-147 loss = mean(rate - y log(rate + eps)); d_rate = (1 - y/(rate+eps))/nb;
//                           d_z = d_rate exp(z - softplus); d_pre = d_z W2 (1 - a^2)
//   adam_step       174-189 finite check per block (W1,b1,W2,b2), m/v update, bias correction
//   train           211-250 per-epoch rng.permutation(n), ceil(n/B) minibatches (short tail kept),
//                           TrainingError on a non-finite batch loss, history = mean batch loss
//
// CTA layout (warp-specialised):
//   consumer warps : one model per group of G lanes.  Lane g owns hidden units
//                    j = g, g+G, ... (W1 row, b1, W2 and their Adam moments in
//                    registers); the only cross-lane traffic per sample is one
//                    butterfly all-reduce of the output pre-activation.  SC
//                    minibatch samples are processed together (independent
//                    dependency chains), and the next chunk's rows are
//                    prefetched from L2 while the current one computes.
//   producer warp  : lane i replays model i's NumPy PCG64 stream and writes
//                    epoch e+1's Fisher-Yates permutation into a shared-memory
//                    double buffer while the consumer trains on epoch e, so the
//                    sequential shuffle is off the training critical path.
//   Hand-off: per-model produced/consumed epoch counters in shared memory.
#include <cstdio>
#include <stdlib.h>

#include <algorithm>
#include <cmath>
#include <type_traits>
#include <vector>

#include "common.cuh"
#include "f64math.cuh"
#include "launch.h"
#include "pcg64.cuh"

namespace bbml {

template <typename T>
struct Arith;
template <>
struct Arith<double> {  // numpy elementwise: separately rounded mul/add/div (no FMA)
  __device__ static __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
  __device__ static __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
  __device__ static __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }
  __device__ static __forceinline__ double div(double a, double b) { return __ddiv_rn(a, b); }
};
template <>
struct Arith<float> {  // FP32 kernel: contraction allowed, fast (2 ulp) division
  __device__ static __forceinline__ float mul(float a, float b) { return a * b; }
  __device__ static __forceinline__ float add(float a, float b) { return a + b; }
  __device__ static __forceinline__ float sub(float a, float b) { return a - b; }
  __device__ static __forceinline__ float div(float a, float b) { return __fdividef(a, b); }
};

template <typename T>
__device__ __forceinline__ void adam_update(T& p, T& m, T& v, T g, T bc1, T bc2, T lr) {
  using A = Arith<T>;
  const T b1 = T(0.9), b2 = T(0.999);
  const T c1 = T(1.0 - 0.9), c2 = T(1.0 - 0.999);
  m = A::add(A::mul(b1, m), A::mul(c1, g));
  v = A::add(A::mul(b2, v), A::mul(c2, A::mul(g, g)));
  const T mh = A::div(m, bc1);
  const T vh = A::div(v, bc2);
  p = A::sub(p, A::div(A::mul(lr, mh), A::add(f_sqrt(vh), T(1e-8))));
}

// FP32 Adam with the bias corrections applied as precomputed reciprocals:
// one sqrt and one division per parameter.
__device__ __forceinline__ void adam_fast(float& p, float& m, float& v, float g, float i1, float i2,
                                          float lr) {
  m = 0.9f * m + 0.1f * g;
  v = 0.999f * v + 0.001f * (g * g);
  float s;
  asm("sqrt.approx.f32 %0, %1;" : "=f"(s) : "f"(v * i2));  // MUFU.SQRT
  p -= __fdividef(lr * (m * i1), s + 1e-8f);
}

__device__ __forceinline__ float act_tanh(float x) { return tanh_fast(x); }
__device__ __forceinline__ double act_tanh(double x) { return tanh(x); }

__device__ __forceinline__ int ld_volatile(const int* p) { return *(volatile const int*)p; }
__device__ __forceinline__ void st_volatile(int* p, int v) { *(volatile int*)p = v; }

constexpr int kConsumedDone = 1 << 30;

// uint16 permutations always live in shared memory, int32 ones (series too
// long for the shared-memory double buffer) in global memory.  Keeping the
// address space a compile-time property lets the compiler emit LDS/STS
// instead of generic loads (which go through L1TEX with global latency).
template <typename PermT>
__host__ __device__ constexpr bool perm_smem() {
  return sizeof(PermT) == 2;
}

// Fisher-Yates of arange(n) from the top index down (Generator.permutation)
template <typename PermT>
__device__ __forceinline__ void fisher_yates(Pcg64& rng, PermT* perm, int n) {
  for (int i = 0; i < n; ++i) perm[i] = (PermT)i;
  for (int i = n - 1; i > 0; --i) {
    const int j = (int)rng.interval32((uint32_t)i);
    const PermT a = perm[i];
    perm[i] = perm[j];
    perm[j] = a;
  }
}

// ---------------------------------------------------------------------------
// Warp-cooperative permutation producer.
//
// numpy's Generator.permutation(n) is Fisher-Yates from i = n-1 down, each j
// drawn by random_interval(i): masked rejection over the buffered 32-bit
// PCG64 stream (low half of each next64 first).  The sequential part is only
// the accept/swap scan; the draws themselves are an LCG, so the warp
// produces 32 consecutive next64 outputs at once by jump-ahead
// (s_{k+l} = a^l s_k + inc * sum_{t<l} a^t, per-lane constants), stages the
// 64 uint32 draws in shared memory, and lane 0 consumes them.  When an epoch
// ends mid-batch, the stream is rewound to exactly the next64 calls numpy
// would have made (with the half-consumed high word buffered), so epoch e+1
// continues bit-identically.
// ---------------------------------------------------------------------------
struct ProdModel {
  unsigned long long s_hi, s_lo, inc_hi, inc_lo;
  uint32_t buf32;
  int has32, next_ep, n, epochs, pad0, pad1, pad2;
};

__device__ __forceinline__ u128 shfl_u128(u128 v, int src) {
  const unsigned long long hi = __shfl_sync(0xffffffffu, (unsigned long long)(v >> 64), src);
  const unsigned long long lo = __shfl_sync(0xffffffffu, (unsigned long long)v, src);
  return ((u128)hi << 64) | lo;
}

__device__ __forceinline__ unsigned long long xsl_rr(u128 s) {
  const unsigned long long hi = (unsigned long long)(s >> 64), lo = (unsigned long long)s;
  const unsigned long long x = hi ^ lo;
  const unsigned rot = (unsigned)(hi >> 58);
  return (x >> rot) | (x << ((64u - rot) & 63u));
}

template <typename PermT>
__device__ void perm_producer_warp(const PnnLaunch& L, int groups, int pw, int npw, int* produced,
                                   int* consumed, PermT* sperm, ProdModel* pm, uint32_t* ring) {
  const int lane = threadIdx.x & 31;
  const unsigned FULL = 0xffffffffu;
  // lane l holds A = a^(l+1), Gs = sum_{t<=l} a^t  (s_{k+l+1} = A s_k + Gs * inc)
  const u128 a = Pcg64::mult();
  u128 A = a, Gs = 1;
  for (int t = 0; t < lane; ++t) {
    A = A * a;
    Gs = Gs * a + 1;
  }
  if (lane == 0) {
    for (int m = pw; m < groups; m += npw) {
      const int64_t gid = (int64_t)blockIdx.x * groups + m;
      ProdModel st{};
      if (gid < L.n_tasks) {
        const bbml_pnn_task tk = L.tasks[gid];
        Pcg64 rng;
        rng.seed(tk.seed);
        const int P = tk.h * (tk.d + 2) + 1;
        for (int i = 0; i < P; ++i) rng.next64();  // init_model draws (pnn.py:100-103)
        st.s_hi = (unsigned long long)(rng.state >> 64);
        st.s_lo = (unsigned long long)rng.state;
        st.inc_hi = (unsigned long long)(rng.inc >> 64);
        st.inc_lo = (unsigned long long)rng.inc;
        st.n = tk.n;
        st.epochs = tk.epochs;
      }
      pm[m] = st;
    }
  }
  __syncwarp();
  unsigned sleep_ns = 100;
  while (true) {
    bool alive = false, progress = false;
    for (int m = pw; m < groups; m += npw) {
      const int64_t gid = (int64_t)blockIdx.x * groups + m;
      if (gid >= L.n_tasks) continue;
      const int e = pm[m].next_ep;
      if (e >= pm[m].epochs) continue;
      const int c = ld_volatile(consumed + m);
      if (c >= kConsumedDone) {  // consumer stopped (diverged): retire the model
        __syncwarp();
        if (lane == 0) pm[m].next_ep = pm[m].epochs;
        __syncwarp();
        continue;
      }
      alive = true;
      if (c < e - 1) continue;  // buffer (e & 1) still in use by epoch e - 2
      const int n = pm[m].n;
      PermT* perm = (perm_smem<PermT>() ? sperm + (int64_t)m * 2 * L.perm_cap
                                    : (PermT*)L.perm_global + 2 * L.perm_offset[gid]) +
                    (e & 1) * (perm_smem<PermT>() ? (int64_t)L.perm_cap : (int64_t)n);
      for (int x = lane; x < n; x += 32) perm[x] = (PermT)x;
      u128 s = ((u128)pm[m].s_hi << 64) | pm[m].s_lo;
      const u128 inc = ((u128)pm[m].inc_hi << 64) | pm[m].inc_lo;
      const u128 C = Gs * inc;
      int has32 = pm[m].has32;
      uint32_t buf = pm[m].buf32;
      int i = n - 1;
      __syncwarp();
      if (i > 0 && has32) {
        if (lane == 0) {
          const uint32_t v = buf & (0xffffffffu >> __clz(i));
          if ((int)v <= i) {
            const PermT t = perm[i];
            perm[i] = perm[v];
            perm[v] = t;
            --i;
          }
        }
        i = __shfl_sync(FULL, i, 0);
        has32 = 0;
      }
      while (i > 0) {
        const u128 st = A * s + C;
        const unsigned long long o = xsl_rr(st);
        ring[2 * lane] = (uint32_t)o;
        ring[2 * lane + 1] = (uint32_t)(o >> 32);
        __syncwarp();
        int q = 0;
        if (lane == 0) {
          // Serial accept / swap scan (lane 0).  Draws come in groups of 8 (two
          // 16-byte shared loads issued one group ahead); the scan is
          // branch-free -- a rejected draw (or one past the end) swaps slot 0
          // with itself -- and the rejection mask is maintained incrementally
          // (it halves exactly when i drops to mask >> 1) instead of a
          // find-leading-one per draw: 74 instead of 207 cycles per element
          // (tools/micro/fyscan.cu), the same permutation.
          uint32_t mask = 0xffffffffu >> __clz(i | 1);
          const uint4* r4 = (const uint4*)ring;
          uint4 c0 = r4[0], c1 = r4[1];
#pragma unroll 1
          for (int g = 0; g < 8 && i > 0; ++g) {
            uint4 n0 = c0, n1 = c1;
            if (g < 7) {
              n0 = r4[2 * g + 2];
              n1 = r4[2 * g + 3];
            }
            const uint32_t d8[8] = {c0.x, c0.y, c0.z, c0.w, c1.x, c1.y, c1.z, c1.w};
#pragma unroll
            for (int k = 0; k < 8; ++k) {
              const bool live = i > 0;
              q += live;
              const uint32_t v = d8[k] & mask;
              const bool acc = live && (int)v <= i;
              const int ii = acc ? i : 0, vv = acc ? (int)v : 0;
              const PermT x = perm[ii], y = perm[vv];
              perm[ii] = y;
              perm[vv] = x;
              i -= acc;
              mask = ((uint32_t)i <= (mask >> 1)) ? (mask >> 1) : mask;
            }
            c0 = n0;
            c1 = n1;
          }
        }
        q = __shfl_sync(FULL, q, 0);
        i = __shfl_sync(FULL, i, 0);
        if (q < 64) {  // stopped mid-batch: rewind to the next64 calls actually made
          const int used = (q + 1) >> 1;
          s = shfl_u128(st, used - 1);
          has32 = q & 1;
          buf = has32 ? ring[q] : 0u;
        } else {
          s = shfl_u128(st, 31);
          has32 = 0;
        }
        __syncwarp();
      }
      if (lane == 0) {
        pm[m].s_hi = (unsigned long long)(s >> 64);
        pm[m].s_lo = (unsigned long long)s;
        pm[m].has32 = has32;
        pm[m].buf32 = buf;
        pm[m].next_ep = e + 1;
        __threadfence_block();
        st_volatile(produced + m, e + 1);
      }
      __syncwarp();
      progress = true;
    }
    if (!alive) break;
    // FP32: short fixed poll (epochs of short series take ~10 us; a 2 us poll
    // measured slower on app20).  FP64 epochs are several times longer and
    // the spinning producer steals issue slots from the consumer warps of
    // its SM sub-partition, so the poll backs off exponentially up to
    // L.poll_cap_ns and resets whenever an epoch was produced.
    if (!progress) {
      __nanosleep(sleep_ns);
      sleep_ns = min(2 * sleep_ns, (unsigned)L.poll_cap_ns);
    } else {
      sleep_ns = 100;
    }
  }
}

// shared-memory carve-up common to both trainers:
//   [produced | consumed] ints, ProdModel[groups], ring[npw][64], perm buffers
struct PnnSmem {
  int* produced;
  int* consumed;
  ProdModel* pm;
  uint32_t* ring;
  unsigned char* perm;
};

__host__ __device__ inline size_t pnn_smem_header(int groups, int npw) {
  size_t b = 16 * ((2 * groups * sizeof(int) + 15) / 16);
  b += groups * sizeof(ProdModel);
  b += npw * 64 * sizeof(uint32_t);
  return 16 * ((b + 15) / 16);
}

__device__ inline PnnSmem pnn_smem(unsigned char* raw, int groups, int npw) {
  PnnSmem S;
  S.produced = (int*)raw;
  S.consumed = S.produced + groups;
  size_t off = 16 * ((2 * groups * sizeof(int) + 15) / 16);
  S.pm = (ProdModel*)(raw + off);
  off += groups * sizeof(ProdModel);
  S.ring = (uint32_t*)(raw + off);
  S.perm = raw + pnn_smem_header(groups, npw);
  return S;
}

template <typename T, int DM, int SC, typename PermT>
__device__ __forceinline__ void load_chunk(T (&xs)[SC][DM], T (&ys)[SC], const PermT* perm,
                                           int base, int cnt, const double* __restrict__ X,
                                           const double* __restrict__ Y, int xs_stride, int d) {
#pragma unroll
  for (int c = 0; c < SC; ++c) {
    const int row = (int)perm[base + (c < cnt ? c : 0)];
#pragma unroll
    for (int k = 0; k < DM; ++k)
      xs[c][k] = (k < d) ? T(__ldg(X + (int64_t)row * xs_stride + k)) : T(0);
    ys[c] = T(__ldg(Y + row));
  }
}

template <typename T, int DM, int HM, int G, int SC, typename PermT>
__global__ void pnn_train_kernel(PnnLaunch L) {
  static_assert(G == 1 || G == 2 || G == 4 || G == 8 || G == 16 || G == 32, "group size");
  constexpr int U = (HM + G - 1) / G;
  using A = Arith<T>;

  const int groups = L.groups_per_cta;
  const int cons_threads = ((groups * G + 31) / 32) * 32;
  const int npw = ((int)blockDim.x - cons_threads) / 32;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const PnnSmem SM = pnn_smem(smem_raw, groups, npw);
  int* produced = SM.produced;
  int* consumed = SM.consumed;
  PermT* sperm = (PermT*)SM.perm;
  if (threadIdx.x < groups) {
    produced[threadIdx.x] = 0;
    consumed[threadIdx.x] = 0;
  }
  __syncthreads();

  // ===================== producer warps =====================
  if ((int)threadIdx.x >= cons_threads) {
    const int pw = ((int)threadIdx.x - cons_threads) >> 5;
    perm_producer_warp<PermT>(L, groups, pw, npw, produced, consumed, sperm, SM.pm, SM.ring + 64 * pw);
    return;
  }

  // ===================== consumer groups =====================
  const int lane = threadIdx.x & 31;
  const int g = threadIdx.x % G;
  const int gi = threadIdx.x / G;
  const int64_t gid = (int64_t)blockIdx.x * groups + gi;
  if (gi >= groups || gid >= L.n_tasks) return;
  const unsigned gmask = (G == 32) ? 0xffffffffu : (((1u << G) - 1u) << (lane & ~(G - 1)));

  const bbml_pnn_task tk = L.tasks[gid];
  const int orig = L.orig_index[gid];
  const int n = tk.n, d = tk.d, h = tk.h, B = tk.batch;
  const double* __restrict__ X = L.X + tk.row_begin * (int64_t)L.x_stride;
  const double* __restrict__ Y = L.y + tk.row_begin;
  const PermT* pbase = perm_smem<PermT>() ? sperm + (int64_t)gi * 2 * L.perm_cap
                                      : (const PermT*)L.perm_global + 2 * L.perm_offset[gid];
  const int64_t cap = perm_smem<PermT>() ? L.perm_cap : n;

  // ---- init (pnn.py:97-104): every lane replays the P draws, keeps its own
  T w1[U][DM], b1[U], w2[U];
  T mw1[U][DM], vw1[U][DM], mb1[U], vb1[U], mw2[U], vw2[U];
  T b2;
  {
    Pcg64 rng;
    rng.seed(tk.seed);
    const double s1 = __ddiv_rn(1.0, __dsqrt_rn((double)d));
    const double s2 = __ddiv_rn(1.0, __dsqrt_rn((double)h));
#pragma unroll
    for (int u = 0; u < U; ++u) {
      b1[u] = w2[u] = mb1[u] = vb1[u] = mw2[u] = vw2[u] = T(0);
#pragma unroll
      for (int k = 0; k < DM; ++k) w1[u][k] = mw1[u][k] = vw1[u][k] = T(0);
    }
    for (int j = 0; j < h; ++j)
      for (int k = 0; k < d; ++k) {
        const double v = rng.uniform(-s1, s1);
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
          for (int kk = 0; kk < DM; ++kk)
            if (j == g + u * G && kk == k) w1[u][kk] = T(v);
      }
    for (int j = 0; j < h; ++j) {
      const double v = rng.uniform(-s1, s1);
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (j == g + u * G) b1[u] = T(v);
    }
    for (int j = 0; j < h; ++j) {
      const double v = rng.uniform(-s2, s2);
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (j == g + u * G) w2[u] = T(v);
    }
    b2 = T(rng.uniform(-s2, s2));
  }
  T mb2 = T(0), vb2 = T(0);
  const T eps = T(tk.eps), lr = T(tk.lr);

  int64_t t = 0;
  double p1 = 1.0, p2 = 1.0;  // running beta^t (FP32 path only)
  int status = BBML_MODEL_OK, fail_epoch = 0, fail_block = 0;
  double fail_value = 0.0;
  const int nbatches = (n + B - 1) / B;

  T gw1[U][DM], gb1[U], gw2[U], gb2;
  auto zero_grads = [&]() {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      gb1[u] = gw2[u] = T(0);
#pragma unroll
      for (int k = 0; k < DM; ++k) gw1[u][k] = T(0);
    }
    gb2 = T(0);
  };

  for (int ep = 0; ep < tk.epochs; ++ep) {
    while (ld_volatile(produced + gi) <= ep) {
    }
    __threadfence_block();
    const PermT* perm = pbase + (ep & 1) * cap;
    double epoch_loss = 0.0;
    zero_grads();
    T bloss = T(0);

    int bs = 0, s0 = 0;
    T xs[SC][DM], ys[SC];
    load_chunk<T, DM, SC, PermT>(xs, ys, perm, 0, min(SC, min(B, n)), X, Y, L.x_stride, d);
    while (true) {
      const int nb = min(B, n - bs);
      const int cnt = min(SC, nb - s0);
      int nbs = bs, ns0 = s0 + SC;
      if (ns0 >= nb) {
        nbs = bs + B;
        ns0 = 0;
      }
      const bool more = nbs < n;
      T nx[SC][DM], ny[SC];
      if (more) {
        const int nnb = min(B, n - nbs);
        load_chunk<T, DM, SC, PermT>(nx, ny, perm, nbs + ns0, min(SC, nnb - ns0), X, Y,
                                     L.x_stride, d);
      }
      // ---- forward: owned hidden units, partial output pre-activation
      T a[SC][U], zs[SC];
#pragma unroll
      for (int c = 0; c < SC; ++c) {
        T zp = T(0);
#pragma unroll
        for (int u = 0; u < U; ++u) {
          T pre = b1[u];
#pragma unroll
          for (int k = 0; k < DM; ++k) pre += w1[u][k] * xs[c][k];
          a[c][u] = f_tanh(pre);
          zp += a[c][u] * w2[u];
        }
        zs[c] = zp;
      }
#pragma unroll
      for (int m = 1; m < G; m <<= 1)
#pragma unroll
        for (int c = 0; c < SC; ++c) zs[c] += shfl_xor(zs[c], m, gmask, G);
      // ---- loss and back-propagation through softplus
      const T nb_t = T(nb);
#pragma unroll
      for (int c = 0; c < SC; ++c) {
        const bool valid = c < cnt;
        const T z = zs[c] + b2;
        const T sp = softplus(z);
        const T rate = A::add(sp, eps);
        const T re = A::add(rate, eps);
        const T lc = A::sub(rate, A::mul(ys[c], f_log(re)));
        const T drate = A::div(A::sub(T(1), A::div(ys[c], re)), nb_t);
        const T dz = valid ? A::mul(drate, f_exp(A::sub(z, sp))) : T(0);
        if (valid) bloss += lc;
        gb2 += dz;
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const T av = a[c][u];
          gw2[u] += av * dz;
          const T dp = A::mul(A::mul(dz, w2[u]), A::sub(T(1), A::mul(av, av)));
          gb1[u] += dp;
#pragma unroll
          for (int k = 0; k < DM; ++k) gw1[u][k] += dp * xs[c][k];
        }
      }
      if (ns0 == 0) {  // ---- end of minibatch: checks + Adam (pnn.py:243-247)
        const T loss = A::div(bloss, nb_t);
        if (!f_finite(loss)) {
          status = BBML_MODEL_DIVERGED;
          fail_epoch = ep;
          fail_value = (double)loss;
          break;
        }
        bool bad_w1 = false, bad_b1 = false, bad_w2 = false;
#pragma unroll
        for (int u = 0; u < U; ++u) {
#pragma unroll
          for (int k = 0; k < DM; ++k) bad_w1 |= !f_finite(gw1[u][k]);
          bad_b1 |= !f_finite(gb1[u]);
          bad_w2 |= !f_finite(gw2[u]);
        }
        bad_w1 = __any_sync(gmask, bad_w1);
        bad_b1 = __any_sync(gmask, bad_b1);
        bad_w2 = __any_sync(gmask, bad_w2);
        if (bad_w1 || bad_b1 || bad_w2 || !f_finite(gb2)) {
          status = BBML_MODEL_NONFINITE_GRAD;
          fail_epoch = ep;
          fail_block = bad_w1 ? 0 : bad_b1 ? 1 : bad_w2 ? 2 : 3;
          break;
        }
        ++t;
        T bc1, bc2;
        if (sizeof(T) == 8) {
          bc1 = T(1.0 - pow(0.9, (double)t));
          bc2 = T(1.0 - pow(0.999, (double)t));
        } else {
          p1 *= 0.9;
          p2 *= 0.999;
          bc1 = T(1.0 - p1);
          bc2 = T(1.0 - p2);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
#pragma unroll
          for (int k = 0; k < DM; ++k)
            adam_update(w1[u][k], mw1[u][k], vw1[u][k], gw1[u][k], bc1, bc2, lr);
          adam_update(b1[u], mb1[u], vb1[u], gb1[u], bc1, bc2, lr);
          adam_update(w2[u], mw2[u], vw2[u], gw2[u], bc1, bc2, lr);
        }
        adam_update(b2, mb2, vb2, gb2, bc1, bc2, lr);
        epoch_loss += (double)loss;
        zero_grads();
        bloss = T(0);
      }
      if (!more) break;
#pragma unroll
      for (int c = 0; c < SC; ++c) {
        ys[c] = ny[c];
#pragma unroll
        for (int k = 0; k < DM; ++k) xs[c][k] = nx[c][k];
      }
      bs = nbs;
      s0 = ns0;
    }
    __syncwarp(gmask);  // every lane is done reading this epoch's buffer
    if (status != BBML_MODEL_OK) break;
    if (g == 0) {
      if (tk.hist_offset >= 0) L.history[tk.hist_offset + ep] = epoch_loss / nbatches;
      __threadfence_block();
      st_volatile(consumed + gi, ep + 1);
    }
  }
  if (g == 0) st_volatile(consumed + gi, kConsumedDone);  // release the producer lane

  // ---- outputs (pack order)
  double* W = L.weights + tk.w_offset;
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const int j = g + u * G;
    if (j < h) {
#pragma unroll
      for (int kk = 0; kk < DM; ++kk)
        if (kk < d) W[j * d + kk] = (double)w1[u][kk];
      W[h * d + j] = (double)b1[u];
      W[h * d + h + j] = (double)w2[u];
    }
  }
  if (g == 0) {
    W[h * d + 2 * h] = (double)b2;
    bbml_model_status st{};
    st.code = status;
    st.epochs = status == BBML_MODEL_OK ? tk.epochs : fail_epoch;
    st.detail = fail_block;
    st.value = fail_value;
    L.status[orig] = st;
  }
}

// ------------------------------------------------------------------------
// Latency-optimised kernel for h <= 16 (the reference default is h = 10):
// one model per warp.  lane = (sample half sg, hidden unit j): the 16-lane
// half sg owns samples [sg*SP, sg*SP+SP) of each chunk of 2*SP minibatch
// samples, lane j owns unit j (its parameters and Adam moments are
// replicated in both halves and stay bitwise identical).  Per chunk:
//   forward    : SP tanh per lane, z all-reduced over the 16 units (4 shfl)
//   loss chain : lane j < SP runs sample j's softplus / log / exp / div chain
//                once (instead of every lane repeating every sample), then
//                d_z is broadcast with SP shuffles
//   backward   : per-unit gradient sums over the lane's SP samples, then one
//                xor-16 shuffle joins the halves at the end of the minibatch
// ------------------------------------------------------------------------
// NPW producer warps per CTA of 4 models: 4 (one per model) for long series,
// 1 shared producer for short ones, 8 CTAs per SM (48 registers: the spills
// cost less than the latency the extra 24 warps hide; sweep PNN 1.83 -> 0.71 s).
// The long-series variant is left unconstrained: ptxas' larger allocation
// (~240 registers) measured ~25% lower per-step latency on the critical path.
template <typename T, int DM, int SP, typename PermT>
__device__ __forceinline__ void pnn_lat_body(const PnnLaunch& L) {
  using A = Arith<T>;
  const int groups = L.groups_per_cta;  // one model per consumer warp
  const int cons_threads = groups * 32;
  const int npw = ((int)blockDim.x - cons_threads) / 32;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const PnnSmem SM = pnn_smem(smem_raw, groups, npw);
  int* produced = SM.produced;
  int* consumed = SM.consumed;
  PermT* sperm = (PermT*)SM.perm;
  if (threadIdx.x < groups) {
    produced[threadIdx.x] = 0;
    consumed[threadIdx.x] = 0;
  }
  __syncthreads();
  if ((int)threadIdx.x >= cons_threads) {
    const int pw = ((int)threadIdx.x - cons_threads) >> 5;
    perm_producer_warp<PermT>(L, groups, pw, npw, produced, consumed, sperm, SM.pm, SM.ring + 64 * pw);
    return;
  }
  const int lane = threadIdx.x & 31;
  const int gi = threadIdx.x >> 5;
  const int64_t gid = (int64_t)blockIdx.x * groups + gi;
  if (gid >= L.n_tasks) return;
  const int sg = lane >> 4, j = lane & 15;
  const unsigned FULL = 0xffffffffu;

  const bbml_pnn_task tk = L.tasks[gid];
  const int orig = L.orig_index[gid];
  const int n = tk.n, d = tk.d, h = tk.h, B = tk.batch;
  const double* __restrict__ X = L.X + tk.row_begin * (int64_t)L.x_stride;
  const double* __restrict__ Y = L.y + tk.row_begin;
  const PermT* pbase = perm_smem<PermT>() ? sperm + (int64_t)gi * 2 * L.perm_cap
                                      : (const PermT*)L.perm_global + 2 * L.perm_offset[gid];
  const int64_t cap = perm_smem<PermT>() ? L.perm_cap : n;

  // ---- init (pnn.py:97-104)
  T w1[DM], b1 = T(0), w2 = T(0), b2;
  T mw1[DM], vw1[DM], mb1 = T(0), vb1 = T(0), mw2 = T(0), vw2 = T(0), mb2 = T(0), vb2 = T(0);
#pragma unroll
  for (int k = 0; k < DM; ++k) w1[k] = mw1[k] = vw1[k] = T(0);
  {
    Pcg64 rng;
    rng.seed(tk.seed);
    const double s1 = __ddiv_rn(1.0, __dsqrt_rn((double)d));
    const double s2 = __ddiv_rn(1.0, __dsqrt_rn((double)h));
    for (int jj = 0; jj < h; ++jj)
      for (int k = 0; k < d; ++k) {
        const double v = rng.uniform(-s1, s1);
#pragma unroll
        for (int kk = 0; kk < DM; ++kk)
          if (jj == j && kk == k) w1[kk] = T(v);
      }
    for (int jj = 0; jj < h; ++jj) {
      const double v = rng.uniform(-s1, s1);
      if (jj == j) b1 = T(v);
    }
    for (int jj = 0; jj < h; ++jj) {
      const double v = rng.uniform(-s2, s2);
      if (jj == j) w2 = T(v);
    }
    b2 = T(rng.uniform(-s2, s2));
  }
  const T eps = T(tk.eps), lr = T(tk.lr);

  int64_t t = 0;
  double p1 = 1.0, p2 = 1.0;
  int status = BBML_MODEL_OK, fail_epoch = 0, fail_block = 0;
  double fail_value = 0.0;
  const int nbatches = (n + B - 1) / B;
  constexpr int C = 2 * SP;

  T gw1[DM], gb1, gw2, gb2, bloss;
  auto zero_grads = [&]() {
#pragma unroll
    for (int k = 0; k < DM; ++k) gw1[k] = T(0);
    gb1 = gw2 = gb2 = bloss = T(0);
  };
  // rows of samples [off + sg*SP, off + sg*SP + SP) of the chunk (clamped to
  // valid); the FP32 kernel reads the pre-converted float rows so the
  // prefetched values land directly in their registers (no conversion stall)
  const int rstride = sizeof(T) == 8 ? L.x_stride : L.xf_stride;
  const T* __restrict__ XT = (sizeof(T) == 8 ? (const T*)(const void*)L.X : (const T*)(const void*)L.Xf) +
                             tk.row_begin * (int64_t)rstride;
  const T* __restrict__ YT = (sizeof(T) == 8 ? (const T*)(const void*)L.y : (const T*)(const void*)L.yf) +
                             tk.row_begin;
  const bool vec4 = sizeof(T) == 4 && DM <= 4 && rstride == 4;
  const bool y_in_x = vec4 && L.y_in_x;
  // Prefetch: the raw load registers are filled one chunk ahead and only
  // read (masked / unpacked) when that chunk is consumed, so the L2 latency
  // overlaps the previous chunk's compute instead of stalling at the load.
  struct Raw {
    float4 v[SP];
    T x[SP][DM];
    T y[SP];
  };
  auto load = [&](Raw& r, const PermT* perm, int off, int cnt) {
#pragma unroll
    for (int i = 0; i < SP; ++i) {
      const int c = sg * SP + i;
      const int row = (int)perm[off + (c < cnt ? c : 0)];
      if constexpr (sizeof(T) == 4 && DM <= 4) {
        if (vec4) {
          r.v[i] = __ldg((const float4*)(XT + (int64_t)row * 4));
          if (!y_in_x) r.y[i] = __ldg(YT + row);
          continue;
        }
      }
#pragma unroll
      for (int k = 0; k < DM; ++k) r.x[i][k] = (k < d) ? __ldg(XT + (int64_t)row * rstride + k) : T(0);
      r.y[i] = __ldg(YT + row);
    }
  };
  auto unpack = [&](const Raw& r, T (&xs)[SP][DM], T (&ys)[SP]) {
#pragma unroll
    for (int i = 0; i < SP; ++i) {
      if constexpr (sizeof(T) == 4 && DM <= 4) {
        if (vec4) {
          const float e[4] = {r.v[i].x, r.v[i].y, r.v[i].z, r.v[i].w};
#pragma unroll
          for (int k = 0; k < DM; ++k) xs[i][k] = (k < d) ? e[k] : 0.0f;
          ys[i] = y_in_x ? r.v[i].w : r.y[i];
          continue;
        }
      }
#pragma unroll
      for (int k = 0; k < DM; ++k) xs[i][k] = r.x[i][k];
      ys[i] = r.y[i];
    }
  };

  for (int ep = 0; ep < tk.epochs; ++ep) {
    while (ld_volatile(produced + gi) <= ep) {
    }
    __threadfence_block();
    const PermT* perm = pbase + (ep & 1) * cap;
    T eloss = T(0);
    zero_grads();
    int bs = 0, s0 = 0;
    // ping-pong prefetch buffers: a register copy (cur = nxt) would force the
    // in-flight loads to complete, so the two buffers alternate roles instead
    Raw rb0, rb1;
    bool flip = false;
    load(rb0, perm, 0, min(C, min(B, n)));
    while (true) {
      const int nb = min(B, n - bs);
      const int cnt = min(C, nb - s0);
      int nbs = bs, ns0 = s0 + C;
      if (ns0 >= nb) {
        nbs = bs + B;
        ns0 = 0;
      }
      const bool more = nbs < n;
      T xs[SP][DM], ys[SP];
      const int ncnt = more ? min(C, min(B, n - nbs) - ns0) : 0;
      if (!flip) {
        unpack(rb0, xs, ys);
        if (more) load(rb1, perm, nbs + ns0, ncnt);
      } else {
        unpack(rb1, xs, ys);
        if (more) load(rb0, perm, nbs + ns0, ncnt);
      }
      flip = !flip;

      // forward
      T a[SP], z[SP];
#pragma unroll
      for (int i = 0; i < SP; ++i) {
        T pre = b1;
#pragma unroll
        for (int k = 0; k < DM; ++k) pre += w1[k] * xs[i][k];
        a[i] = act_tanh(pre);
        z[i] = a[i] * w2;
      }
#pragma unroll
      for (int m = 1; m < 16; m <<= 1)
#pragma unroll
        for (int i = 0; i < SP; ++i) z[i] += __shfl_xor_sync(FULL, z[i], m);
      // loss chain of sample (sg, j) on lane j < SP
      T zj = z[0], yj = ys[0];
#pragma unroll
      for (int i = 1; i < SP; ++i)
        if (j == i) {
          zj = z[i];
          yj = ys[i];
        }
      const bool mine = j < SP && (sg * SP + j) < cnt;
      const T nb_t = T(nb);
      const T zz = zj + b2;
      const T sp = softplus(zz);
      const T rate = A::add(sp, eps);
      const T re = A::add(rate, eps);
      const T drate = A::div(A::sub(T(1), A::div(yj, re)), nb_t);
      const T dzj = mine ? A::mul(drate, f_exp(A::sub(zz, sp))) : T(0);
      if (mine) bloss += A::sub(rate, A::mul(yj, f_log(re)));
      // backward (own unit, own half's samples)
#pragma unroll
      for (int i = 0; i < SP; ++i) {
        const T dz = __shfl_sync(FULL, dzj, (lane & 16) | i);
        gb2 += dz;
        gw2 += a[i] * dz;
        const T dp = A::mul(A::mul(dz, w2), A::sub(T(1), A::mul(a[i], a[i])));
        gb1 += dp;
#pragma unroll
        for (int k = 0; k < DM; ++k) gw1[k] += dp * xs[i][k];
      }
      if (ns0 == 0) {  // end of minibatch
#pragma unroll
        for (int k = 0; k < DM; ++k) gw1[k] += __shfl_xor_sync(FULL, gw1[k], 16);
        gb1 += __shfl_xor_sync(FULL, gb1, 16);
        gw2 += __shfl_xor_sync(FULL, gw2, 16);
        gb2 += __shfl_xor_sync(FULL, gb2, 16);
        // one warp-wide OR of every finiteness predicate (loss first, then the
        // adam_step block order W1, b1, W2, b2; pnn.py:244-245, 180-183)
        bool bw1 = false;
#pragma unroll
        for (int k = 0; k < DM; ++k) bw1 |= !f_finite(gw1[k]);
        const unsigned bits = (!f_finite(bloss) ? 1u : 0u) | (bw1 ? 2u : 0u) |
                              (!f_finite(gb1) ? 4u : 0u) | (!f_finite(gw2) ? 8u : 0u) |
                              (!f_finite(gb2) ? 16u : 0u);
        const unsigned any = __reduce_or_sync(FULL, bits);
        if (any) {
          T lsum = bloss;
#pragma unroll
          for (int m = 1; m < 32; m <<= 1) lsum += __shfl_xor_sync(FULL, lsum, m);
          const T loss = A::div(lsum, nb_t);
          if ((any & 1u) || !f_finite(loss)) {
            status = BBML_MODEL_DIVERGED;
            fail_epoch = ep;
            fail_value = (double)loss;
            break;
          }
          status = BBML_MODEL_NONFINITE_GRAD;
          fail_epoch = ep;
          fail_block = (any & 2u) ? 0 : (any & 4u) ? 1 : (any & 8u) ? 2 : 3;
          break;
        }
        ++t;
        if constexpr (sizeof(T) == 8) {
          const T bc1 = T(1.0 - pow(0.9, (double)t));
          const T bc2 = T(1.0 - pow(0.999, (double)t));
#pragma unroll
          for (int k = 0; k < DM; ++k) adam_update(w1[k], mw1[k], vw1[k], gw1[k], bc1, bc2, lr);
          adam_update(b1, mb1, vb1, gb1, bc1, bc2, lr);
          adam_update(w2, mw2, vw2, gw2, bc1, bc2, lr);
          adam_update(b2, mb2, vb2, gb2, bc1, bc2, lr);
        } else {
          p1 *= 0.9;
          p2 *= 0.999;
          const T i1 = __fdividef(1.0f, (float)(1.0 - p1)), i2 = __fdividef(1.0f, (float)(1.0 - p2));
#pragma unroll
          for (int k = 0; k < DM; ++k) adam_fast(w1[k], mw1[k], vw1[k], gw1[k], i1, i2, lr);
          adam_fast(b1, mb1, vb1, gb1, i1, i2, lr);
          adam_fast(w2, mw2, vw2, gw2, i1, i2, lr);
          adam_fast(b2, mb2, vb2, gb2, i1, i2, lr);
        }
        eloss += A::div(bloss, nb_t);  // this lane's share of the batch mean
        zero_grads();
      }
      if (!more) break;
      bs = nbs;
      s0 = ns0;
    }
    __syncwarp();
    if (status != BBML_MODEL_OK) break;
    if (tk.hist_offset >= 0) {
      double el = (double)eloss;
#pragma unroll
      for (int m = 1; m < 32; m <<= 1) el += __shfl_xor_sync(FULL, el, m);
      if (lane == 0) L.history[tk.hist_offset + ep] = el / nbatches;
    }
    if (lane == 0) {
      __threadfence_block();
      st_volatile(consumed + gi, ep + 1);
    }
  }
  if (lane == 0) st_volatile(consumed + gi, kConsumedDone);

  double* W = L.weights + tk.w_offset;
  if (sg == 0 && j < h) {
#pragma unroll
    for (int kk = 0; kk < DM; ++kk)
      if (kk < d) W[j * d + kk] = (double)w1[kk];
    W[h * d + j] = (double)b1;
    W[h * d + h + j] = (double)w2;
  }
  if (lane == 0) {
    W[h * d + 2 * h] = (double)b2;
    bbml_model_status st{};
    st.code = status;
    st.epochs = status == BBML_MODEL_OK ? tk.epochs : fail_epoch;
    st.detail = fail_block;
    st.value = fail_value;
    L.status[orig] = st;
  }
}

// ------------------------------------------------------------------------
// FP64 trainer for h <= 16 (the drop-in's default arithmetic and the bench
// headline).  Same warp-per-model lane map as pnn_lat_body (lane = (sample
// half sg, hidden unit j)) with numpy's elementwise rounding (no FMA
// contraction in the elementwise chain), rebuilt around what an FP64 step
// costs on sm_100a, where every FP64 instruction is issue-bound (64 FP64
// lanes / SM) and the per-model chain is sequential:
//   * Adam bias corrections 1 - beta^t come from a host table computed with
//     libm pow (the value Python's float pow gives the reference,
//     pnn.py:185-186) instead of two device pow() calls per step; beyond the
//     table both are exactly 1.0 and the divisions by them are skipped
//     (x / 1.0 == x exactly), which leaves one sqrt and one division per
//     parameter for all but the first ~37k steps.
//   * minibatch rows are staged into shared memory by cp.async (8-byte
//     LDGSTS, one chunk ahead, per-warp double buffer) instead of being
//     prefetched into registers: the row gather stays off the critical
//     path without 2 x SP x (DM+1) doubles of live registers (the register
//     prefetch spilled at DM = 4 in FP64).
//   * each half-warp runs Adam for half of its unit's parameters; the
//     gradient halves and the updated weights are exchanged with one
//     xor-16 shuffle per parameter pair.
// ------------------------------------------------------------------------
// TMA bulk copies (cp.async.bulk, SASS UBLKCP) into shared memory, completion
// tracked by a per-buffer mbarrier (expected transaction bytes + parity).
__device__ __forceinline__ unsigned smem_addr(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  unsigned done = 0;
  while (!done) {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(done)
        : "r"(smem_addr(bar)), "r"(parity)
        : "memory");
  }
}
__device__ __forceinline__ void tma_bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar))
      : "memory");
}

// pnn.py:184-188 with numpy's rounding, branch-free (f64math.cuh).
// BC = false: both bias corrections are exactly 1.0 (x / 1.0 == x), so the
// two divisions by them are dropped.
__device__ __forceinline__ double sqrt_any_bf(double x) { return sqrt_nonneg_bf(x); }
template <bool BC>
__device__ __forceinline__ void adam_exact(double& p, double& m, double& v, double g, double bc1,
                                           double bc2, double lr) {
  m = __dadd_rn(__dmul_rn(0.9, m), __dmul_rn(1.0 - 0.9, g));
  v = __dadd_rn(__dmul_rn(0.999, v), __dmul_rn(1.0 - 0.999, __dmul_rn(g, g)));
  const double mh = BC ? div_rn_bf(m, bc1) : m;
  const double vh = BC ? div_rn_bf(v, bc2) : v;
  p = __dsub_rn(p, div_rn_bf(__dmul_rn(lr, mh), __dadd_rn(sqrt_any_bf(vh), 1e-8)));
}

// staging: per consumer warp, 2 buffers x 2 halves x SP row records of
// L.rec doubles ([x_0 .. x_{W-1}, y, pad], 16-byte multiple), then 2 mbarriers
template <int SP>
__host__ __device__ constexpr int f64_stage_doubles(int rec) {
  return 2 * 2 * SP * rec + 2;
}

// Development-only phase clocks of the FP64 consumer loop (compile with
// -DBBML_PNN_PROF): lane 0 of every consumer warp accumulates clock64() per
// phase; printed to stderr after each bbml_pnn_train call.
#ifdef BBML_PNN_PROF
__device__ unsigned long long g_pnn_prof[8];
#define PP_T(v) long long v = clock64()
#define PP_ADD(k, t0)                                                                  \
  do {                                                                                 \
    if (lane == 0) atomicAdd(&g_pnn_prof[k], (unsigned long long)(clock64() - (t0))); \
  } while (0)
#else
#define PP_T(v) (void)0
#define PP_ADD(k, t0) (void)0
#endif

template <int DM, int SP, typename PermT>
__device__ __forceinline__ void pnn_f64_body(const PnnLaunch& L) {
  const int RW = L.rec;       // staged row record: x[0..W), y at W = L.rec_y, pad
  const int YI = L.rec_y;
  constexpr int C = 2 * SP;   // samples per chunk (both halves)
  constexpr int NP = DM + 2;  // per-unit parameters: w1[0..DM), b1, w2
  const int groups = L.groups_per_cta;
  const int cons_threads = groups * 32;
  const int npw = ((int)blockDim.x - cons_threads) / 32;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const PnnSmem SM = pnn_smem(smem_raw, groups, npw);
  int* produced = SM.produced;
  int* consumed = SM.consumed;
  PermT* sperm = (PermT*)SM.perm;
  double* stage_all = (double*)(smem_raw + L.stage_off);
  if (threadIdx.x < groups) {
    produced[threadIdx.x] = 0;
    consumed[threadIdx.x] = 0;
  }
  __syncthreads();
  if ((int)threadIdx.x >= cons_threads) {
    const int pw = ((int)threadIdx.x - cons_threads) >> 5;
    perm_producer_warp<PermT>(L, groups, pw, npw, produced, consumed, sperm, SM.pm, SM.ring + 64 * pw);
    return;
  }
  const int lane = threadIdx.x & 31;
  const int gi = threadIdx.x >> 5;
  const int64_t gid = (int64_t)blockIdx.x * groups + gi;
  if (gid >= L.n_tasks) return;
  const int sg = lane >> 4, j = lane & 15;
  const unsigned FULL = 0xffffffffu;
  double* stage = stage_all + gi * f64_stage_doubles<SP>(RW);
  uint64_t* bars = (uint64_t*)(stage + 2 * 2 * SP * RW);  // one mbarrier per staging buffer
  if (lane == 0) {
    mbar_init(bars, 1);
    mbar_init(bars + 1, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  unsigned parity = 0;  // bit b: phase parity buffer b waits for next
  int inflight = -1;    // buffer with a bulk copy not yet waited for

  const bbml_pnn_task tk = L.tasks[gid];
  const int orig = L.orig_index[gid];
  const int n = tk.n, d = tk.d, h = tk.h, B = tk.batch;
  const PermT* pbase = perm_smem<PermT>() ? sperm + (int64_t)gi * 2 * L.perm_cap
                                      : (const PermT*)L.perm_global + 2 * L.perm_offset[gid];
  const int64_t cap = perm_smem<PermT>() ? L.perm_cap : n;

  // ---- init (pnn.py:97-104): unit j's parameters p[0..DM) = W1[j, :], p[DM] = b1[j], p[DM+1] = W2[j]
  double p[NP], m1[NP], m2[NP];
#pragma unroll
  for (int q = 0; q < NP; ++q) p[q] = m1[q] = m2[q] = 0.0;
  double b2, mb2 = 0.0, vb2 = 0.0;
  {
    Pcg64 rng;
    rng.seed(tk.seed);
    const double s1 = __ddiv_rn(1.0, __dsqrt_rn((double)d));
    const double s2 = __ddiv_rn(1.0, __dsqrt_rn((double)h));
    for (int jj = 0; jj < h; ++jj)
      for (int k = 0; k < d; ++k) {
        const double v = rng.uniform(-s1, s1);
#pragma unroll
        for (int kk = 0; kk < DM; ++kk)
          if (jj == j && kk == k) p[kk] = v;
      }
    for (int jj = 0; jj < h; ++jj) {
      const double v = rng.uniform(-s1, s1);
      if (jj == j) p[DM] = v;
    }
    for (int jj = 0; jj < h; ++jj) {
      const double v = rng.uniform(-s2, s2);
      if (jj == j) p[DM + 1] = v;
    }
    b2 = rng.uniform(-s2, s2);
  }
  const double eps = tk.eps, lr = tk.lr;
  int64_t t = 0;
  int status = BBML_MODEL_OK, fail_epoch = 0, fail_block = 0;
  double fail_value = 0.0;
  const int nbatches = (n + B - 1) / B;

  // one TMA bulk copy per row record: lane (sg, j < SP) fetches sample
  // sg*SP + j of the chunk (samples past the minibatch fetch sample 0's row:
  // finite, and their d_z is 0); lane 0 posts the chunk's byte count first
  const double* __restrict__ R = L.rows + tk.row_begin * (int64_t)RW;
  const unsigned rec_bytes = (unsigned)RW * 8u;
  auto issue = [&](int buf, const PermT* perm, int off, int cnt) {
    if (lane == 0) mbar_expect_tx(bars + buf, (unsigned)C * rec_bytes);
    __syncwarp();
    if (j < SP) {
      const int c = sg * SP + j;
      const int row = (int)perm[off + (c < cnt ? c : 0)];
      tma_bulk_g2s(stage + ((buf * 2 + sg) * SP + j) * RW, R + (int64_t)row * RW, rec_bytes, bars + buf);
    }
    inflight = buf;
  };
  auto wait = [&](int buf) {
    mbar_wait(bars + buf, (parity >> buf) & 1u);
    parity ^= 1u << buf;
    if (inflight == buf) inflight = -1;
  };

  double g[NP], gb2, bloss;
  auto zero_grads = [&]() {
#pragma unroll
    for (int q = 0; q < NP; ++q) g[q] = 0.0;
    gb2 = bloss = 0.0;
  };
  for (int ep = 0; ep < tk.epochs; ++ep) {
    PP_T(tp);
    while (ld_volatile(produced + gi) <= ep) {
    }
    __threadfence_block();
    PP_ADD(5, tp);
    const PermT* perm = pbase + (ep & 1) * cap;
    double eloss = 0.0;
    zero_grads();
    int bs = 0, s0 = 0, buf = 0;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    issue(0, perm, 0, min(C, min(B, n)));
    double2 bc = t < L.bc_len ? __ldg(L.bc + t) : make_double2(1.0, 1.0);
    while (true) {
      const int nb = min(B, n - bs);
      const int cnt = min(C, nb - s0);
      int nbs = bs, ns0 = s0 + C;
      if (ns0 >= nb) {
        nbs = bs + B;
        ns0 = 0;
      }
      const bool more = nbs < n;
      const int cur_inflight = inflight;  // the copy into `buf` (issued one chunk ago)
      if (more) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic reads of buf^1 before the async overwrite
        issue(buf ^ 1, perm, nbs + ns0, min(C, min(B, n - nbs) - ns0));
      }
      (void)cur_inflight;
      PP_T(t0);
      wait(buf);
      PP_ADD(0, t0);
      PP_T(t1);
      const double* rows = stage + (buf * 2 + sg) * SP * RW;

      // forward (own unit, own half's samples)
      double a[SP], z[SP];
#pragma unroll
      for (int i = 0; i < SP; ++i) {
        double pre = p[DM];
#pragma unroll
        for (int k = 0; k < DM; ++k) pre += p[k] * rows[i * RW + k];
        a[i] = tanh_bf(pre);
        z[i] = a[i] * p[DM + 1];
      }
#pragma unroll
      for (int mm = 1; mm < 16; mm <<= 1)
#pragma unroll
        for (int i = 0; i < SP; ++i) z[i] += __shfl_xor_sync(FULL, z[i], mm);
      PP_ADD(1, t1);
      PP_T(t2);
      // loss chain of sample (sg, j) on lane j < SP (pnn.py:131-138)
      double zj = z[0];
#pragma unroll
      for (int i = 1; i < SP; ++i)
        if (j == i) zj = z[i];
      const double yj = j < SP ? rows[j * RW + YI] : 0.5;
      const bool mine = j < SP && (sg * SP + j) < cnt;
      const double nb_t = (double)nb;
      const double zz = __dadd_rn(zj, b2);
      // softplus = numpy logaddexp(0, z) = max(z, 0) + log1p(exp(-|z|))
      const double ez = exp_neg_bf(-fabs(zz));
      const double sp = __dadd_rn(fmax(zz, 0.0), log1p_bf(ez));
      const double rate = __dadd_rn(sp, eps);
      const double re = __dadd_rn(rate, eps);
      const double drate = div_rn_bf(__dsub_rn(1.0, div_rn_bf(yj, re)), nb_t);
      // d softplus / dz = sigmoid(z): the reference's exp(z - softplus(z))
      // (pnn.py:138) evaluated as 1/(1+e) or e/(1+e) from the e = exp(-|z|)
      // above (<= 1.5 ulp apart), off the log1p -> division chain
      const double sg1 = div_rn_bf(zz >= 0.0 ? 1.0 : ez, __dadd_rn(1.0, ez));
      const double dzj = mine ? __dmul_rn(drate, sg1) : 0.0;
      if (mine) bloss += __dsub_rn(rate, __dmul_rn(yj, log_bf(re)));
      PP_ADD(2, t2);
      PP_T(t3);
      // backward (pnn.py:139-146)
#pragma unroll
      for (int i = 0; i < SP; ++i) {
        const double dz = __shfl_sync(FULL, dzj, (lane & 16) | i);
        gb2 += dz;
        g[DM + 1] += a[i] * dz;
        const double dp = __dmul_rn(__dmul_rn(dz, p[DM + 1]), __dsub_rn(1.0, __dmul_rn(a[i], a[i])));
        g[DM] += dp;
#pragma unroll
        for (int k = 0; k < DM; ++k) g[k] += dp * rows[i * RW + k];
      }
      __syncwarp();  // every lane has read this staging buffer
      PP_ADD(3, t3);
      PP_T(t4);
      buf ^= 1;
      if (ns0 == 0) {  // end of minibatch: checks + Adam (pnn.py:243-247, 174-189)
        // gradient halves: lane sg owns parameters q with q % 2 == sg; one
        // xor-16 shuffle per pair sends the partner's partial sum and
        // receives the partner's partial of an own parameter
#pragma unroll
        for (int q = 0; q < NP; q += 2) {
          if (q + 1 < NP) {
            const double send = sg ? g[q] : g[q + 1];
            const double recv = __shfl_xor_sync(FULL, send, 16);
            if (sg) g[q + 1] += recv;
            else g[q] += recv;
          } else {
            g[q] += __shfl_xor_sync(FULL, g[q], 16);
          }
        }
        gb2 += __shfl_xor_sync(FULL, gb2, 16);
        bool bw1 = false, bb1 = false, bw2 = false;
#pragma unroll
        for (int q = 0; q < NP; ++q) {
          const bool own = (q % 2 == sg) || (q + 1 == NP && NP % 2 == 1);
          const bool bad = own && !isfinite(g[q]) && (q >= DM || q < d) && j < h;
          if (q < DM) bw1 |= bad;
          else if (q == DM) bb1 |= bad;
          else bw2 |= bad;
        }
        const unsigned bits = (!isfinite(bloss) ? 1u : 0u) | (bw1 ? 2u : 0u) | (bb1 ? 4u : 0u) |
                              (bw2 ? 8u : 0u) | (!isfinite(gb2) ? 16u : 0u);
        const unsigned any = __reduce_or_sync(FULL, bits);
        PP_ADD(6, t4);
        PP_T(t6);
        if (any) {
          double lsum = bloss;
#pragma unroll
          for (int mm = 1; mm < 32; mm <<= 1) lsum += __shfl_xor_sync(FULL, lsum, mm);
          const double loss = __ddiv_rn(lsum, nb_t);
          if ((any & 1u) || !isfinite(loss)) {
            status = BBML_MODEL_DIVERGED;
            fail_epoch = ep;
            fail_value = loss;
            break;
          }
          status = BBML_MODEL_NONFINITE_GRAD;
          fail_epoch = ep;
          fail_block = (any & 2u) ? 0 : (any & 4u) ? 1 : (any & 8u) ? 2 : 3;
          break;
        }
        ++t;
        const double bc1 = bc.x, bc2 = bc.y;
        bc = t < L.bc_len ? __ldg(L.bc + t) : make_double2(1.0, 1.0);  // next step's, early
        // slot i of lane (sg, j) is parameter q = 2i + sg of unit j, so every
        // lane runs the same NP/2 (branch-free, overlapping) updates; lanes
        // of padded units / inputs compute on zeros and keep their values.
        // b2 rides in slot 0 of the first padded unit's lane (h < 16) and is
        // broadcast, else it takes one more slot on every lane.
        const bool b2_slot = h < 16;
        const bool b2_lane = b2_slot && sg == 0 && j == h;
        auto adam_all = [&](auto bc_tag) {
          constexpr bool BC = decltype(bc_tag)::value;
          // all NP/2 updates first, then the commits as selects: lane-divergent
          // stores (sg, real, b2_lane) as branches would split the updates
          // into separate blocks and serialise their latency chains
          double np_[NP / 2], nm_[NP / 2], nv_[NP / 2];
#pragma unroll
          for (int i = 0; i < NP / 2; ++i) {
            const bool b2i = i == 0 && b2_lane;
            double pv = sg ? p[2 * i + 1] : p[2 * i];
            double mv = sg ? m1[2 * i + 1] : m1[2 * i];
            double vv = sg ? m2[2 * i + 1] : m2[2 * i];
            double gv = sg ? g[2 * i + 1] : g[2 * i];
            pv = b2i ? b2 : pv;
            mv = b2i ? mb2 : mv;
            vv = b2i ? vb2 : vv;
            gv = b2i ? gb2 : gv;
            adam_exact<BC>(pv, mv, vv, gv, bc1, bc2, lr);
            np_[i] = pv;
            nm_[i] = mv;
            nv_[i] = vv;
          }
#pragma unroll
          for (int i = 0; i < NP / 2; ++i) {
            const bool b2i = i == 0 && b2_lane;
            const int q = 2 * i + sg;
            const bool real = j < h && (q >= DM || q < d) && !b2i;
            const bool lo = real && !sg, hi = real && sg;
            p[2 * i] = lo ? np_[i] : p[2 * i];
            m1[2 * i] = lo ? nm_[i] : m1[2 * i];
            m2[2 * i] = lo ? nv_[i] : m2[2 * i];
            p[2 * i + 1] = hi ? np_[i] : p[2 * i + 1];
            m1[2 * i + 1] = hi ? nm_[i] : m1[2 * i + 1];
            m2[2 * i + 1] = hi ? nv_[i] : m2[2 * i + 1];
            if (i == 0) {
              b2 = b2i ? np_[0] : b2;
              mb2 = b2i ? nm_[0] : mb2;
              vb2 = b2i ? nv_[0] : vb2;
            }
          }
          if (b2_slot) b2 = __shfl_sync(FULL, b2, h);
          else adam_exact<BC>(b2, mb2, vb2, gb2, bc1, bc2, lr);
        };
        if (bc1 != 1.0 || bc2 != 1.0) adam_all(std::true_type{});  // warp-uniform (t is per model)
        else adam_all(std::false_type{});
        PP_ADD(7, t6);
        // updated weights back to the partner half
#pragma unroll
        for (int q = 0; q + 1 < NP; q += 2) {
          const double send = sg ? p[q + 1] : p[q];
          const double recv = __shfl_xor_sync(FULL, send, 16);
          if (sg) p[q] = recv;
          else p[q + 1] = recv;
        }
        eloss += div_rn_bf(bloss, nb_t);  // this lane's share of the batch mean
        zero_grads();
      }
      PP_ADD(4, t4);
      if (!more) break;
      bs = nbs;
      s0 = ns0;
    }
    __syncwarp();
    if (status != BBML_MODEL_OK) break;
    if (tk.hist_offset >= 0) {
      double el = eloss;
#pragma unroll
      for (int mm = 1; mm < 32; mm <<= 1) el += __shfl_xor_sync(FULL, el, mm);
      if (lane == 0) L.history[tk.hist_offset + ep] = el / nbatches;
    }
    if (lane == 0) {
      __threadfence_block();
      st_volatile(consumed + gi, ep + 1);
    }
  }
  if (inflight >= 0) wait(inflight);  // a run that stopped early leaves no copy in flight
  if (lane == 0) st_volatile(consumed + gi, kConsumedDone);

  double* W = L.weights + tk.w_offset;
  if (sg == 0 && j < h) {
#pragma unroll
    for (int kk = 0; kk < DM; ++kk)
      if (kk < d) W[j * d + kk] = p[kk];
    W[h * d + j] = p[DM];
    W[h * d + h + j] = p[DM + 1];
  }
  if (lane == 0) {
    W[h * d + 2 * h] = b2;
    bbml_model_status st{};
    st.code = status;
    st.epochs = status == BBML_MODEL_OK ? tk.epochs : fail_epoch;
    st.detail = fail_block;
    st.value = fail_value;
    L.status[orig] = st;
  }
}

template <int DM, int SP, typename PermT>
__global__ void __launch_bounds__(256, 1) pnn_f64_kernel(PnnLaunch L) {
  pnn_f64_body<DM, SP, PermT>(L);
}
// long series, 128 registers: two CTAs (or one plus shorter work) per SM
template <int DM, int SP, typename PermT>
__global__ void __launch_bounds__(256, 2) pnn_f64_kernel_half(PnnLaunch L) {
  pnn_f64_body<DM, SP, PermT>(L);
}
// short series: 4 consumer + 1 shared producer warp
template <int DM, int SP, typename PermT>
__global__ void __launch_bounds__(160, 3) pnn_f64_kernel_shared(PnnLaunch L) {
  pnn_f64_body<DM, SP, PermT>(L);
}
template <int DM, int SP, typename PermT>
__global__ void __launch_bounds__(160, 4) pnn_f64_kernel_shared4(PnnLaunch L) {
  pnn_f64_body<DM, SP, PermT>(L);
}
// FP64 CTA shapes (development knobs, defaults from one-box A/B; short-series
// CTAs per SM 3 vs 4: suite16 FP64 step 1 069-1 078 vs 1 092-1 106 ms and
// 14.9 vs 92 MB of DRAM traffic per PNN call -- the 96-register variant
// spills, tools/r2r.sh):
//   BBML_F64_LONG_NPW  = 1 | 2 | 4   producer warps per CTA for n >= kLongSeries
//   BBML_F64_SHORT_MINB = 3 | 4      CTAs per SM for the shared-producer kernel
static int env_int(const char* name, int dflt) {
  const char* e = getenv(name);
  return e ? atoi(e) : dflt;
}
static int f64_long_npw() {
  static const int v = env_int("BBML_F64_LONG_NPW", 4);
  return v;
}
static int f64_long_groups() {
  static const int v = env_int("BBML_F64_LONG_GROUPS", 4);
  return (v == 1 || v == 2) ? v : 4;
}
static int f64_long_minb() {
  static const int v = env_int("BBML_F64_LONG_MINB", 1);
  return v;
}
static int f64_short_npw() {
  static const int v = env_int("BBML_F64_SHORT_NPW", 1);
  return v;
}
static int f64_short_minb() {
  static const int v = env_int("BBML_F64_SHORT_MINB", 3);
  return v;
}

// long series: 4 consumer + 4 producer warps, register allocation unconstrained
template <typename T, int DM, int SP, typename PermT>
__global__ void pnn_lat_kernel(PnnLaunch L) {
  pnn_lat_body<T, DM, SP, PermT>(L);
}
// short series: 4 consumer + 1 shared producer warp, 8 CTAs per SM (A/B over
// 2..10 CTAs per SM on the sweep and suite16 workloads: 8 is fastest)
template <typename T, int DM, int SP, typename PermT>
__global__ void __launch_bounds__(160, 8) pnn_lat_kernel_shared(PnnLaunch L) {
  pnn_lat_body<T, DM, SP, PermT>(L);
}
// 4 consumer + 2 producer warps (each producer serves 2 models), 2 CTAs per SM
template <typename T, int DM, int SP, typename PermT>
__global__ void __launch_bounds__(192, 2) pnn_lat_kernel_np2(PnnLaunch L) {
  pnn_lat_body<T, DM, SP, PermT>(L);
}

// producer warps per CTA for long-series buckets (tuning knob BBML_PNN_NPW = 1|2|4)
static int long_npw() {
  static const int v = [] {
    const char* e = getenv("BBML_PNN_NPW");
    // default 4: one-box A/B on suite16 R=32 (r01): NPW=4 636.9 ms vs NPW=2 660.8 ms
    const int x = e ? atoi(e) : 4;
    return (x == 1 || x == 2 || x == 4) ? x : 4;
  }();
  return v;
}

// ------------------------------------------------------------------------
// host dispatch
// ------------------------------------------------------------------------

// FP32 row copy: 16-byte rows {x0..x3} when x_stride <= 4, with y folded
// into slot 3 when x_stride <= 3 (one LDG.128 per sample in the hot loop).
__global__ void to_float_kernel(const double* __restrict__ X, int xs, float* __restrict__ Xf,
                                int xfs, const double* __restrict__ y, float* __restrict__ yf,
                                int64_t rows) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < rows;
       r += (int64_t)gridDim.x * blockDim.x) {
    for (int k = 0; k < xfs; ++k) Xf[r * xfs + k] = k < xs ? (float)X[r * xs + k] : 0.0f;
    const float yv = (float)y[r];
    yf[r] = yv;
    if (xs <= 3 && xfs == 4) Xf[r * 4 + 3] = yv;
  }
}

// FP64 row records for the TMA staging: [x_0 .. x_{W-1} (zero past
// x_stride), y, zero pad] with W = rec_y, rec = W + 1 rounded up to an even
// count (16-byte multiple, the bulk-copy granularity).
__global__ void to_records_kernel(const double* __restrict__ X, int xs, const double* __restrict__ y,
                                  int rec_y, int rec, double* __restrict__ out, int64_t rows) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < rows * rec;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / rec;
    const int k = (int)(e - r * rec);
    out[e] = k < xs ? X[r * xs + k] : k == rec_y ? y[r] : 0.0;
  }
}

static int bucket_d(int d) { return d <= 2 ? 2 : d <= 4 ? 4 : 16; }
static int bucket_h(int h) { return h <= 16 ? 16 : 64; }
// series at least this long get a dedicated producer warp (see launch_variant)
constexpr int kLongSeries = 2048;
// BBML_PNN_SPLIT=1 launches short series separately with a shared producer
// warp (more CTAs per SM).  Off by default: measured slower on suite16
// because the co-resident short-series warps stretch the critical chains.
static bool split_long_short() {
  static const bool on = [] {
    const char* e = getenv("BBML_PNN_SPLIT");
    return e && e[0] == '1';
  }();
  return on;
}
static int bucket_n(int n) { return (split_long_short() && n < kLongSeries) ? 0 : 1; }

template <typename T, int DM, int HM, typename PermT>
static cudaError_t launch_variant(PnnLaunch L, int64_t nmax, size_t smem_limit, cudaStream_t s) {
  constexpr bool LAT = HM <= 16;  // h <= 16: warp-per-model latency kernel
  constexpr int G = 32;
  constexpr int SC = 10;
  // 4 models per CTA.  Long series: one warp-cooperative producer warp per
  // model (one sequential Fisher-Yates scan keeps up with one consumer warp).
  // Short series (n < kLongSeries): one producer serves the 4 models, so the
  // CTA is 5 warps and eight CTAs fit per SM.
  const bool shared_prod = LAT && nmax < kLongSeries && !(sizeof(T) == 8 && f64_short_npw() > 1);
  // FP64 long series: models per CTA (BBML_F64_LONG_GROUPS; fewer models per
  // CTA = a smaller register footprint, so other groups co-reside on the SM)
  const int groups_max = (sizeof(T) == 8 && LAT && !shared_prod) ? f64_long_groups() : 4;
  const int npw_long = !LAT ? groups_max
                     : sizeof(T) == 8 ? (nmax < kLongSeries ? f64_short_npw() : f64_long_npw())
                                      : long_npw();
  const int npw_max = shared_prod ? 1 : npw_long;
  const size_t flags = pnn_smem_header(groups_max, groups_max);
  const size_t per_group = 2 * (size_t)nmax * sizeof(PermT);
  int groups = perm_smem<PermT>() ? (int)std::min<size_t>(groups_max, (smem_limit - flags) / per_group) : 0;
  size_t smem;
  int npw;
  if (groups >= 1) {
    npw = std::min(groups, npw_max);
    L.perm_in_smem = 1;
    L.perm_cap = (int32_t)nmax;
    smem = pnn_smem_header(groups, npw) + (size_t)groups * per_group;
  } else {
    groups = groups_max;
    npw = groups;
    L.perm_in_smem = 0;
    L.perm_cap = 0;
    smem = pnn_smem_header(groups, npw);
  }
  L.groups_per_cta = groups;
  const int cons = ((groups * G + 31) / 32) * 32;
  const int prod = 32 * npw;
  const int blocks = (int)ceil_div(L.n_tasks, groups);
  constexpr bool F64 = LAT && sizeof(T) == 8;
  if (F64) {  // per-warp row staging after the permutation buffers
    L.stage_off = (int32_t)(16 * ((smem + 15) / 16));
    smem = L.stage_off + (size_t)groups * f64_stage_doubles<5>(L.rec) * sizeof(double);
  }
  auto k = !LAT ? pnn_train_kernel<T, DM, HM, G, SC, PermT>
                : F64 ? (shared_prod ? (f64_short_minb() == 4 ? pnn_f64_kernel_shared4<DM, 5, PermT>
                                                              : pnn_f64_kernel_shared<DM, 5, PermT>)
                         : f64_long_minb() == 2 ? pnn_f64_kernel_half<DM, 5, PermT>
                                                : pnn_f64_kernel<DM, 5, PermT>)
                      : (npw == 1 ? pnn_lat_kernel_shared<T, DM, 5, PermT>
                                  : npw == 2 ? pnn_lat_kernel_np2<T, DM, 5, PermT>
                                             : pnn_lat_kernel<T, DM, 5, PermT>);
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  k<<<blocks, cons + prod, smem, s>>>(L);
  return cudaGetLastError();
}

// uint16 in shared memory whenever one model's double buffer fits, else int32
// in global memory.  The launcher's workspace allocation and the variant
// choice both ask this one predicate (they must agree: the int32 variant
// dereferences L.perm_global).
static bool perm_fits_smem(int64_t nmax, size_t smem_limit) {
  return nmax <= 65535 && pnn_smem_header(4, 4) + 2 * (size_t)nmax * sizeof(uint16_t) <= smem_limit;
}

template <typename T, int DM, int HM>
static cudaError_t launch_dm_hm(const PnnLaunch& L, int64_t nmax, size_t smem_limit,
                                cudaStream_t s) {
  if (perm_fits_smem(nmax, smem_limit)) return launch_variant<T, DM, HM, uint16_t>(L, nmax, smem_limit, s);
  if (L.perm_global == nullptr) return cudaErrorInvalidValue;  // launcher invariant violated
  return launch_variant<T, DM, HM, int32_t>(L, nmax, smem_limit, s);
}

template <typename T>
static cudaError_t launch_bucket(int dm, int hm, const PnnLaunch& L, int64_t nmax,
                                 size_t smem_limit, cudaStream_t s) {
  if (dm <= 2) {
    return hm <= 16 ? launch_dm_hm<T, 2, 16>(L, nmax, smem_limit, s)
                    : launch_dm_hm<T, 2, 64>(L, nmax, smem_limit, s);
  } else if (dm <= 4) {
    return hm <= 16 ? launch_dm_hm<T, 4, 16>(L, nmax, smem_limit, s)
                    : launch_dm_hm<T, 4, 64>(L, nmax, smem_limit, s);
  }
  return hm <= 16 ? launch_dm_hm<T, 16, 16>(L, nmax, smem_limit, s)
                  : launch_dm_hm<T, 16, 64>(L, nmax, smem_limit, s);
}

// {1 - 0.9^t, 1 - 0.999^t} for t = 1.. until both round to exactly 1.0,
// with the host libm pow: the reference evaluates `1 - beta**t` with Python
// float pow (pnn.py:185-186), i.e. the same C library call.
static const std::vector<double2>& adam_bias_table() {
  static const std::vector<double2> tab = [] {
    std::vector<double2> v;
    for (int t = 1;; ++t) {
      const double a = 1.0 - std::pow(0.9, (double)t), b = 1.0 - std::pow(0.999, (double)t);
      if (a == 1.0 && b == 1.0) break;
      v.push_back(make_double2(a, b));
    }
    return v;
  }();
  return tab;
}

bbml_status pnn_train_launch(const bbml_pnn_task* tasks, int32_t n_tasks, const double* X,
                             const double* y, int32_t x_stride, double* weights, double* history,
                             bbml_model_status* status, int32_t precision, cudaStream_t stream) {
  std::vector<int> idx(n_tasks);
  for (int i = 0; i < n_tasks; ++i) {
    const bbml_pnn_task& t = tasks[i];
    if (t.n < 1 || t.d < 1 || t.h < 1 || t.epochs < 1 || t.batch < 1 || t.row_begin < 0 ||
        t.w_offset < 0 || t.seed.n_words < 1 || t.seed.n_words > BBML_MAX_ENTROPY_WORDS) {
      set_error("pnn task %d: invalid field", i);
      return BBML_ERR_INVALID;
    }
    if (t.d > BBML_MAX_INPUTS || t.h > BBML_PNN_MAX_HIDDEN) {
      set_error("pnn task %d: d=%d h=%d outside the supported envelope", i, t.d, t.h);
      return BBML_ERR_UNSUPPORTED;
    }
    if (t.hist_offset >= 0 && history == nullptr) {
      set_error("pnn task %d: history requested but history == NULL", i);
      return BBML_ERR_INVALID;
    }
    idx[i] = i;
  }
  auto cost = [&](int i) {
    const bbml_pnn_task& t = tasks[i];
    return (double)t.epochs * (double)((t.n + t.batch - 1) / t.batch);
  };
  // homogeneous launches per (d, h) bucket; longest sequential chains first
  std::stable_sort(idx.begin(), idx.end(), [&](int a, int b) {
    const int ka = bucket_d(tasks[a].d) * 1000 + bucket_h(tasks[a].h) * 2 + bucket_n(tasks[a].n);
    const int kb = bucket_d(tasks[b].d) * 1000 + bucket_h(tasks[b].h) * 2 + bucket_n(tasks[b].n);
    if (ka != kb) return ka < kb;
    return cost(a) > cost(b);
  });
  auto cost_sorted = [](const bbml_pnn_task& t) {
    return (double)t.epochs * (double)((t.n + t.batch - 1) / t.batch);
  };
  std::vector<bbml_pnn_task> sorted(n_tasks);
  std::vector<int32_t> orig(n_tasks);
  std::vector<int64_t> poff(n_tasks);
  int64_t total = 0;
  for (int i = 0; i < n_tasks; ++i) {
    sorted[i] = tasks[idx[i]];
    orig[i] = idx[i];
    poff[i] = total;
    total += sorted[i].n;
  }
  ScratchBuffer scratch(stream);
  bbml_pnn_task* d_tasks = nullptr;
  int32_t* d_orig = nullptr;
  int64_t* d_poff = nullptr;
  bbml_status st;
  if ((st = scratch.alloc(&d_tasks, n_tasks)) != BBML_OK) return st;
  if ((st = scratch.alloc(&d_orig, n_tasks)) != BBML_OK) return st;
  if ((st = scratch.alloc(&d_poff, n_tasks)) != BBML_OK) return st;
  if ((st = scratch.upload(d_tasks, sorted.data(), n_tasks)) != BBML_OK) return st;
  if ((st = scratch.upload(d_orig, orig.data(), n_tasks)) != BBML_OK) return st;
  if ((st = scratch.upload(d_poff, poff.data(), n_tasks)) != BBML_OK) return st;

  int dev = 0;
  cudaGetDevice(&dev);
  int smem_optin = 0;
  cudaDeviceGetAttribute(&smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  const size_t smem_limit = std::min<size_t>((size_t)smem_optin, 200 * 1024);

  float* d_xf = nullptr;  // FP32 kernels: one conversion pass over the rows they read
  float* d_yf = nullptr;
  int xf_stride = x_stride;
  if (precision == 32) {
    int64_t rows = 0;
    for (int i = 0; i < n_tasks; ++i) rows = std::max<int64_t>(rows, sorted[i].row_begin + sorted[i].n);
    xf_stride = x_stride <= 4 ? 4 : x_stride;
    if ((st = scratch.alloc(&d_xf, rows * xf_stride)) != BBML_OK) return st;
    if ((st = scratch.alloc(&d_yf, rows)) != BBML_OK) return st;
    to_float_kernel<<<(int)std::min<int64_t>(ceil_div(rows, 256), 4096), 256, 0, stream>>>(
        X, x_stride, d_xf, xf_stride, y, d_yf, rows);
  }
  // FP64: 16-byte-multiple row records for the TMA staging (see pnn_f64_body)
  double* d_rec = nullptr;
  int rec_y = 0, rec = 0;
  if (precision == 64) {
    int dmax = 1;
    int64_t rows = 0;
    for (int i = 0; i < n_tasks; ++i) {
      dmax = std::max(dmax, sorted[i].d);
      rows = std::max<int64_t>(rows, sorted[i].row_begin + sorted[i].n);
    }
    rec_y = std::max(x_stride, bucket_d(dmax));  // every bucket's DM <= rec_y
    rec = (rec_y + 2) & ~1;
    if ((st = scratch.alloc(&d_rec, std::max<int64_t>(rows, 1) * rec)) != BBML_OK) return st;
    const int64_t tot = rows * rec;
    if (tot > 0)
      to_records_kernel<<<(int)std::min<int64_t>(ceil_div(tot, 256), 4096), 256, 0, stream>>>(
          X, x_stride, y, rec_y, rec, d_rec, rows);
  }
  // FP64: Adam bias-correction table (see pnn_f64_body)
  double2* d_bc = nullptr;
  const std::vector<double2>& bc_host = adam_bias_table();
  if (precision == 64) {
    if ((st = scratch.alloc(&d_bc, (int64_t)bc_host.size())) != BBML_OK) return st;
    if ((st = scratch.upload(d_bc, bc_host.data(), (int64_t)bc_host.size())) != BBML_OK) return st;
  }
  // shape groups (homogeneous launches); all scratch is allocated before the fork
  std::vector<std::pair<int, int>> groups_rng;
  int32_t* d_perm = nullptr;  // global double-buffer workspace, only if some bucket needs it
  for (int b0 = 0; b0 < n_tasks;) {
    int b1 = b0;
    int64_t nmax = 0;
    while (b1 < n_tasks && bucket_d(sorted[b1].d) == bucket_d(sorted[b0].d) &&
           bucket_h(sorted[b1].h) == bucket_h(sorted[b0].h) &&
           bucket_n(sorted[b1].n) == bucket_n(sorted[b0].n)) {
      nmax = std::max<int64_t>(nmax, sorted[b1].n);
      ++b1;
    }
    if (!perm_fits_smem(nmax, smem_limit) && d_perm == nullptr) {
      if ((st = scratch.alloc(&d_perm, 2 * total)) != BBML_OK) return st;
    }
    groups_rng.push_back({b0, b1});
    b0 = b1;
  }
  // the group holding the longest sequential chain launches first, so its
  // CTAs are resident before the shorter groups fill the SMs
  // (off by default: A/B on suite16 FP64, tools/r2k.sh -- the long CTAs then
  // hold whole SMs while the BR-BPNN call waits; step 1089 -> 1126 ms)
  if (env_int("BBML_PNN_LONG_FIRST", 0)) {
    auto chain = [&](const std::pair<int, int>& g) {
      double c = 0.0;
      for (int i = g.first; i < g.second; ++i) c = std::max(c, cost_sorted(sorted[i]));
      return c;
    };
    std::stable_sort(groups_rng.begin(), groups_rng.end(),
                     [&](const std::pair<int, int>& a, const std::pair<int, int>& b) { return chain(a) > chain(b); });
  }
  StreamFork fork(stream, (int)groups_rng.size());
  for (size_t gno = 0; gno < groups_rng.size(); ++gno) {
    const int begin = groups_rng[gno].first, end = groups_rng[gno].second;
    const int dm = bucket_d(sorted[begin].d), hm = bucket_h(sorted[begin].h);
    int64_t nmax = 0;
    for (int i = begin; i < end; ++i) nmax = std::max<int64_t>(nmax, sorted[i].n);
    cudaStream_t stream = fork.child((int)gno);
    PnnLaunch L{};
    L.tasks = d_tasks + begin;
    L.orig_index = d_orig + begin;
    L.perm_offset = d_poff + begin;
    L.n_tasks = end - begin;
    L.X = X;
    L.y = y;
    L.Xf = d_xf;
    L.yf = d_yf;
    L.xf_stride = xf_stride;
    L.y_in_x = (precision == 32 && x_stride <= 3) ? 1 : 0;
    L.x_stride = x_stride;
    L.weights = weights;
    L.history = history;
    L.status = status;
    L.perm_global = d_perm;
    L.poll_cap_ns = precision == 64 ? 2000 : 100;
    L.bc = d_bc;
    L.bc_len = precision == 64 ? (int32_t)bc_host.size() : 0;
    L.rows = d_rec;
    L.rec = rec;
    L.rec_y = rec_y;
    cudaError_t e = precision == 32 ? launch_bucket<float>(dm, hm, L, nmax, smem_limit, stream)
                                    : launch_bucket<double>(dm, hm, L, nmax, smem_limit, stream);
    if (e != cudaSuccess) return cuda_status(e, "pnn_train launch");
  }
  if ((st = fork.join()) != BBML_OK) return st;
#ifdef BBML_PNN_PROF
  {
    unsigned long long pr[8];
    cudaStreamSynchronize(stream);
    cudaMemcpyFromSymbol(pr, g_pnn_prof, sizeof(pr));
    fprintf(stderr, "[pnn_prof] Mcycles tma-wait %.1f forward %.1f loss %.1f backward %.1f batch-end %.1f (grads+checks %.1f, adam %.1f) epoch-wait %.1f\n",
            pr[0] * 1e-6, pr[1] * 1e-6, pr[2] * 1e-6, pr[3] * 1e-6, pr[4] * 1e-6, pr[6] * 1e-6, pr[7] * 1e-6, pr[5] * 1e-6);
    const unsigned long long z[8] = {};
    cudaMemcpyToSymbol(g_pnn_prof, z, sizeof(z));
  }
#endif
  return scratch.release();
}

}  // namespace bbml

// ------------------------------------------------------------------------
// unit level: pnn.loss_and_grads (pnn.py:121-147) for one (model, batch) per
// thread, FP64.  Used by the drop-in loss_and_grads and the FD-gradient tests.
// ------------------------------------------------------------------------
namespace bbml {

__global__ void pnn_loss_grad_kernel(const bbml_pred_task* __restrict__ tasks, int n_tasks,
                                     const double* __restrict__ X, const double* __restrict__ Y,
                                     int xs, const double* __restrict__ weights, double nll_eps,
                                     double* __restrict__ loss, double* __restrict__ grads) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_tasks) return;
  const bbml_pred_task tk = tasks[i];
  const int d = tk.d, h = tk.h, n = tk.n;
  const int hd = h * d;
  const double* w = weights + tk.w_offset;
  double* g = grads + tk.w_offset;
  for (int p = 0; p < h * (d + 2) + 1; ++p) g[p] = 0.0;
  double lsum = 0.0;
  for (int s = 0; s < n; ++s) {
    const double* x = X + (tk.row_begin + s) * xs;
    const double y = Y[tk.row_begin + s];
    double z = 0.0;
    for (int j = 0; j < h; ++j) {
      double pre = 0.0;
      for (int k = 0; k < d; ++k) pre = fma(x[k], w[j * d + k], pre);
      z = fma(tanh(__dadd_rn(pre, w[hd + j])), w[hd + h + j], z);
    }
    z = __dadd_rn(z, w[hd + 2 * h]);
    const double sp = softplus(z);
    const double rate = __dadd_rn(sp, tk.eps);
    const double re = __dadd_rn(rate, nll_eps);
    lsum += __dsub_rn(rate, __dmul_rn(y, log(re)));
    const double dz = __dmul_rn(__ddiv_rn(__dsub_rn(1.0, __ddiv_rn(y, re)), (double)n),
                                exp(__dsub_rn(z, sp)));
    for (int j = 0; j < h; ++j) {
      double pre = 0.0;
      for (int k = 0; k < d; ++k) pre = fma(x[k], w[j * d + k], pre);
      const double a = tanh(__dadd_rn(pre, w[hd + j]));
      const double dp = __dmul_rn(__dmul_rn(dz, w[hd + h + j]), __dsub_rn(1.0, __dmul_rn(a, a)));
      for (int k = 0; k < d; ++k) g[j * d + k] = fma(dp, x[k], g[j * d + k]);
      g[hd + j] += dp;
      g[hd + h + j] = fma(a, dz, g[hd + h + j]);
    }
    g[hd + 2 * h] += dz;
  }
  loss[i] = lsum / n;
}

bbml_status pnn_loss_grad_launch(const bbml_pred_task* tasks, int32_t n_tasks, const double* X,
                                 const double* y, int32_t x_stride, const double* weights,
                                 double nll_eps, double* loss, double* grads, cudaStream_t s) {
  for (int i = 0; i < n_tasks; ++i) {
    const bbml_pred_task& t = tasks[i];
    if (t.n < 1 || t.d < 1 || t.h < 1 || t.row_begin < 0 || t.w_offset < 0) {
      set_error("loss_grad task %d: invalid field", i);
      return BBML_ERR_INVALID;
    }
  }
  if (n_tasks == 0) return BBML_OK;
  ScratchBuffer scratch(s);
  bbml_pred_task* d_tasks = nullptr;
  bbml_status st;
  if ((st = scratch.alloc(&d_tasks, n_tasks)) != BBML_OK) return st;
  if ((st = scratch.upload(d_tasks, tasks, n_tasks)) != BBML_OK) return st;
  pnn_loss_grad_kernel<<<(n_tasks + 63) / 64, 64, 0, s>>>(d_tasks, n_tasks, X, y, x_stride,
                                                          weights, nll_eps, loss, grads);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_status(e, "loss_grad launch");
  return scratch.release();
}

}  // namespace bbml
