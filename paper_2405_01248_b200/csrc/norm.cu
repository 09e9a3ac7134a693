// Normalisation kernels (K5/K6 in SURVEY §2.4) and the attention softmax.
//
// GroupNorm(+SiLU) over NHWC [N][HW][C] activations, G groups of C/G
// contiguous channels. Forward = 2 launches:
//   gn_partial   grid (chunks, N): each CTA streams a pixel range with 16-byte
//                loads, keeps per-channel Welford (count, mean, M2) per thread,
//                merges them (Chan) per channel then per group, and writes one
//                partial per (n, chunk, g)  -> no atomics, deterministic
//   gn_apply     merges the chunk partials of its sample in shared memory and
//                normalises (+affine, +SiLU) its pixel range.
// Backward = 2 launches with the same split (per-group sums of g*dy0 and
// g*dy0*xhat, and per-channel dgamma/dbeta accumulated into fp32 buffers).
//
// LayerNorm over rows of C (one warp per row, two-pass in registers), with
// either a per-channel affine or a per-sample adaLN modulation
// y = xhat * (1 + scale[b]) + shift[b] (b = row / rows_per_sample).
// Softmax over fp32 score rows (scale, optional causal mask) -> P in T, and its
// backward dS = scale * P * (dP - rowsum(dP * P)).
#include <cstdlib>
#include <string>
#include "common.cuh"
#include "dpipe.h"

namespace dp {
void set_error(const std::string& s);
int ew_check(const char* what);

template <typename T>
struct NV {
  static constexpr int V = 16 / sizeof(T);
};

template <typename T>
DP_DEV void ld16(const T* p, float* f) {
  uint4 u = *reinterpret_cast<const uint4*>(p);
  if constexpr (sizeof(T) == 4) {
    f[0] = __uint_as_float(u.x);
    f[1] = __uint_as_float(u.y);
    f[2] = __uint_as_float(u.z);
    f[3] = __uint_as_float(u.w);
  } else {
    const __nv_bfloat16* b = reinterpret_cast<const __nv_bfloat16*>(&u);
#pragma unroll
    for (int i = 0; i < 8; ++i) f[i] = __bfloat162float(b[i]);
  }
}
template <typename T>
DP_DEV void st16(T* p, const float* f) {
  uint4 u;
  if constexpr (sizeof(T) == 4) {
    u.x = __float_as_uint(f[0]);
    u.y = __float_as_uint(f[1]);
    u.z = __float_as_uint(f[2]);
    u.w = __float_as_uint(f[3]);
  } else {
    u.x = pack_bf16x2(f[0], f[1]);
    u.y = pack_bf16x2(f[2], f[3]);
    u.z = pack_bf16x2(f[4], f[5]);
    u.w = pack_bf16x2(f[6], f[7]);
  }
  *reinterpret_cast<uint4*>(p) = u;
}

struct Welford {
  float n, mean, m2;
};
DP_DEV Welford wf_merge(Welford a, Welford b) {
  const float n = a.n + b.n;
  if (n == 0.f) return a;
  const float d = b.mean - a.mean;
  const float fb = b.n / n;
  Welford r;
  r.n = n;
  r.mean = a.mean + d * fb;
  r.m2 = a.m2 + b.m2 + d * d * a.n * fb;
  return r;
}

// ------------------------------------------------------------------ GroupNorm
// Grid (pixel chunks, N, channel blocks); a channel block covers whole groups, so one CTA
// owns the statistics of its groups over its pixel chunk. Small feature maps (U-Net 4x4 ..
// 16x16 levels) get parallelism from channel blocks, large ones (VAE 256x256) from chunks.
// Every thread keeps a fixed 16-byte channel vector and strides over pixels (coalesced rows);
// the CTA reduces per channel through shared memory (no atomics), then one warp per group
// merges the channels with shuffles. Stats are shifted sums (shift = the chunk's first value
// of each channel) -> (count, mean, M2) per (sample, chunk, group); the apply / backward
// kernels merge the chunk partials of a group with one warp (lanes over chunks, shuffle
// Chan merge), so no step of either kernel is a serial chain over chunks or channels.
constexpr int GN_THREADS = 256;
constexpr int GN_WARPS = GN_THREADS / 32;
constexpr int GN_MAX_C = 2560;
#ifndef GN_BWD_MINB
#define GN_BWD_MINB 2  // resident CTAs per SM the backward kernels are register-limited to (3, 4 spill)
#endif

struct GnGeom {
  int chunks, ppc, nblk, CB;
};

template <int V>
static GnGeom gn_geom(int N, int HW, int C, int G) {
  // ~8 waves of CTAs (several resident per SM) with at least 512 pixels per chunk; small maps get
  // their parallelism from channel blocks instead (fewer partials to merge per group)
  static const int minpix = [] {  // pixels per chunk floor (DP_GN_MINPIX: experiments)
    const char* e = getenv("DP_GN_MINPIX");
    return e && atoi(e) > 0 ? atoi(e) : 512;  // swept 32..512 on the VAE / U-Net maps (tools/gn_bench.py)
  }();
  int target = (8 * kNumSMs + N - 1) / N;
  const int maxc = (HW + minpix - 1) / minpix;
  GnGeom g{};
  g.chunks = target < maxc ? target : maxc;
  if (g.chunks < 1) g.chunks = 1;
  g.ppc = (HW + g.chunks - 1) / g.chunks;
  g.chunks = (HW + g.ppc - 1) / g.ppc;
  g.nblk = 1;
  // wide layers (e.g. 4096 concat channels of a 2B U-Net decoder) are split into channel blocks
  // of whole groups so that a block's per-channel shared arrays fit (GN_MAX_C)
  while (C / g.nblk > GN_MAX_C && g.nblk * 2 <= G && G % (g.nblk * 2) == 0) g.nblk *= 2;
  while ((long long)g.chunks * N * g.nblk < 2 * kNumSMs && g.nblk * 2 <= G && G % (g.nblk * 2) == 0 &&
         (C / (g.nblk * 2)) % V == 0)
    g.nblk *= 2;
  g.CB = C / g.nblk;
  return g;
}

// thread layout for a block of CVB channel vectors: vector cv0 + tid % width, pixel lane tid / width
struct GnLanes {
  int width, rows_par, cv, rl;
  DP_DEV GnLanes(int CVB, int cv0) {
    width = min(GN_THREADS, CVB - cv0);
    rows_par = GN_THREADS / width;
    cv = cv0 + threadIdx.x % width;
    rl = threadIdx.x / width;
  }
};

// Sum the per-thread vectors red[rl][ch] over the pixel lanes: thread -> channel.
DP_DEV void gn_lane_sum(const float* red, int rows_par, int nch, int c, float& s) {
  s = 0.f;
  for (int r = 0; r < rows_par; ++r) s += red[r * nch + c];
}

DP_DEV Welford wf_shfl_merge(Welford a) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    Welford b{__shfl_xor_sync(0xffffffffu, a.n, o), __shfl_xor_sync(0xffffffffu, a.mean, o),
              __shfl_xor_sync(0xffffffffu, a.m2, o)};
    a = wf_merge(a, b);
  }
  return a;
}

template <typename T>
__global__ void __launch_bounds__(GN_THREADS)
    gn_partial_kernel(const T* __restrict__ x, int HW, int C, int G, int ppc, int CB,
                      float* __restrict__ part) {
  DP_PDL_ENTRY();
  constexpr int V = NV<T>::V;
  const int n = blockIdx.y, chunk = blockIdx.x, nchunks = gridDim.x;
  const int c0 = blockIdx.z * CB;  // first channel of this block
  const int CVB = CB / V;
  const int p0 = chunk * ppc;
  const int p1 = min(HW, p0 + ppc);
  const float cnt = static_cast<float>(p1 - p0);
  __shared__ float r1[GN_THREADS * 8], r2[GN_THREADS * 8];
  __shared__ float cmean[GN_MAX_C], cm2[GN_MAX_C];
  const T* xs = x + (int64_t)n * HW * C + c0;
  for (int cv0 = 0; cv0 < CVB; cv0 += GN_THREADS) {
    const GnLanes L(CVB, cv0);
    const int nch = L.width * V;
    if (L.rl < L.rows_par) {
      float k[V], a1[V], a2[V];
      ld16(xs + (int64_t)p0 * C + L.cv * V, k);
#pragma unroll
      for (int j = 0; j < V; ++j) a1[j] = a2[j] = 0.f;
      const T* xp = xs + (int64_t)(p0 + L.rl) * C + L.cv * V;
      const int64_t step = (int64_t)L.rows_par * C;
      int p = p0 + L.rl;
      for (; p + 3 * L.rows_par < p1; p += 4 * L.rows_par, xp += 4 * step) {
        float f[4][V];
#pragma unroll
        for (int u = 0; u < 4; ++u) ld16(xp + u * step, f[u]);
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int j = 0; j < V; ++j) {
            const float d = f[u][j] - k[j];
            a1[j] += d;
            a2[j] = fmaf(d, d, a2[j]);
          }
      }
      for (; p < p1; p += L.rows_par, xp += step) {
        float f[V];
        ld16(xp, f);
#pragma unroll
        for (int j = 0; j < V; ++j) {
          const float d = f[j] - k[j];
          a1[j] += d;
          a2[j] = fmaf(d, d, a2[j]);
        }
      }
      const int o = L.rl * nch + (L.cv - cv0) * V;
#pragma unroll
      for (int j = 0; j < V; ++j) {
        r1[o + j] = a1[j];
        r2[o + j] = a2[j];
      }
    }
    __syncthreads();
    for (int c = threadIdx.x; c < nch; c += GN_THREADS) {
      float s1, s2;
      gn_lane_sum(r1, L.rows_par, nch, c, s1);
      gn_lane_sum(r2, L.rows_par, nch, c, s2);
      const float m = s1 / cnt;
      const int cc = cv0 * V + c;
      cmean[cc] = to_f(xs[(int64_t)p0 * C + cc]) + m;
      cm2[cc] = fmaxf(s2 - s1 * m, 0.f);
    }
    __syncthreads();
  }
  // one warp per group: equal-count channels -> group (count, mean, M2)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int cg = C / G;
  const int g0 = c0 / cg, gb = CB / cg;
  for (int gi = warp; gi < gb; gi += GN_WARPS) {
    float sm = 0.f;
    for (int c = lane; c < cg; c += 32) sm += cmean[gi * cg + c];
    const float mg = warp_sum(sm) / cg;
    float s = 0.f;
    for (int c = lane; c < cg; c += 32) {
      const float d = cmean[gi * cg + c] - mg;
      s += cm2[gi * cg + c] + cnt * d * d;
    }
    s = warp_sum(s);
    if (lane == 0) {
      float* o = part + (((int64_t)n * nchunks + chunk) * G + g0 + gi) * 3;
      o[0] = cnt * cg;
      o[1] = mg;
      o[2] = s;
    }
  }
}

template <typename T>
__global__ void __launch_bounds__(GN_THREADS, 4)
    gn_apply_kernel(const T* __restrict__ x, const float* __restrict__ gamma,
                    const float* __restrict__ beta, T* __restrict__ y,
                    float* __restrict__ mean_out, float* __restrict__ rstd_out,
                    const float* __restrict__ part, int HW, int C, int G, int ppc, int CB, float eps,
                    int silu_on, const float* __restrict__ sums) {
  DP_PDL_ENTRY();
  constexpr int V = NV<T>::V;
  const int n = blockIdx.y, chunk = blockIdx.x, nchunks = gridDim.x;
  const int c0 = blockIdx.z * CB;
  const int cg = C / G;
  const int g0 = c0 / cg, gb = CB / cg;
  __shared__ float s_mean[256], s_rstd[256];
  __shared__ float s_a[GN_MAX_C], s_b[GN_MAX_C];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int gi = warp; gi < gb; gi += GN_WARPS) {
    Welford a{0.f, 0.f, 0.f};
    if (sums) {
      // (sum, sum of squares) accumulated by the producing conv's epilogue
      const float cnt = static_cast<float>(HW) * cg;
      float s1 = 0.f, s2 = 0.f;
      const int nsamp = gridDim.y;
      for (int k = 0; k < DP_GN_SLOTS; ++k) {
        const float* q = sums + (((int64_t)k * nsamp + n) * G + g0 + gi) * 2;
        s1 += q[0];
        s2 += q[1];
      }
      a.n = cnt;
      a.mean = s1 / cnt;
      a.m2 = fmaxf(s2 - s1 * a.mean, 0.f);
    } else {
      for (int k = lane; k < nchunks; k += 32) {
        const float* q = part + (((int64_t)n * nchunks + k) * G + g0 + gi) * 3;
        a = wf_merge(a, Welford{q[0], q[1], q[2]});
      }
      a = wf_shfl_merge(a);
    }
    if (lane == 0) {
      s_mean[gi] = a.mean;
      s_rstd[gi] = rsqrtf(a.m2 / fmaxf(a.n, 1.f) + eps);
      if (chunk == 0) {
        mean_out[n * G + g0 + gi] = s_mean[gi];
        rstd_out[n * G + g0 + gi] = s_rstd[gi];
      }
    }
  }
  __syncthreads();
  for (int c = threadIdx.x; c < CB; c += GN_THREADS) {
    const int gi = c / cg;
    const float a = s_rstd[gi] * (gamma ? gamma[c0 + c] : 1.f);
    s_a[c] = a;
    s_b[c] = (gamma ? beta[c0 + c] : 0.f) - s_mean[gi] * a;
  }
  __syncthreads();
  const int CVB = CB / V;
  const int p0 = chunk * ppc;
  const int p1 = min(HW, p0 + ppc);
  const int64_t base = (int64_t)n * HW * C + c0;
  for (int cv0 = 0; cv0 < CVB; cv0 += GN_THREADS) {
    const GnLanes L(CVB, cv0);
    if (L.rl >= L.rows_par) continue;
    float a[V], b[V];
#pragma unroll
    for (int j = 0; j < V; ++j) {
      a[j] = s_a[L.cv * V + j];
      b[j] = s_b[L.cv * V + j];
    }
    const int64_t step = (int64_t)L.rows_par * C;
    const T* xp = x + base + (int64_t)(p0 + L.rl) * C + L.cv * V;
    T* yp = y + base + (int64_t)(p0 + L.rl) * C + L.cv * V;
    int p = p0 + L.rl;
    for (; p + 3 * L.rows_par < p1; p += 4 * L.rows_par, xp += 4 * step, yp += 4 * step) {
      float f[4][V];
#pragma unroll
      for (int u = 0; u < 4; ++u) ld16(xp + u * step, f[u]);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
#pragma unroll
        for (int j = 0; j < V; ++j) {
          float v = fmaf(f[u][j], a[j], b[j]);
          if (silu_on) v = silu_t<T>(v);
          f[u][j] = v;
        }
        st16(yp + u * step, f[u]);
      }
    }
    for (; p < p1; p += L.rows_par, xp += step, yp += step) {
      float f[V];
      ld16(xp, f);
#pragma unroll
      for (int j = 0; j < V; ++j) {
        float v = fmaf(f[j], a[j], b[j]);
        if (silu_on) v = silu_t<T>(v);
        f[j] = v;
      }
      st16(yp, f);
    }
  }
}

// backward pass 1: per-channel sums of dy0 and dy0*xhat (dbeta, dgamma: one atomic per channel
// and CTA) and per-group partials A = sum gamma*dy0, B = sum gamma*dy0*xhat (dy0 = dy through
// the optional SiLU)
template <typename T>
__global__ void __launch_bounds__(GN_THREADS, GN_BWD_MINB)
    gn_bwd_partial_kernel(const T* __restrict__ x, const T* __restrict__ dy,
                          const float* __restrict__ gamma, const float* __restrict__ beta,
                          const float* __restrict__ mean, const float* __restrict__ rstd, int HW,
                          int C, int G, int ppc, int CB, int silu_on, float* __restrict__ dgamma,
                          float* __restrict__ dbeta, float* __restrict__ part) {
  DP_PDL_ENTRY();
  constexpr int V = NV<T>::V;
  const int n = blockIdx.y, chunk = blockIdx.x, nchunks = gridDim.x;
  const int c0 = blockIdx.z * CB;
  const int CVB = CB / V;
  const int p0 = chunk * ppc;
  const int p1 = min(HW, p0 + ppc);
  const int cg = C / G;
  __shared__ float r1[GN_THREADS * 8], r2[GN_THREADS * 8];
  __shared__ float s_a[GN_MAX_C], s_b[GN_MAX_C];
  const int64_t base = (int64_t)n * HW * C + c0;
  for (int cv0 = 0; cv0 < CVB; cv0 += GN_THREADS) {
    const GnLanes L(CVB, cv0);
    const int nch = L.width * V;
    if (L.rl < L.rows_par) {
      float sa[V], sb[V], mu[V], rs[V], ga[V], be[V];
#pragma unroll
      for (int j = 0; j < V; ++j) {
        const int c = c0 + L.cv * V + j;
        mu[j] = mean[n * G + c / cg];
        rs[j] = rstd[n * G + c / cg];
        ga[j] = gamma ? gamma[c] : 1.f;
        be[j] = gamma ? beta[c] : 0.f;
        sa[j] = sb[j] = 0.f;
      }
      const int64_t step = (int64_t)L.rows_par * C;
      int64_t off = base + (int64_t)(p0 + L.rl) * C + L.cv * V;
      auto acc = [&](const float* fx, const float* fd) {
#pragma unroll
        for (int j = 0; j < V; ++j) {
          const float xh = (fx[j] - mu[j]) * rs[j];
          float d = fd[j];
          if (silu_on) {
            const float y0 = fmaf(xh, ga[j], be[j]);
            const float s = sigmoid_t<T>(y0);  // one MUFU (bf16) / MUFU rcp without the IEEE fixup (fp32)
            d *= s * (1.f + y0 * (1.f - s));
          }
          sa[j] += d;
          sb[j] = fmaf(d, xh, sb[j]);
        }
      };
      int p = p0 + L.rl;
      // 4 pixels' x and dy loads issued before any arithmetic (8 x 16 B in flight per thread)
      for (; p + 3 * L.rows_par < p1; p += 4 * L.rows_par, off += 4 * step) {
        float fx[4][V], fd[4][V];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          ld16(x + off + u * step, fx[u]);
          ld16(dy + off + u * step, fd[u]);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) acc(fx[u], fd[u]);
      }
      for (; p < p1; p += L.rows_par, off += step) {
        float fx[V], fd[V];
        ld16(x + off, fx);
        ld16(dy + off, fd);
        acc(fx, fd);
      }
      const int o = L.rl * nch + (L.cv - cv0) * V;
#pragma unroll
      for (int j = 0; j < V; ++j) {
        r1[o + j] = sa[j];
        r2[o + j] = sb[j];
      }
    }
    __syncthreads();
    for (int c = threadIdx.x; c < nch; c += GN_THREADS) {
      float a, b;
      gn_lane_sum(r1, L.rows_par, nch, c, a);
      gn_lane_sum(r2, L.rows_par, nch, c, b);
      const int cc = cv0 * V + c;
      s_a[cc] = a;
      s_b[cc] = b;
      if (dgamma) {
        atomicAdd(dgamma + c0 + cc, b);
        atomicAdd(dbeta + c0 + cc, a);
      }
    }
    __syncthreads();
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g0 = c0 / cg, gb = CB / cg;
  for (int gi = warp; gi < gb; gi += GN_WARPS) {
    float A = 0.f, B = 0.f;
    for (int c = lane; c < cg; c += 32) {
      const float ga = gamma ? gamma[c0 + gi * cg + c] : 1.f;
      A += ga * s_a[gi * cg + c];
      B += ga * s_b[gi * cg + c];
    }
    A = warp_sum(A);
    B = warp_sum(B);
    if (lane == 0) {
      float* o = part + (((int64_t)n * nchunks + chunk) * G + g0 + gi) * 2;
      o[0] = A;
      o[1] = B;
    }
  }
}

template <typename T>
__global__ void __launch_bounds__(GN_THREADS, GN_BWD_MINB)
    gn_bwd_apply_kernel(const T* __restrict__ x, const T* __restrict__ dy,
                        const float* __restrict__ gamma, const float* __restrict__ beta,
                        const float* __restrict__ mean, const float* __restrict__ rstd,
                        const float* __restrict__ part, int HW, int C, int G, int ppc, int CB,
                        int silu_on, T* __restrict__ dx, int accumulate) {
  DP_PDL_ENTRY();
  constexpr int V = NV<T>::V;
  const int n = blockIdx.y, chunk = blockIdx.x, nchunks = gridDim.x;
  const int c0 = blockIdx.z * CB;
  const int cg = C / G;
  const int g0 = c0 / cg, gb = CB / cg;
  __shared__ float s_A[256], s_B[256];
  const float inv_m = 1.f / (static_cast<float>(HW) * cg);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int gi = warp; gi < gb; gi += GN_WARPS) {
    float A = 0.f, B = 0.f;
    for (int k = lane; k < nchunks; k += 32) {
      const float* q = part + (((int64_t)n * nchunks + k) * G + g0 + gi) * 2;
      A += q[0];
      B += q[1];
    }
    A = warp_sum(A);
    B = warp_sum(B);
    if (lane == 0) {
      s_A[gi] = A * inv_m;
      s_B[gi] = B * inv_m;
    }
  }
  __syncthreads();
  const int CVB = CB / V;
  const int p0 = chunk * ppc;
  const int p1 = min(HW, p0 + ppc);
  const int64_t base = (int64_t)n * HW * C + c0;
  for (int cv0 = 0; cv0 < CVB; cv0 += GN_THREADS) {
    const GnLanes L(CVB, cv0);
    if (L.rl >= L.rows_par) continue;
    float mu[V], rs[V], ga[V], be[V], gA[V], gB[V];
#pragma unroll
    for (int j = 0; j < V; ++j) {
      const int cl = L.cv * V + j;
      const int gi = cl / cg;
      mu[j] = mean[n * G + g0 + gi];
      rs[j] = rstd[n * G + g0 + gi];
      ga[j] = gamma ? gamma[c0 + cl] : 1.f;
      be[j] = gamma ? beta[c0 + cl] : 0.f;
      gA[j] = s_A[gi];
      gB[j] = s_B[gi];
    }
    const int64_t step = (int64_t)L.rows_par * C;
    int64_t off = base + (int64_t)(p0 + L.rl) * C + L.cv * V;
    auto one = [&](const float* fx, const float* fd, float* fo) {
#pragma unroll
      for (int j = 0; j < V; ++j) {
        const float xh = (fx[j] - mu[j]) * rs[j];
        float d = fd[j];
        if (silu_on) {
          const float y0 = fmaf(xh, ga[j], be[j]);
          const float sg = sigmoid_t<T>(y0);
          d *= sg * (1.f + y0 * (1.f - sg));
        }
        const float v = rs[j] * (ga[j] * d - gA[j] - xh * gB[j]);
        fo[j] = accumulate ? fo[j] + v : v;
      }
    };
    int p = p0 + L.rl;
    // 2 pixels' loads (x, dy, optional dx) issued before the arithmetic
    for (; p + L.rows_par < p1; p += 2 * L.rows_par, off += 2 * step) {
      float fx[2][V], fd[2][V], fo[2][V];
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        ld16(x + off + u * step, fx[u]);
        ld16(dy + off + u * step, fd[u]);
        if (accumulate) ld16(dx + off + u * step, fo[u]);
      }
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        one(fx[u], fd[u], fo[u]);
        st16(dx + off + u * step, fo[u]);
      }
    }
    for (; p < p1; p += L.rows_par, off += step) {
      float fx[V], fd[V], fo[V];
      ld16(x + off, fx);
      ld16(dy + off, fd);
      if (accumulate) ld16(dx + off, fo);
      one(fx, fd, fo);
      st16(dx + off, fo);
    }
  }
}

// ------------------------------------------------------------------ LayerNorm
// one warp per row; per-lane strided elements (coalesced across the warp)
// one warp per row; lane owns 16-byte vectors lane, lane+32, ... (NVEC per lane) -> fully
// coalesced 512-byte warp accesses, the row kept in registers for the two-pass statistics
// RMSNorm (T5 layer norm: no mean subtraction, no bias): y = x * rsqrt(mean(x^2) + eps) * gamma.
// Forward only (the T5 text encoder is frozen); one warp per row like ln_fwd.
template <typename T, int NVEC>
__global__ void __launch_bounds__(256)
    rms_fwd_kernel(const T* __restrict__ x, const float* __restrict__ gamma, T* __restrict__ y,
                   int64_t rows, int C, float eps) {
  DP_PDL_ENTRY();
  constexpr int V = NV<T>::V;
  const int lane = threadIdx.x & 31;
  const int64_t row = blockIdx.x * 8LL + (threadIdx.x >> 5);
  if (row >= rows) return;
  const int CV = C / V;
  const T* xr = x + row * C;
  float v[NVEC][V];
  float q = 0.f;
#pragma unroll
  for (int k = 0; k < NVEC; ++k) {
    const int cv = lane + 32 * k;
    if (cv < CV) {
      ld16(xr + cv * V, v[k]);
    } else {
#pragma unroll
      for (int j = 0; j < V; ++j) v[k][j] = 0.f;
    }
#pragma unroll
    for (int j = 0; j < V; ++j) q = fmaf(v[k][j], v[k][j], q);
  }
  const float rs = rsqrtf(warp_sum(q) / C + eps);
  T* yr = y + row * C;
#pragma unroll
  for (int k = 0; k < NVEC; ++k) {
    const int cv = lane + 32 * k;
    if (cv < CV) {
      float o[V];
#pragma unroll
      for (int j = 0; j < V; j += 4) {  // gamma as 16-byte loads
        const float4 g4 = __ldg(reinterpret_cast<const float4*>(gamma + cv * V + j));
        o[j] = v[k][j] * rs * g4.x;
        o[j + 1] = v[k][j + 1] * rs * g4.y;
        o[j + 2] = v[k][j + 2] * rs * g4.z;
        o[j + 3] = v[k][j + 3] * rs * g4.w;
      }
      st16(yr + cv * V, o);
    }
  }
}

template <typename T, int NVEC>
__global__ void __launch_bounds__(256)
    ln_fwd_kernel(const T* __restrict__ x, const float* __restrict__ gamma,
                  const float* __restrict__ beta, const T* __restrict__ mod,
                  int64_t mod_ld, int shift_off, int scale_off, int rps, T* __restrict__ y,
                  float* __restrict__ mean_out, float* __restrict__ rstd_out, int64_t rows, int C,
                  float eps) {
  DP_PDL_ENTRY();
  constexpr int V = NV<T>::V;
  const int lane = threadIdx.x & 31;
  const int CV = C / V;
  // per-lane affine parameters loaded once (16-byte loads) for all the warp's rows: per-element
  // scalar gamma/beta loads had been 8x the row's own load instructions
  // (rows of <= 4 vectors per lane; wider rows load them per vector inside the row loop)
  constexpr bool HOIST = NVEC <= 4;
  float ga[HOIST ? NVEC : 1][V], be[HOIST ? NVEC : 1][V];
  if (HOIST && gamma) {
#pragma unroll
    for (int k = 0; k < NVEC; ++k) {
      const int cv = lane + 32 * k;
      if (cv < CV) {
#pragma unroll
        for (int j = 0; j < V; j += 4) {
          const float4 g4 = __ldg(reinterpret_cast<const float4*>(gamma + cv * V + j));
          const float4 b4 = __ldg(reinterpret_cast<const float4*>(beta + cv * V + j));
          ga[HOIST ? k : 0][j] = g4.x; ga[HOIST ? k : 0][j + 1] = g4.y;
          ga[HOIST ? k : 0][j + 2] = g4.z; ga[HOIST ? k : 0][j + 3] = g4.w;
          be[HOIST ? k : 0][j] = b4.x; be[HOIST ? k : 0][j + 1] = b4.y;
          be[HOIST ? k : 0][j + 2] = b4.z; be[HOIST ? k : 0][j + 3] = b4.w;
        }
      }
    }
  }
  // warps stride over rows: the grid is one wave of resident blocks (dp_layer_norm_fwd)
  for (int64_t row = blockIdx.x * 8LL + (threadIdx.x >> 5); row < rows; row += gridDim.x * 8LL) {
  const T* xr = x + row * C;
  float v[NVEC][V];
  float s = 0.f;
#pragma unroll
  for (int k = 0; k < NVEC; ++k) {
    const int cv = lane + 32 * k;
    if (cv < CV) {
      ld16(xr + cv * V, v[k]);
    } else {
#pragma unroll
      for (int j = 0; j < V; ++j) v[k][j] = 0.f;
    }
#pragma unroll
    for (int j = 0; j < V; ++j) s += v[k][j];
  }
  const float mu = warp_sum(s) / C;
  float q = 0.f;
#pragma unroll
  for (int k = 0; k < NVEC; ++k) {
    if (lane + 32 * k < CV) {
#pragma unroll
      for (int j = 0; j < V; ++j) {
        const float d = v[k][j] - mu;
        q += d * d;
      }
    }
  }
  const float rs = rsqrtf(warp_sum(q) / C + eps);
  if (lane == 0) {
    mean_out[row] = mu;
    rstd_out[row] = rs;
  }
  T* yr = y + row * C;
  const T* mr = mod ? mod + (row / rps) * mod_ld : nullptr;
#pragma unroll
  for (int k = 0; k < NVEC; ++k) {
    const int cv = lane + 32 * k;
    if (cv < CV) {
      float o[V], gv[V], bv[V];
      if (gamma) {
        if constexpr (HOIST) {
#pragma unroll
          for (int j = 0; j < V; ++j) {
            gv[j] = ga[HOIST ? k : 0][j];
            bv[j] = be[HOIST ? k : 0][j];
          }
        } else {
#pragma unroll
          for (int j = 0; j < V; j += 4) {
            const float4 g4 = __ldg(reinterpret_cast<const float4*>(gamma + cv * V + j));
            const float4 b4 = __ldg(reinterpret_cast<const float4*>(beta + cv * V + j));
            gv[j] = g4.x; gv[j + 1] = g4.y; gv[j + 2] = g4.z; gv[j + 3] = g4.w;
            bv[j] = b4.x; bv[j + 1] = b4.y; bv[j + 2] = b4.z; bv[j + 3] = b4.w;
          }
        }
      }
#pragma unroll
      for (int j = 0; j < V; ++j) {
        const int c = cv * V + j;
        float t = (v[k][j] - mu) * rs;
        if (gamma) t = fmaf(t, gv[j], bv[j]);
        if (mr) t = fmaf(t, 1.f + to_f(mr[scale_off + c]), to_f(mr[shift_off + c]));
        o[j] = t;
      }
      st16(yr + cv * V, o);
    }
  }
  }
}

// Backward of LayerNorm: warps stride over rows (grid sized to the SMs); with affine params
// each lane also accumulates dgamma (dy * xhat) and dbeta (dy) of its channels over its rows in
// registers, the 8 warps of a block merge them in shared memory and the block adds them to the
// fp32 gradients with one atomic per channel (no second pass over x and dy).
template <typename T, int NVEC, bool PG>
__global__ void __launch_bounds__(256)
    ln_bwd_kernel(const T* __restrict__ x, const T* __restrict__ dy,
                  const float* __restrict__ gamma, const T* __restrict__ mod, int64_t mod_ld,
                  int scale_off, int rps, const float* __restrict__ mean,
                  const float* __restrict__ rstd, T* __restrict__ dx, int64_t rows, int C,
                  int accumulate, float* __restrict__ dgamma, float* __restrict__ dbeta) {
  DP_PDL_ENTRY();
  constexpr int V = NV<T>::V;
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int CV = C / V;
  constexpr bool pg = PG;
  float ag[PG ? NVEC : 1][V], ab[PG ? NVEC : 1][V];
#pragma unroll
  for (int k = 0; k < (PG ? NVEC : 1); ++k)
#pragma unroll
    for (int j = 0; j < V; ++j) ag[k][j] = ab[k][j] = 0.f;
  for (int64_t row = blockIdx.x * 8LL + warp; row < rows; row += gridDim.x * 8LL) {
    const float mu = mean[row], rs = rstd[row];
    const T* xr = x + row * C;
    const T* dr = dy + row * C;
    const T* mr = mod ? mod + (row / rps) * mod_ld : nullptr;
    float xh[NVEC][V], g[NVEC][V];
    float s1 = 0.f, s2 = 0.f;
#pragma unroll
    for (int k = 0; k < NVEC; ++k) {
      const int cv = lane + 32 * k;
      if (cv < CV) {
        ld16(xr + cv * V, xh[k]);
        ld16(dr + cv * V, g[k]);
        float gv[V];  // gamma of this vector: 16-byte loads (not one scalar load per element)
        if (gamma) {
#pragma unroll
          for (int j = 0; j < V; j += 4) {
            const float4 g4 = __ldg(reinterpret_cast<const float4*>(gamma + cv * V + j));
            gv[j] = g4.x; gv[j + 1] = g4.y; gv[j + 2] = g4.z; gv[j + 3] = g4.w;
          }
        }
#pragma unroll
        for (int j = 0; j < V; ++j) {
          const int c = cv * V + j;
          xh[k][j] = (xh[k][j] - mu) * rs;
          float d = g[k][j];
          if constexpr (PG) {
            ag[k][j] = fmaf(d, xh[k][j], ag[k][j]);
            ab[k][j] += d;
          }
          if (gamma) d *= gv[j];
          if (mr) d *= 1.f + to_f(mr[scale_off + c]);
          g[k][j] = d;
          s1 += d;
          s2 += d * xh[k][j];
        }
      }
    }
    s1 = warp_sum(s1) / C;
    s2 = warp_sum(s2) / C;
    T* xo = dx + row * C;
#pragma unroll
    for (int k = 0; k < NVEC; ++k) {
      const int cv = lane + 32 * k;
      if (cv < CV) {
        float o[V], prev[V];
        if (accumulate) ld16(xo + cv * V, prev);
#pragma unroll
        for (int j = 0; j < V; ++j) {
          o[j] = rs * (g[k][j] - s1 - xh[k][j] * s2);
          if (accumulate) o[j] += prev[j];
        }
        st16(xo + cv * V, o);
      }
    }
  }
  if constexpr (!PG) return;
  __shared__ float sg[PG ? 2048 : 1], sb[PG ? 2048 : 1];
  for (int c = threadIdx.x; c < C; c += 256) sg[c] = sb[c] = 0.f;
  __syncthreads();
#pragma unroll
  for (int k = 0; k < (PG ? NVEC : 1); ++k) {
    const int cv = lane + 32 * k;
    if (cv < CV) {
#pragma unroll
      for (int j = 0; j < V; ++j) {
        atomicAdd(&sg[cv * V + j], ag[k][j]);
        atomicAdd(&sb[cv * V + j], ab[k][j]);
      }
    }
  }
  __syncthreads();
  for (int c = threadIdx.x; c < C; c += 256) {
    atomicAdd(dgamma + c, sg[c]);
    atomicAdd(dbeta + c, sb[c]);
  }
}

// Parameter gradients of LayerNorm: grid (CV/CVB, nseg). Segment = rows_per_seg rows; block = CVB channel
// vectors (a divisor of the row's CV vectors: no idle lanes at C = 320 / 640 / 1280, where 32-vector blocks
// left up to 3/8 of the lanes idle) x 256/CVB row lanes.
// affine: dgamma[c] += sum dy*xhat, dbeta[c] += sum dy (fp32 atomics)
// mod:    dmod[b][scale_off+c] = sum_{rows of b} dy*gamma?*xhat_aff, dmod[b][shift_off+c] = sum dy
//         (segment = sample b; stored, not accumulated)
template <typename T>
__global__ void __launch_bounds__(256)
    ln_param_grad_kernel(const T* __restrict__ x, const T* __restrict__ dy,
                         const float* __restrict__ mean, const float* __restrict__ rstd,
                         int64_t rows, int C, int rows_per_seg, float* __restrict__ dgamma,
                         float* __restrict__ dbeta, T* __restrict__ dmod, int64_t dmod_ld,
                         int shift_off, int scale_off, int CVB) {
  DP_PDL_ENTRY();
  constexpr int V = NV<T>::V;
  const int RL = 256 / CVB;
  const int lv = threadIdx.x % CVB, ry = threadIdx.x / CVB;
  const int cv = blockIdx.x * CVB + lv;
  const int64_t r0 = (int64_t)blockIdx.y * rows_per_seg;
  const int64_t r1 = min(rows, r0 + rows_per_seg);
  float a[V], b[V];
#pragma unroll
  for (int j = 0; j < V; ++j) a[j] = b[j] = 0.f;
  if (ry < RL) {
#pragma unroll 2
    for (int64_t r = r0 + ry; r < r1; r += RL) {
      float fx[V], fd[V];
      ld16(x + r * C + cv * V, fx);
      ld16(dy + r * C + cv * V, fd);
      const float mu = mean[r], rs = rstd[r];
#pragma unroll
      for (int j = 0; j < V; ++j) {
        a[j] = fmaf(fd[j], (fx[j] - mu) * rs, a[j]);
        b[j] += fd[j];
      }
    }
  }
  __shared__ float ra[256 * 8], rb[256 * 8];
  if (ry < RL) {
#pragma unroll
    for (int j = 0; j < V; ++j) {
      ra[ry * CVB * V + lv * V + j] = a[j];
      rb[ry * CVB * V + lv * V + j] = b[j];
    }
  }
  __syncthreads();
  for (int t = threadIdx.x; t < CVB * V; t += 256) {
    const int c = blockIdx.x * CVB * V + t;
    float sa = 0.f, sb = 0.f;
    for (int k = 0; k < RL; ++k) {
      sa += ra[k * CVB * V + t];
      sb += rb[k * CVB * V + t];
    }
    if (dmod) {
      dmod[blockIdx.y * dmod_ld + scale_off + c] = from_f<T>(sa);
      dmod[blockIdx.y * dmod_ld + shift_off + c] = from_f<T>(sb);
    } else {
      atomicAdd(dgamma + c, sa);
      atomicAdd(dbeta + c, sb);
    }
  }
}

// channel vectors per ln_param_grad block: the divisor of CV (<= 64) that keeps the most of 256 threads busy
static int ln_pg_cvb(int CV) {
  int best = -1, cvb = 1;
  for (int d = 1; d <= 64 && d <= CV; ++d)
    if (CV % d == 0 && (256 / d) * d >= best) {
      best = (256 / d) * d;
      cvb = d;
    }
  return cvb;
}

// ------------------------------------------------------------------ softmax (attention)
// P[r][j] = softmax_j(scale * S[r][j]) with causal mask j > (r % Lq) + causal_off when causal.
template <typename T>
__global__ void __launch_bounds__(256)
    softmax_fwd_kernel(const float* __restrict__ S, T* __restrict__ P, int64_t rows, int cols,
                       int ld, float scale, int causal, int Lq) {
  DP_PDL_ENTRY();
  const int lane = threadIdx.x & 31;
  const int64_t row = blockIdx.x * 8LL + (threadIdx.x >> 5);
  if (row >= rows) return;
  const float* sr = S + row * ld;
  T* pr = P + row * ld;
  const int lim = causal ? static_cast<int>(row % Lq) + 1 : cols;
  float mx = -INFINITY;
  for (int j = lane; j < lim; j += 32) mx = fmaxf(mx, sr[j] * scale);
  mx = warp_max(mx);
  float sum = 0.f;
  for (int j = lane; j < lim; j += 32) sum += __expf(sr[j] * scale - mx);
  sum = warp_sum(sum);
  const float inv = 1.f / sum;
  for (int j = lane; j < cols; j += 32) pr[j] = from_f<T>(j < lim ? __expf(sr[j] * scale - mx) * inv : 0.f);
}

// dS[r][j] = scale * P * (dP - sum_k dP*P)   (dP fp32 from the dO V^T GEMM)
template <typename T>
__global__ void __launch_bounds__(256)
    softmax_bwd_kernel(const T* __restrict__ P, const float* __restrict__ dP, T* __restrict__ dS,
                       int64_t rows, int cols, int ld, float scale) {
  DP_PDL_ENTRY();
  const int lane = threadIdx.x & 31;
  const int64_t row = blockIdx.x * 8LL + (threadIdx.x >> 5);
  if (row >= rows) return;
  const T* pr = P + row * ld;
  const float* dr = dP + row * ld;
  float s = 0.f;
  for (int j = lane; j < cols; j += 32) s += to_f(pr[j]) * dr[j];
  s = warp_sum(s);
  T* o = dS + row * ld;
  for (int j = lane; j < cols; j += 32) o[j] = from_f<T>(scale * to_f(pr[j]) * (dr[j] - s));
}

}  // namespace dp

using namespace dp;

#define DISPATCH_T(dtype, ...)        \
  do {                                \
    if ((dtype) == DP_F32) {          \
      using T = float;                \
      __VA_ARGS__;                    \
    } else {                          \
      using T = __nv_bfloat16;        \
      __VA_ARGS__;                    \
    }                                 \
  } while (0)

#define ST reinterpret_cast<cudaStream_t>(stream)
template <typename T>
static const T* cp(const void* p) {
  return reinterpret_cast<const T*>(p);
}
template <typename T>
static T* mp(void* p) {
  return reinterpret_cast<T*>(p);
}

static int gn_validate(int dtype, int C, int G) {
  const int V = dtype == DP_F32 ? 4 : 8;
  if (G <= 0 || C % G || C % V || G > 256) {
    set_error("group_norm: need C % G == 0, C % 8 == 0 (bf16) / 4 (fp32), G <= 256");
    return DP_ERR_ARGS;
  }
  int nb = 1;
  while (C / nb > GN_MAX_C && nb * 2 <= G && G % (nb * 2) == 0) nb *= 2;
  if (C / nb > GN_MAX_C || (C / nb) % V) {
    set_error("group_norm: channels per group block exceed 2560");
    return DP_ERR_ARGS;
  }
  return 0;
}

static GnGeom gn_geom_rt(int dtype, int N, int HW, int C, int G) {
  return dtype == DP_F32 ? gn_geom<4>(N, HW, C, G) : gn_geom<8>(N, HW, C, G);
}

// ------------------------------------------------------------------ LayerNorm, row groups (bf16)
// LPR = 2^lpr_log2 lanes per row, so a warp normalises 32/LPR rows at once with NV 16-byte vectors per lane
// (C = 320: 8 lanes x 5 vectors, 4 rows per warp; 640: 16 x 5; 1280: 32 x 5). The warp-per-row kernels
// above kept one row in flight per warp and left most lanes of the second vector idle for C = 320;
// with 4 rows' loads in flight per warp the U-Net LayerNorms run at a multiple of their bandwidth.
// The raw bf16 rows stay in registers across both passes (no fp32 copy); shuffles stay inside a
// row group (xor offsets < LPR).
DP_DEV void unpack8(const uint4& u, float (&f)[8]) {
  const __nv_bfloat16* b = reinterpret_cast<const __nv_bfloat16*>(&u);
#pragma unroll
  for (int i = 0; i < 8; ++i) f[i] = __bfloat162float(b[i]);
}
DP_DEV float group_sum(float v, int lpr) {
  for (int o = lpr >> 1; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
DP_DEV void load8f(const float* p, float (&f)[8]) {
  const float4 a = __ldg(reinterpret_cast<const float4*>(p));
  const float4 b = __ldg(reinterpret_cast<const float4*>(p + 4));
  f[0] = a.x; f[1] = a.y; f[2] = a.z; f[3] = a.w; f[4] = b.x; f[5] = b.y; f[6] = b.z; f[7] = b.w;
}

template <int NV>
__global__ void __launch_bounds__(256, 3)
    lnq_fwd_kernel(const __nv_bfloat16* __restrict__ x, const float* __restrict__ gamma,
                   const float* __restrict__ beta, __nv_bfloat16* __restrict__ y,
                   float* __restrict__ mean_out, float* __restrict__ rstd_out, int64_t rows, int C,
                   int lpr_log2, float eps) {
  DP_PDL_ENTRY();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int lpr = 1 << lpr_log2, sub = lane & (lpr - 1), rsub = lane >> lpr_log2;
  const int rpw = 32 >> lpr_log2;
  const int CV = C >> 3;
  const float inv_c = 1.f / C;
  for (int64_t r0 = ((int64_t)blockIdx.x * 8 + warp) * rpw; r0 < rows; r0 += (int64_t)gridDim.x * 8 * rpw) {
    const int64_t row = r0 + rsub;
    const bool rv = row < rows;
    uint4 raw[NV];
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      const int cv = sub + k * lpr;
      raw[k] = make_uint4(0, 0, 0, 0);
      if (rv && cv < CV) raw[k] = *reinterpret_cast<const uint4*>(x + row * C + cv * 8);
    }
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      float f[8];
      unpack8(raw[k], f);
#pragma unroll
      for (int j = 0; j < 8; ++j) s += f[j];
    }
    const float mu = group_sum(s, lpr) * inv_c;
    float q = 0.f;
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      if (sub + k * lpr < CV) {
        float f[8];
        unpack8(raw[k], f);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const float d = f[j] - mu;
          q = fmaf(d, d, q);
        }
      }
    }
    const float rs = rsqrtf(group_sum(q, lpr) * inv_c + eps);
    if (rv && sub == 0) {
      mean_out[row] = mu;
      rstd_out[row] = rs;
    }
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      const int cv = sub + k * lpr;
      if (rv && cv < CV) {
        float f[8], o[8];
        unpack8(raw[k], f);
        if (gamma) {
          float g[8], b[8];
          load8f(gamma + cv * 8, g);
          load8f(beta + cv * 8, b);
#pragma unroll
          for (int j = 0; j < 8; ++j) o[j] = fmaf((f[j] - mu) * rs, g[j], b[j]);
        } else {
#pragma unroll
          for (int j = 0; j < 8; ++j) o[j] = (f[j] - mu) * rs;
        }
        st16(y + row * C + cv * 8, o);
      }
    }
  }
}

template <int NV, bool PG>
__global__ void __launch_bounds__(128, PG ? 2 : 4)
    lnq_bwd_kernel(const __nv_bfloat16* __restrict__ x, const __nv_bfloat16* __restrict__ dy,
                   const float* __restrict__ gamma, const float* __restrict__ mean,
                   const float* __restrict__ rstd, __nv_bfloat16* __restrict__ dx, int64_t rows, int C,
                   int lpr_log2, int accumulate, float* __restrict__ dgamma, float* __restrict__ dbeta) {
  DP_PDL_ENTRY();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int lpr = 1 << lpr_log2, sub = lane & (lpr - 1), rsub = lane >> lpr_log2;
  const int rpw = 32 >> lpr_log2;
  const int CV = C >> 3;
  const float inv_c = 1.f / C;
  float ag[PG ? NV : 1][8], ab[PG ? NV : 1][8];
#pragma unroll
  for (int k = 0; k < (PG ? NV : 1); ++k)
#pragma unroll
    for (int j = 0; j < 8; ++j) ag[k][j] = ab[k][j] = 0.f;
  for (int64_t r0 = ((int64_t)blockIdx.x * 4 + warp) * rpw; r0 < rows; r0 += (int64_t)gridDim.x * 4 * rpw) {
    const int64_t row = r0 + rsub;
    const bool rv = row < rows;
    uint4 rx[NV], rd[NV];
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      const int cv = sub + k * lpr;
      rx[k] = rd[k] = make_uint4(0, 0, 0, 0);
      if (rv && cv < CV) {
        rx[k] = *reinterpret_cast<const uint4*>(x + row * C + cv * 8);
        rd[k] = *reinterpret_cast<const uint4*>(dy + row * C + cv * 8);
      }
    }
    const float mu = rv ? mean[row] : 0.f, rs = rv ? rstd[row] : 0.f;
    float s1 = 0.f, s2 = 0.f;
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      const int cv = sub + k * lpr;
      if (cv < CV) {
        float fx[8], fd[8], g[8];
        unpack8(rx[k], fx);
        unpack8(rd[k], fd);
        if (gamma) load8f(gamma + cv * 8, g);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const float xh = (fx[j] - mu) * rs;
          if constexpr (PG) {
            ag[k][j] = fmaf(fd[j], xh, ag[k][j]);
            ab[k][j] += fd[j];
          }
          const float d = gamma ? fd[j] * g[j] : fd[j];
          s1 += d;
          s2 = fmaf(d, xh, s2);
        }
      }
    }
    s1 = group_sum(s1, lpr) * inv_c;
    s2 = group_sum(s2, lpr) * inv_c;
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      const int cv = sub + k * lpr;
      if (rv && cv < CV) {
        float fx[8], fd[8], g[8], o[8];
        unpack8(rx[k], fx);
        unpack8(rd[k], fd);
        if (gamma) load8f(gamma + cv * 8, g);
        __nv_bfloat16* xo = dx + row * C + cv * 8;
        float prev[8];
        if (accumulate) ld16(xo, prev);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const float xh = (fx[j] - mu) * rs;
          const float d = gamma ? fd[j] * g[j] : fd[j];
          o[j] = rs * (d - s1 - xh * s2);
          if (accumulate) o[j] += prev[j];
        }
        st16(xo, o);
      }
    }
  }
  if constexpr (PG) {
    // lanes with the same `sub` own the same channels: merge the row groups by shuffles, then one
    // shared-memory add per channel per warp and one global atomic per channel per block
    __shared__ float sg[2048], sb[2048];
    for (int c = threadIdx.x; c < C; c += 128) sg[c] = sb[c] = 0.f;
    __syncthreads();
#pragma unroll
    for (int k = 0; k < NV; ++k)
#pragma unroll
      for (int j = 0; j < 8; ++j)
        for (int o = lpr; o < 32; o <<= 1) {
          ag[k][j] += __shfl_xor_sync(0xffffffffu, ag[k][j], o);
          ab[k][j] += __shfl_xor_sync(0xffffffffu, ab[k][j], o);
        }
    if (rsub == 0) {
#pragma unroll
      for (int k = 0; k < NV; ++k) {
        const int cv = sub + k * lpr;
        if (cv < CV)
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            atomicAdd(&sg[cv * 8 + j], ag[k][j]);
            atomicAdd(&sb[cv * 8 + j], ab[k][j]);
          }
      }
    }
    __syncthreads();
    for (int c = threadIdx.x; c < C; c += 128) {
      atomicAdd(dgamma + c, sg[c]);
      atomicAdd(dbeta + c, sb[c]);
    }
  }
}

// lanes per row (log2) and vectors per lane for the row-group LayerNorm (bf16, C % 8 == 0): NV in
// {4, 5, 8}, LPR <= 32; 0 = not covered (the warp-per-row kernels)
static int lnq_plan(int C, int& nv) {
  const int CV = C / 8;
  for (int cand : {5, 4, 8}) {
    for (int l = 0; l <= 5; ++l) {
      const int lpr = 1 << l;
      if (lpr * cand >= CV && lpr * (cand - 1) < CV && (lpr * cand - CV) * 5 <= lpr * cand) {
        nv = cand;
        return l + 1;
      }
    }
  }
  return 0;
}
static bool lnq_enabled() {
  static const int v = [] {
    const char* e = getenv("DP_LN_GROUPS");  // experiments: 0 = warp-per-row kernels
    return e ? atoi(e) : 1;
  }();
  return v != 0;
}

extern "C" {

size_t dp_group_norm_workspace(int N, int HW, int G) {
  // chunking depends only on N and HW (channel blocks do not change the partial count)
  const GnGeom g = gn_geom<8>(N, HW, G * 8, G);
  return sizeof(float) * 3 * (size_t)N * g.chunks * G;
}

int dp_group_norm_fwd(int dtype, const void* x, const float* gamma, const float* beta, void* y,
                      float* mean, float* rstd, int N, int HW, int C, int G, float eps, int silu,
                      float* workspace, dp_stream_t stream) {
  if (N <= 0 || HW <= 0) return 0;
  if (int e = gn_validate(dtype, C, G)) return e;
  const GnGeom g = gn_geom_rt(dtype, N, HW, C, G);
  dim3 grid(g.chunks, N, g.nblk);
  DISPATCH_T(dtype, launch_k(gn_partial_kernel<T>, dim3(grid), dim3(GN_THREADS), 0, ST, cp<T>(x), HW, C, G, g.ppc, g.CB,
                                                                        workspace));
  DISPATCH_T(dtype, launch_k(gn_apply_kernel<T>, dim3(grid), dim3(GN_THREADS), 0, ST, 
                        cp<T>(x), gamma, beta, mp<T>(y), mean, rstd, workspace, HW, C, G, g.ppc, g.CB,
                        eps, silu, static_cast<const float*>(nullptr)));
  return ew_check("group_norm_fwd");
}

int dp_group_norm_fwd_sums(int dtype, const void* x, const float* gamma, const float* beta, void* y,
                           float* mean, float* rstd, int N, int HW, int C, int G, float eps, int silu,
                           const float* sums, dp_stream_t stream) {
  if (N <= 0 || HW <= 0) return 0;
  if (int e = gn_validate(dtype, C, G)) return e;
  if (!sums) {
    set_error("group_norm_fwd_sums: statistics required");
    return DP_ERR_ARGS;
  }
  const GnGeom g = gn_geom_rt(dtype, N, HW, C, G);
  dim3 grid(g.chunks, N, g.nblk);
  DISPATCH_T(dtype, launch_k(gn_apply_kernel<T>, dim3(grid), dim3(GN_THREADS), 0, ST,
                        cp<T>(x), gamma, beta, mp<T>(y), mean, rstd, static_cast<const float*>(nullptr), HW, C, G,
                        g.ppc, g.CB, eps, silu, sums));
  return ew_check("group_norm_fwd_sums");
}

int dp_group_norm_bwd(int dtype, const void* x, const void* dy, const float* gamma,
                      const float* beta, const float* mean, const float* rstd, void* dx,
                      float* dgamma, float* dbeta, int N, int HW, int C, int G, int silu,
                      int accumulate, float* workspace, dp_stream_t stream) {
  if (N <= 0 || HW <= 0) return 0;
  if (int e = gn_validate(dtype, C, G)) return e;
  const GnGeom g = gn_geom_rt(dtype, N, HW, C, G);
  dim3 grid(g.chunks, N, g.nblk);
  DISPATCH_T(dtype, launch_k(gn_bwd_partial_kernel<T>, dim3(grid), dim3(GN_THREADS), 0, ST, 
                        cp<T>(x), cp<T>(dy), gamma, beta, mean, rstd, HW, C, G, g.ppc, g.CB, silu,
                        dgamma, dbeta, workspace));
  DISPATCH_T(dtype, launch_k(gn_bwd_apply_kernel<T>, dim3(grid), dim3(GN_THREADS), 0, ST, 
                        cp<T>(x), cp<T>(dy), gamma, beta, mean, rstd, workspace, HW, C, G, g.ppc, g.CB,
                        silu, mp<T>(dx), accumulate));
  return ew_check("group_norm_bwd");
}

#define LN_PER_DISPATCH(C, KERNEL, ...)                                               \
  do {                                                                                \
    const int nvec = ((C) / NV<T>::V + 31) / 32;                                      \
    if (nvec <= 1) {                                                                  \
      launch_k(KERNEL<T, 1>, dim3(grid), dim3(256), 0, ST, __VA_ARGS__);                                \
    } else if (nvec <= 2) {                                                           \
      launch_k(KERNEL<T, 2>, dim3(grid), dim3(256), 0, ST, __VA_ARGS__);                                \
    } else if (nvec <= 4) {                                                           \
      launch_k(KERNEL<T, 4>, dim3(grid), dim3(256), 0, ST, __VA_ARGS__);                                \
    } else if (nvec <= 8) {                                                           \
      launch_k(KERNEL<T, 8>, dim3(grid), dim3(256), 0, ST, __VA_ARGS__);                                \
    } else {                                                                          \
      launch_k(KERNEL<T, 16>, dim3(grid), dim3(256), 0, ST, __VA_ARGS__);                               \
    }                                                                                 \
  } while (0)

// resident 256-thread blocks per SM of a kernel (cached per function pointer)
static int ln_blocks_per_sm(const void* kern) {
  static const void* keys[32];
  static int vals[32];
  static int n = 0;
  for (int i = 0; i < n; ++i)
    if (keys[i] == kern) return vals[i];
  int v = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, kern, 256, 0) != cudaSuccess || v < 1) v = 1;
  if (n < 32) {
    keys[n] = kern;
    vals[n++] = v;
  }
  return v;
}

// resident 128-thread blocks per SM (the row-group backward)
static int ln_blocks_per_sm128(const void* kern) {
  static const void* keys[16];
  static int vals[16];
  static int n = 0;
  for (int i = 0; i < n; ++i)
    if (keys[i] == kern) return vals[i];
  int v = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, kern, 128, 0) != cudaSuccess || v < 1) v = 1;
  if (n < 16) {
    keys[n] = kern;
    vals[n++] = v;
  }
  return v;
}

int dp_layer_norm_fwd(int dtype, const void* x, const float* gamma, const float* beta,
                      const void* mod, int64_t mod_ld, int shift_off, int scale_off,
                      int rows_per_sample, void* y, float* mean, float* rstd, int64_t rows, int C,
                      float eps, dp_stream_t stream) {
  if (rows <= 0) return 0;
  if (C > 2048 || (gamma && mod) || C % (dtype == DP_F32 ? 4 : 8) ||
      (reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(y) | reinterpret_cast<uintptr_t>(gamma) |
       reinterpret_cast<uintptr_t>(beta)) % 16) {
    set_error("layer_norm: C <= 2048, C % 8 == 0 (bf16) / 4 (fp32), 16-byte aligned rows, "
              "affine and modulation exclusive");
    return DP_ERR_ARGS;
  }
  if (dtype == DP_BF16 && !mod && lnq_enabled()) {
    int nv = 0;
    const int plan = lnq_plan(C, nv);
    // full-warp rows (C >= 1024): the warp-per-row forward measured as fast or faster (tools/ln_bench.py)
    if (plan && plan - 1 < 5) {
      const int l = plan - 1;
      const int64_t groups = (rows + (32 >> l) - 1) / (32 >> l);
      const void* kern = nv == 4 ? (const void*)lnq_fwd_kernel<4> : nv == 5 ? (const void*)lnq_fwd_kernel<5>
                                                                           : (const void*)lnq_fwd_kernel<8>;
      const int64_t want = (groups + 7) / 8;
      static const bool full = getenv("DP_LNQ_FULLGRID") != nullptr;  // experiments: one block per 8 row groups
      const int64_t cap = full ? want : (int64_t)ln_blocks_per_sm(kern) * kNumSMs;
      const dim3 grid(static_cast<unsigned>(want < cap ? want : cap));
      auto go = [&](auto k) {
        launch_k(k, grid, dim3(256), 0, ST, cp<__nv_bfloat16>(x), gamma, beta, mp<__nv_bfloat16>(y), mean, rstd,
                 rows, C, l, eps);
      };
      if (nv == 4) go(lnq_fwd_kernel<4>);
      else if (nv == 5) go(lnq_fwd_kernel<5>);
      else go(lnq_fwd_kernel<8>);
      return ew_check("layer_norm_fwd");
    }
  }
  const int64_t want = (rows + 7) / 8;
  static const bool one_block_per_8_rows = getenv("DP_LN_FWD_BLOCKS") != nullptr;  // A/B experiments
  DISPATCH_T(dtype, {
    const int nvec = (C / NV<T>::V + 31) / 32;
    const void* kern = nvec <= 1   ? (const void*)ln_fwd_kernel<T, 1>
                       : nvec <= 2 ? (const void*)ln_fwd_kernel<T, 2>
                       : nvec <= 4 ? (const void*)ln_fwd_kernel<T, 4>
                       : nvec <= 8 ? (const void*)ln_fwd_kernel<T, 8>
                                   : (const void*)ln_fwd_kernel<T, 16>;
    const int64_t cap = one_block_per_8_rows ? want : (int64_t)ln_blocks_per_sm(kern) * kNumSMs;
    const dim3 grid(static_cast<unsigned>(want < cap ? want : cap));
    LN_PER_DISPATCH(C, ln_fwd_kernel, cp<T>(x), gamma, beta, cp<T>(mod), mod_ld, shift_off, scale_off,
                    rows_per_sample > 0 ? rows_per_sample : 1, mp<T>(y), mean, rstd, rows, C, eps);
  });
  return ew_check("layer_norm_fwd");
}

int dp_rms_norm_fwd(int dtype, const void* x, const float* gamma, void* y, int64_t rows, int C,
                    float eps, dp_stream_t stream) {
  if (rows <= 0) return 0;
  const int V = dtype == DP_F32 ? 4 : 8;
  if (C % V || C > 32 * 8 * V || reinterpret_cast<uintptr_t>(gamma) % 16) {
    set_error("rms_norm: need C % 8 == 0 (bf16) / 4 (fp32), C <= 256 vectors, 16-byte aligned gamma");
    return DP_ERR_ARGS;
  }
  dim3 grid(static_cast<unsigned>((rows + 7) / 8));
  DISPATCH_T(dtype, LN_PER_DISPATCH(C, rms_fwd_kernel, cp<T>(x), gamma, mp<T>(y), rows, C, eps));
  return ew_check("rms_norm_fwd");
}

int dp_layer_norm_bwd(int dtype, const void* x, const void* dy, const float* gamma,
                      const void* mod, int64_t mod_ld, int shift_off, int scale_off,
                      int rows_per_sample, const float* mean, const float* rstd, void* dx,
                      float* dgamma, float* dbeta, void* dmod, int64_t dmod_ld, int64_t rows,
                      int C, int accumulate, dp_stream_t stream) {
  if (rows <= 0) return 0;
  if (C > 2048 || (gamma && mod) || C % (dtype == DP_F32 ? 4 : 8) ||
      (reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(dy) | reinterpret_cast<uintptr_t>(dx) |
       reinterpret_cast<uintptr_t>(gamma)) % 16) {
    set_error("layer_norm: C <= 2048, C % 8 == 0 (bf16) / 4 (fp32), 16-byte aligned rows, "
              "affine and modulation exclusive");
    return DP_ERR_ARGS;
  }
  if (dtype == DP_BF16 && !mod && lnq_enabled()) {
    int nv = 0;
    const int plan = lnq_plan(C, nv);
    if (plan) {
      const int l = plan - 1;
      // parameter grads: a separate vectorised pass by default (the fused per-lane partials take ~80
      // registers and halve the row kernel's occupancy; DP_LNQ_PG=1: fused, experiments)
      static const bool fuse_pg = [] {
        const char* e = getenv("DP_LNQ_PG");
        return e && atoi(e) != 0;
      }();
      const bool pgq = gamma && dgamma && fuse_pg;
      if (pgq && nv > 5) goto warp_rows;  // the fused parameter partials would spill: warp-per-row kernels
      const int64_t groups = (rows + (32 >> l) - 1) / (32 >> l);
      const int64_t want = (groups + 3) / 4;
      auto go = [&](auto k) {
        static const bool full = getenv("DP_LNQ_FULLGRID") != nullptr;
        const int64_t cap = full ? want : (int64_t)ln_blocks_per_sm128(reinterpret_cast<const void*>(k)) * kNumSMs;
        launch_k(k, dim3(static_cast<unsigned>(want < cap ? want : cap)), dim3(128), 0, ST, cp<__nv_bfloat16>(x),
                 cp<__nv_bfloat16>(dy), gamma, mean, rstd, mp<__nv_bfloat16>(dx), rows, C, l, accumulate, dgamma,
                 dbeta);
      };
      if (pgq) {
        if (nv == 4) go(lnq_bwd_kernel<4, true>);
        else go(lnq_bwd_kernel<5, true>);
        return ew_check("layer_norm_bwd");
      }
      if (nv == 4) go(lnq_bwd_kernel<4, false>);
      else if (nv == 5) go(lnq_bwd_kernel<5, false>);
      else go(lnq_bwd_kernel<8, false>);
      if (gamma && dgamma) {
        const int CVn = C / 8;
        const int cvb = ln_pg_cvb(CVn);
        const int64_t cb = CVn / cvb;
        int64_t seg = (rows * cb + 2 * kNumSMs - 1) / (2 * kNumSMs);  // ~2 waves
        seg = seg < 64 ? 64 : seg;
        dim3 g2(static_cast<unsigned>(cb), static_cast<unsigned>((rows + seg - 1) / seg));
        launch_k(ln_param_grad_kernel<__nv_bfloat16>, dim3(g2), dim3(256), 0, ST, cp<__nv_bfloat16>(x),
                 cp<__nv_bfloat16>(dy), mean, rstd, rows, C, static_cast<int>(seg), dgamma, dbeta,
                 static_cast<__nv_bfloat16*>(nullptr), (int64_t)0, 0, 0, cvb);
      }
      return ew_check("layer_norm_bwd");
    }
  }
warp_rows:
  const int rps = rows_per_sample > 0 ? rows_per_sample : 1;
  const int nvec = (C / (dtype == DP_F32 ? 4 : 8) + 31) / 32;
  // affine parameter grads fused into the row pass while the per-lane partials fit in registers
  // (C <= 1024 bf16): few fat blocks, each merging its rows' partials once
  const bool pg = gamma && dgamma && nvec <= 4;
  const int64_t want = (rows + 7) / 8;
#define LN_BWD_ARGS cp<T>(x), cp<T>(dy), gamma, cp<T>(mod), mod_ld, scale_off, rps, mean, rstd, mp<T>(dx), \
                    rows, C, accumulate, dgamma, dbeta
  // grid = one wave of the instantiation's resident blocks (register-limited: the wide-row variants
  // fit one 256-thread block per SM, and a second partial wave doubled their time); warps stride
  // over the remaining rows
  DISPATCH_T(dtype, {
    auto go = [&](auto kern) {
      const int64_t cap = (int64_t)ln_blocks_per_sm(reinterpret_cast<const void*>(kern)) * kNumSMs;
      launch_k(kern, dim3(static_cast<unsigned>(want < cap ? want : cap)), dim3(256), 0, ST, LN_BWD_ARGS);
    };
    if (pg) {
      if (nvec <= 1) go(ln_bwd_kernel<T, 1, true>);
      else if (nvec <= 2) go(ln_bwd_kernel<T, 2, true>);
      else go(ln_bwd_kernel<T, 4, true>);
    } else {
      if (nvec <= 1) go(ln_bwd_kernel<T, 1, false>);
      else if (nvec <= 2) go(ln_bwd_kernel<T, 2, false>);
      else if (nvec <= 4) go(ln_bwd_kernel<T, 4, false>);
      else if (nvec <= 8) go(ln_bwd_kernel<T, 8, false>);
      else go(ln_bwd_kernel<T, 16, false>);
    }
  });
#undef LN_BWD_ARGS
  if (gamma && dgamma && !pg) {
    const int CVn = C / (dtype == DP_F32 ? 4 : 8);
    const int cvb = ln_pg_cvb(CVn);
    const int64_t cb = CVn / cvb;
    int64_t seg = (rows * cb + 2 * kNumSMs - 1) / (2 * kNumSMs);  // ~2 waves
    seg = seg < 64 ? 64 : seg;
    dim3 g2(static_cast<unsigned>(cb), static_cast<unsigned>((rows + seg - 1) / seg));
    DISPATCH_T(dtype, launch_k(ln_param_grad_kernel<T>, dim3(g2), dim3(256), 0, ST, 
                          cp<T>(x), cp<T>(dy), mean, rstd, rows, C, seg, dgamma, dbeta, nullptr, 0,
                          0, 0, cvb));
  }
  if (mod && dmod) {
    const int CVn = C / (dtype == DP_F32 ? 4 : 8);
    const int cvb = ln_pg_cvb(CVn);
    dim3 g2(static_cast<unsigned>(CVn / cvb), static_cast<unsigned>(rows / rps));
    DISPATCH_T(dtype, launch_k(ln_param_grad_kernel<T>, dim3(g2), dim3(256), 0, ST, 
                          cp<T>(x), cp<T>(dy), mean, rstd, rows, C, rps, nullptr, nullptr,
                          mp<T>(dmod), dmod_ld, shift_off, scale_off, cvb));
  }
  return ew_check("layer_norm_bwd");
}

int dp_softmax_fwd(int dtype, const float* S, void* P, int64_t rows, int cols, int ld,
                   float scale, int causal, int Lq, dp_stream_t stream) {
  if (rows <= 0) return 0;
  const dim3 grid(static_cast<unsigned>((rows + 7) / 8));
  DISPATCH_T(dtype, launch_k(softmax_fwd_kernel<T>, dim3(grid), dim3(256), 0, ST, S, mp<T>(P), rows, cols, ld, scale,
                                                                  causal, Lq > 0 ? Lq : 1));
  return ew_check("softmax_fwd");
}

int dp_softmax_bwd(int dtype, const void* P, const float* dP, void* dS, int64_t rows, int cols,
                   int ld, float scale, dp_stream_t stream) {
  if (rows <= 0) return 0;
  const dim3 grid(static_cast<unsigned>((rows + 7) / 8));
  DISPATCH_T(dtype, launch_k(softmax_bwd_kernel<T>, dim3(grid), dim3(256), 0, ST, cp<T>(P), dP, mp<T>(dS), rows,
                                                                  cols, ld, scale));
  return ew_check("softmax_bwd");
}

}  // extern "C"
