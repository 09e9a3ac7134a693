// Memory-bound elementwise kernels of the training step (K7 in SURVEY §2.4):
// activations (GELU erf/tanh, SiLU) and their gradients, GEGLU, gated residual
// (adaLN-Zero), diffusion q_sample, fused MSE loss+gradient, sinusoidal
// timestep embedding, token/position embedding gather, channel concat/split
// (U-Net skip concat, self-conditioning input), nearest 2x upsample and its
// adjoint, dtype cast, and the AdamW update over flat fp32 master buffers.
//
// All kernels are grid-stride loops over 16-byte vectors (8 x bf16 or 4 x fp32)
// with a scalar tail, sized to a multiple of the SM count; arithmetic is fp32.
#include <string>
#include <cstdlib>
#include "common.cuh"
#include "dpipe.h"

namespace dp {
void set_error(const std::string& s);

template <typename T>
struct VecT {
  static constexpr int N = 16 / sizeof(T);
};

template <typename T>
DP_DEV void load_vec(const T* p, float (&f)[VecT<T>::N]) {
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
DP_DEV void store_vec(T* p, const float (&f)[VecT<T>::N]) {
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

static inline int ew_grid(int64_t work) {
  int64_t g = (work + 255) / 256;
  const int64_t cap = (int64_t)kNumSMs * 8;
  return static_cast<int>(g < 1 ? 1 : (g > cap ? cap : g));
}

static inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

int ew_check(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) set_error(std::string(what) + ": " + cudaGetErrorString(e));
  return e;
}

// ------------------------------------------------------------------ activations
DP_DEV float gelu_erf(float x) { return 0.5f * x * (1.f + erff(x * 0.70710678118654752f)); }
DP_DEV float gelu_erf_grad(float x) {
  const float cdf = 0.5f * (1.f + erff(x * 0.70710678118654752f));
  const float pdf = 0.39894228040143268f * __expf(-0.5f * x * x);
  return cdf + x * pdf;
}
DP_DEV float gelu_tanh(float x) {
  const float u = 0.79788456080286536f * (x + 0.044715f * x * x * x);
  return 0.5f * x * (1.f + tanhf(u));
}
DP_DEV float gelu_tanh_grad(float x) {
  const float u = 0.79788456080286536f * (x + 0.044715f * x * x * x);
  const float th = tanhf(u);
  const float du = 0.79788456080286536f * (1.f + 3.f * 0.044715f * x * x);
  return 0.5f * (1.f + th) + 0.5f * x * (1.f - th * th) * du;
}
DP_DEV float silu(float x) { return x / (1.f + __expf(-x)); }
DP_DEV float silu_grad(float x) {
  const float s = 1.f / (1.f + __expf(-x));
  return s * (1.f + x * (1.f - s));
}

DP_DEV float act_f(int op, float x) {
  switch (op) {
    case DP_ACT_GELU: return gelu_erf(x);
    case DP_ACT_GELU_TANH: return gelu_tanh(x);
    case DP_ACT_SILU: return silu(x);
    default: return x;
  }
}
DP_DEV float act_g(int op, float x) {
  switch (op) {
    case DP_ACT_GELU: return gelu_erf_grad(x);
    case DP_ACT_GELU_TANH: return gelu_tanh_grad(x);
    case DP_ACT_SILU: return silu_grad(x);
    default: return 1.f;
  }
}

template <typename T>
__global__ void act_fwd_kernel(int op, const T* __restrict__ x, T* __restrict__ y, int64_t n) {
  DP_PDL_ENTRY();
  constexpr int V = VecT<T>::N;
  const int64_t nv = n / V;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nv;
       i += (int64_t)gridDim.x * blockDim.x) {
    float f[V];
    load_vec(x + i * V, f);
#pragma unroll
    for (int j = 0; j < V; ++j) f[j] = act_f(op, f[j]);
    store_vec(y + i * V, f);
  }
  for (int64_t i = nv * V + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    y[i] = from_f<T>(act_f(op, to_f(x[i])));
}

// dx = dy * act'(x)   (accumulate: dx += ...)
template <typename T>
__global__ void act_bwd_kernel(int op, const T* __restrict__ x, const T* __restrict__ dy,
                               T* __restrict__ dx, int64_t n, int accumulate) {
  DP_PDL_ENTRY();
  constexpr int V = VecT<T>::N;
  const int64_t nv = n / V;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nv;
       i += (int64_t)gridDim.x * blockDim.x) {
    float fx[V], fd[V], fo[V];
    load_vec(x + i * V, fx);
    load_vec(dy + i * V, fd);
    if (accumulate) load_vec(dx + i * V, fo);
#pragma unroll
    for (int j = 0; j < V; ++j) fo[j] = (accumulate ? fo[j] : 0.f) + fd[j] * act_g(op, fx[j]);
    store_vec(dx + i * V, fo);
  }
  for (int64_t i = nv * V + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    float o = to_f(dy[i]) * act_g(op, to_f(x[i]));
    if (accumulate) o += to_f(dx[i]);
    dx[i] = from_f<T>(o);
  }
}

// ------------------------------------------------------------------ GEGLU
// x [rows][2F] = [a | g];  y [rows][F] = a * gelu(g)
template <typename T>
__global__ void geglu_fwd_kernel(const T* __restrict__ x, T* __restrict__ y, int64_t rows, int F) {
  DP_PDL_ENTRY();
  const int64_t n = rows * F;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / F;
    const int c = static_cast<int>(i - r * F);
    const float a = to_f(x[r * 2 * F + c]);
    const float g = to_f(x[r * 2 * F + F + c]);
    y[i] = from_f<T>(a * gelu_erf(g));
  }
}
template <typename T>
__global__ void geglu_bwd_kernel(const T* __restrict__ x, const T* __restrict__ dy,
                                 T* __restrict__ dx, int64_t rows, int F) {
  DP_PDL_ENTRY();
  const int64_t n = rows * F;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / F;
    const int c = static_cast<int>(i - r * F);
    const float a = to_f(x[r * 2 * F + c]);
    const float g = to_f(x[r * 2 * F + F + c]);
    const float d = to_f(dy[i]);
    dx[r * 2 * F + c] = from_f<T>(d * gelu_erf(g));
    dx[r * 2 * F + F + c] = from_f<T>(d * a * gelu_erf_grad(g));
  }
}

// ------------------------------------------------------------------ add / scale
// y = alpha * a + beta * b
template <typename T>
__global__ void axpby_kernel(const T* __restrict__ a, const T* __restrict__ b, T* __restrict__ y,
                             int64_t n, float alpha, float beta) {
  DP_PDL_ENTRY();
  constexpr int V = VecT<T>::N;
  const int64_t nv = n / V;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nv;
       i += (int64_t)gridDim.x * blockDim.x) {
    float fa[V], fb[V];
    load_vec(a + i * V, fa);
    if (b) load_vec(b + i * V, fb);
#pragma unroll
    for (int j = 0; j < V; ++j) fa[j] = alpha * fa[j] + (b ? beta * fb[j] : 0.f);
    store_vec(y + i * V, fa);
  }
  for (int64_t i = nv * V + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    y[i] = from_f<T>(alpha * to_f(a[i]) + (b ? beta * to_f(b[i]) : 0.f));
}

// ------------------------------------------------------------------ gated residual (adaLN-Zero)
// y[r][c] = x[r][c] + g[r / rps][g_off + c] * h[r][c]  ; g has row stride g_ld
template <typename T>
__global__ void gate_res_fwd_kernel(const T* __restrict__ x, const T* __restrict__ g, int64_t g_ld,
                                    const T* __restrict__ h, T* __restrict__ y, int64_t rows, int C,
                                    int rps) {
  DP_PDL_ENTRY();
  const int64_t n = rows * C;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / C;
    const int c = static_cast<int>(i - r * C);
    const float gv = to_f(g[(r / rps) * g_ld + c]);
    y[i] = from_f<T>(to_f(x[i]) + gv * to_f(h[i]));
  }
}
// dh = dy * g ; dg[b][c] = sum_r dy*h  (one block per (b, 32-channel slab); deterministic)
template <typename T>
__global__ void gate_res_bwd_kernel(const T* __restrict__ dy, const T* __restrict__ g, int64_t g_ld,
                                    const T* __restrict__ h, T* __restrict__ dh,
                                    T* __restrict__ dg, int64_t dg_ld, int B, int C, int rps) {
  DP_PDL_ENTRY();
  const int b = blockIdx.y;
  const int c = blockIdx.x * 32 + (threadIdx.x & 31);
  const int ry = threadIdx.x >> 5;  // 8 row lanes
  __shared__ float red[8][33];
  float acc = 0.f;
  if (c < C) {
    const float gv = to_f(g[(int64_t)b * g_ld + c]);
    for (int r = ry; r < rps; r += 8) {
      const int64_t idx = ((int64_t)b * rps + r) * C + c;
      const float d = to_f(dy[idx]);
      acc += d * to_f(h[idx]);
      dh[idx] = from_f<T>(d * gv);
    }
  }
  red[ry][threadIdx.x & 31] = acc;
  __syncthreads();
  if (ry == 0 && c < C) {
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += red[k][threadIdx.x];
    dg[(int64_t)b * dg_ld + c] = from_f<T>(s);
  }
}

// ------------------------------------------------------------------ diffusion
// x_t = sqrt_ab[t_b] * x0 + sqrt_1mab[t_b] * noise ; per_sample elements per sample
template <typename T>
__global__ void q_sample_kernel(const T* __restrict__ x0, const T* __restrict__ noise,
                                const int64_t* __restrict__ t, const float* __restrict__ sab,
                                const float* __restrict__ s1mab, T* __restrict__ xt, int64_t n,
                                int64_t per_sample) {
  DP_PDL_ENTRY();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t ts = t[i / per_sample];
    xt[i] = from_f<T>(sab[ts] * to_f(x0[i]) + s1mab[ts] * to_f(noise[i]));
  }
}

// x0_hat = (x_t - sqrt(1-ab) * eps) / sqrt(ab)   (self-conditioning estimate)
template <typename T>
__global__ void pred_x0_kernel(const T* __restrict__ xt, const T* __restrict__ eps,
                               const int64_t* __restrict__ t, const float* __restrict__ sab,
                               const float* __restrict__ s1mab, T* __restrict__ out,
                               int64_t n, int64_t per_sample) {
  DP_PDL_ENTRY();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t ts = t[i / per_sample];
    out[i] = from_f<T>((to_f(xt[i]) - s1mab[ts] * to_f(eps[i])) / sab[ts]);
  }
}

// loss_acc[0] += scale * sum (p - y)^2 ; dp = 2*scale*(p - y)
template <typename T>
__global__ void mse_kernel(const T* __restrict__ p, const T* __restrict__ y, T* __restrict__ dp,
                           float* __restrict__ loss, int64_t n, float scale) {
  DP_PDL_ENTRY();
  float acc = 0.f;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const float d = to_f(p[i]) - to_f(y[i]);
    acc += d * d;
    if (dp) dp[i] = from_f<T>(2.f * scale * d);
  }
  acc = warp_sum(acc);
  __shared__ float red[32];
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x < 32) {
    float v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.f;
    v = warp_sum(v);
    if (threadIdx.x == 0) atomicAdd(loss, v * scale);
  }
}

// out[b][i] = cos(t_b * f_i), out[b][half + i] = sin(t_b * f_i), f_i = exp(-ln(max_period) i / half)
// (the SD/DiT "flip_sin_to_cos" convention: cos first)
template <typename T>
__global__ void timestep_embed_kernel(const int64_t* __restrict__ t, T* __restrict__ out, int B,
                                      int dim, float max_period) {
  DP_PDL_ENTRY();
  const int half = dim / 2;
  const int64_t n = (int64_t)B * half;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int b = static_cast<int>(i / half);
    const int k = static_cast<int>(i - (int64_t)b * half);
    const float freq = expf(-logf(max_period) * static_cast<float>(k) / static_cast<float>(half));
    const float arg = static_cast<float>(t[b]) * freq;
    out[(int64_t)b * dim + k] = from_f<T>(cosf(arg));
    out[(int64_t)b * dim + half + k] = from_f<T>(sinf(arg));
  }
}

// out[r][c] = table[ids[r]][c] + (pos ? pos[r % L][c] : 0)
template <typename T>
__global__ void embed_kernel(const int64_t* __restrict__ ids, const T* __restrict__ table,
                             const T* __restrict__ pos, T* __restrict__ out, int64_t rows, int L,
                             int C) {
  DP_PDL_ENTRY();
  const int64_t n = rows * C;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / C;
    const int c = static_cast<int>(i - r * C);
    float v = to_f(table[ids[r] * C + c]);
    if (pos) v += to_f(pos[(r % L) * C + c]);
    out[i] = from_f<T>(v);
  }
}

// dst[r][0:Ca] = a[r], dst[r][Ca:Ca+Cb] = b[r]   (b may be null -> zeros)
template <typename T>
__global__ void concat_kernel(const T* __restrict__ a, const T* __restrict__ b, T* __restrict__ dst,
                              int64_t rows, int Ca, int Cb) {
  DP_PDL_ENTRY();
  const int C = Ca + Cb;
  const int64_t n = rows * C;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / C;
    const int c = static_cast<int>(i - r * C);
    dst[i] = c < Ca ? a[r * Ca + c] : (b ? b[r * Cb + (c - Ca)] : from_f<T>(0.f));
  }
}
// row-vector variant for narrow unaligned inputs (3 / 4-channel images and latents padded with
// zeros or joined with a channel block): one thread per 16-byte vector of a dst row, gathered from
// a / b element-wise and stored as one vector
template <typename T>
__global__ void concat_rowvec_kernel(const T* __restrict__ a, const T* __restrict__ b, T* __restrict__ dst,
                                     int64_t rows, int Ca, int Cb) {
  DP_PDL_ENTRY();
  constexpr int V = VecT<T>::N;
  const int C = Ca + Cb, CV = C / V;
  const int64_t n = rows * CV;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / CV;
    const int c0 = static_cast<int>(i - r * CV) * V;
    float f[V];
#pragma unroll
    for (int j = 0; j < V; ++j) {
      const int c = c0 + j;
      f[j] = c < Ca ? to_f(a[r * Ca + c]) : (b ? to_f(b[r * Cb + (c - Ca)]) : 0.f);
    }
    store_vec(dst + i * V, f);
  }
}

// a[r] (+)= src[r][0:Ca], b[r] (+)= src[r][Ca:]   (either output may be null)
template <typename T>
__global__ void split_kernel(const T* __restrict__ src, T* __restrict__ a, T* __restrict__ b,
                             int64_t rows, int Ca, int Cb, int acc_a, int acc_b) {
  DP_PDL_ENTRY();
  const int C = Ca + Cb;
  const int64_t n = rows * C;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / C;
    const int c = static_cast<int>(i - r * C);
    const float v = to_f(src[i]);
    if (c < Ca) {
      if (a) {
        T* o = a + r * Ca + c;
        *o = from_f<T>(acc_a ? to_f(*o) + v : v);
      }
    } else if (b) {
      T* o = b + r * Cb + (c - Ca);
      *o = from_f<T>(acc_b ? to_f(*o) + v : v);
    }
  }
}

// NHWC nearest 2x upsample: y[n][2h+i][2w+j][c] = x[n][h][w][c]
template <typename T>
__global__ void upsample2x_kernel(const T* __restrict__ x, T* __restrict__ y, int N, int H, int W,
                                  int C) {
  DP_PDL_ENTRY();
  const int64_t n = (int64_t)N * 2 * H * 2 * W * C;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int c = static_cast<int>(i % C);
    int64_t t = i / C;
    const int w = static_cast<int>(t % (2 * W));
    t /= 2 * W;
    const int h = static_cast<int>(t % (2 * H));
    const int b = static_cast<int>(t / (2 * H));
    y[i] = x[(((int64_t)b * H + h / 2) * W + w / 2) * C + c];
  }
}
template <typename T>
__global__ void upsample2x_bwd_kernel(const T* __restrict__ dy, T* __restrict__ dx, int N, int H,
                                      int W, int C) {
  DP_PDL_ENTRY();
  const int64_t n = (int64_t)N * H * W * C;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int c = static_cast<int>(i % C);
    int64_t t = i / C;
    const int w = static_cast<int>(t % W);
    t /= W;
    const int h = static_cast<int>(t % H);
    const int b = static_cast<int>(t / H);
    const int64_t W2 = 2 * W;
    const int64_t base = (((int64_t)b * 2 * H + 2 * h) * W2 + 2 * w) * C + c;
    dx[i] = from_f<T>(to_f(dy[base]) + to_f(dy[base + C]) + to_f(dy[base + W2 * C]) +
                      to_f(dy[base + W2 * C + C]));
  }
}

// 16-byte channel vectors (C % V == 0): one thread per output pixel-vector of the 2x map, the
// source pixel read once per vector (the scalar kernels above divide per element)
template <typename T>
__global__ void upsample2x_vec_kernel(const T* __restrict__ x, T* __restrict__ y, int N, int H, int W, int C) {
  DP_PDL_ENTRY();
  constexpr int V = VecT<T>::N;
  const int CV = C / V;
  const int64_t n = (int64_t)N * 2 * H * 2 * W * CV;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int cv = static_cast<int>(i % CV);
    const int64_t pix = i / CV;  // (b, h2, w2)
    const int w2 = static_cast<int>(pix % (2 * W));
    const int64_t t = pix / (2 * W);
    const int h2 = static_cast<int>(t % (2 * H));
    const int b = static_cast<int>(t / (2 * H));
    *reinterpret_cast<uint4*>(y + i * V) =
        *reinterpret_cast<const uint4*>(x + (((int64_t)b * H + h2 / 2) * W + w2 / 2) * C + cv * V);
  }
}
template <typename T>
__global__ void upsample2x_bwd_vec_kernel(const T* __restrict__ dy, T* __restrict__ dx, int N, int H, int W,
                                          int C) {
  DP_PDL_ENTRY();
  constexpr int V = VecT<T>::N;
  const int CV = C / V;
  const int64_t n = (int64_t)N * H * W * CV;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int cv = static_cast<int>(i % CV);
    const int64_t pix = i / CV;  // (b, h, w)
    const int w = static_cast<int>(pix % W);
    const int64_t t = pix / W;
    const int h = static_cast<int>(t % H);
    const int b = static_cast<int>(t / H);
    const int64_t W2 = 2 * W;
    const T* s = dy + (((int64_t)b * 2 * H + 2 * h) * W2 + 2 * w) * C + cv * V;
    float a[V], f[V];
    load_vec(s, a);
    load_vec(s + C, f);
#pragma unroll
    for (int j = 0; j < V; ++j) a[j] += f[j];
    load_vec(s + W2 * C, f);
#pragma unroll
    for (int j = 0; j < V; ++j) a[j] += f[j];
    load_vec(s + W2 * C + C, f);
#pragma unroll
    for (int j = 0; j < V; ++j) a[j] += f[j];
    store_vec(dx + i * V, a);
  }
}

template <typename TI, typename TO>
__global__ void cast_kernel(const TI* __restrict__ x, TO* __restrict__ y, int64_t n) {
  DP_PDL_ENTRY();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    y[i] = from_f<TO>(to_f(x[i]));
}

// ------------------------------------------------------------------ AdamW (flat fp32 master)
// decoupled weight decay (torch.optim.AdamW): p -= lr*wd*p; m,v moments; bias-corrected step.
__global__ void adamw_kernel(float* __restrict__ p, const float* __restrict__ g,
                             float* __restrict__ m, float* __restrict__ v,
                             __nv_bfloat16* __restrict__ p_bf16, int64_t n, float lr, float b1,
                             float b2, float eps, float wd, float bc1, float bc2, float gscale,
                             const float* __restrict__ bc_dev, int zero_g) {
  DP_PDL_ENTRY();
  if (bc_dev) {  // bias corrections of a device-side step counter (CUDA-graph replayable)
    bc1 = bc_dev[0];
    bc2 = bc_dev[1];
  }
  const int64_t nv = n / 4;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nv;
       i += (int64_t)gridDim.x * blockDim.x) {
    float4 pp = reinterpret_cast<float4*>(p)[i];
    const float4 gg = reinterpret_cast<const float4*>(g)[i];
    float4 mm = reinterpret_cast<float4*>(m)[i];
    float4 vv = reinterpret_cast<float4*>(v)[i];
    float* pa = &pp.x;
    const float* ga = &gg.x;
    float* ma = &mm.x;
    float* va = &vv.x;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float gj = ga[j] * gscale;
      pa[j] -= lr * wd * pa[j];
      ma[j] = b1 * ma[j] + (1.f - b1) * gj;
      va[j] = b2 * va[j] + (1.f - b2) * gj * gj;
      const float denom = sqrtf(va[j] / bc2) + eps;
      pa[j] -= (lr / bc1) * ma[j] / denom;
    }
    reinterpret_cast<float4*>(p)[i] = pp;
    reinterpret_cast<float4*>(m)[i] = mm;
    reinterpret_cast<float4*>(v)[i] = vv;
    if (zero_g) reinterpret_cast<float4*>(const_cast<float*>(g))[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    if (p_bf16) {
      uint2 o;
      o.x = pack_bf16x2(pa[0], pa[1]);
      o.y = pack_bf16x2(pa[2], pa[3]);
      reinterpret_cast<uint2*>(p_bf16)[i] = o;
    }
  }
  for (int64_t i = nv * 4 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const float gj = g[i] * gscale;
    float pj = p[i];
    pj -= lr * wd * pj;
    const float mj = b1 * m[i] + (1.f - b1) * gj;
    const float vj = b2 * v[i] + (1.f - b2) * gj * gj;
    pj -= (lr / bc1) * mj / (sqrtf(vj / bc2) + eps);
    p[i] = pj;
    m[i] = mj;
    v[i] = vj;
    if (p_bf16) p_bf16[i] = __float2bfloat16_rn(pj);
    if (zero_g) const_cast<float*>(g)[i] = 0.f;
  }
}

// db[c] += sum_r dy[r][c]: grid (ceil(C/32), segments of 512 rows), fp32 atomics per segment
template <typename T>
__global__ void __launch_bounds__(256) bias_grad_kernel(const T* __restrict__ dy, float* __restrict__ db,
                                                        int64_t rows, int C, int seg) {
  DP_PDL_ENTRY();
  const int c = blockIdx.x * 32 + (threadIdx.x & 31);
  const int ry = threadIdx.x >> 5;
  const int64_t r0 = (int64_t)blockIdx.y * seg;
  const int64_t r1 = min(rows, r0 + seg);
  float a = 0.f;
  if (c < C)
    for (int64_t r = r0 + ry; r < r1; r += 8) a += to_f(dy[r * C + c]);
  __shared__ float red[8][33];
  red[ry][threadIdx.x & 31] = a;
  __syncthreads();
  if (ry == 0 && c < C) {
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += red[k][threadIdx.x];
    atomicAdd(db + c, s);
  }
}

// y[r][c] = x[r][c] + e[r / rps][c]  (ResBlock time-embedding add, broadcast over pixels)
template <typename T, bool EV>
__global__ void row_bias_fwd_kernel(const T* __restrict__ x, const T* __restrict__ e, int64_t e_ld,
                                    T* __restrict__ y, int64_t rows, int C, int rps) {
  DP_PDL_ENTRY();
  constexpr int V = VecT<T>::N;
  const int CV = C / V;
  const int64_t n = rows * CV;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / CV;
    const int cv = static_cast<int>(i - r * CV);
    float f[V], g[V];
    load_vec(x + r * C + cv * V, f);
    const T* er = e + (r / rps) * e_ld + cv * V;
    if constexpr (EV) {
      load_vec(er, g);  // 16-byte aligned rows of e (checked by the launcher)
    } else {
#pragma unroll
      for (int j = 0; j < V; ++j) g[j] = to_f(er[j]);
    }
#pragma unroll
    for (int j = 0; j < V; ++j) f[j] += g[j];
    store_vec(y + r * C + cv * V, f);
  }
}
// de[b][c] = sum_{r in sample b} dy[r][c] : grid (ceil(C/32), B), deterministic
template <typename T>
__global__ void __launch_bounds__(256) row_bias_bwd_kernel(const T* __restrict__ dy, T* __restrict__ de,
                                                           int64_t de_ld, int C, int rps, float* __restrict__ db,
                                                           float* __restrict__ db2) {
  DP_PDL_ENTRY();
  const int b = blockIdx.y;
  const int c = blockIdx.x * 32 + (threadIdx.x & 31);
  const int ry = threadIdx.x >> 5;
  float a = 0.f;
  if (c < C)
    for (int r = ry; r < rps; r += 8) a += to_f(dy[((int64_t)b * rps + r) * C + c]);
  __shared__ float red[8][33];
  red[ry][threadIdx.x & 31] = a;
  __syncthreads();
  if (ry == 0 && c < C) {
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += red[k][threadIdx.x];
    de[(int64_t)b * de_ld + c] = from_f<T>(s);
    if (db) atomicAdd(db + c, s);
    if (db2) atomicAdd(db2 + c, s);
  }
}

// de[b][c] = sum_{r in sample b} dy[r][c], 16-byte vectors: block = CVB channel vectors x 256/CVB row
// lanes over one sample's rows (grid (CV/CVB, B)), deterministic (no atomics)
template <typename T>
__global__ void __launch_bounds__(256) row_bias_bwd_vec_kernel(const T* __restrict__ dy, T* __restrict__ de,
                                                               int64_t de_ld, int C, int rps, int CVB,
                                                               float* __restrict__ db, float* __restrict__ db2) {
  DP_PDL_ENTRY();
  constexpr int V = VecT<T>::N;
  const int b = blockIdx.y;
  const int RL = 256 / CVB;
  const int lv = threadIdx.x % CVB, rl = threadIdx.x / CVB;
  const int cv = blockIdx.x * CVB + lv;
  float acc[V];
#pragma unroll
  for (int j = 0; j < V; ++j) acc[j] = 0.f;
  if (rl < RL) {
    const T* p = dy + (int64_t)b * rps * C + cv * V;
    int r = rl;
    for (; r + 3 * RL < rps; r += 4 * RL) {
      float f[4][V];
#pragma unroll
      for (int u = 0; u < 4; ++u) load_vec(p + (int64_t)(r + u * RL) * C, f[u]);
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int j = 0; j < V; ++j) acc[j] += f[u][j];
    }
    for (; r < rps; r += RL) {
      float f[V];
      load_vec(p + (int64_t)r * C, f);
#pragma unroll
      for (int j = 0; j < V; ++j) acc[j] += f[j];
    }
  }
  __shared__ float red[256 * 8];
  if (rl < RL) {
#pragma unroll
    for (int j = 0; j < V; ++j) red[rl * CVB * V + lv * V + j] = acc[j];
  }
  __syncthreads();
  for (int t = threadIdx.x; t < CVB * V; t += 256) {
    float s = 0.f;
    for (int k = 0; k < RL; ++k) s += red[k * CVB * V + t];
    de[(int64_t)b * de_ld + blockIdx.x * CVB * V + t] = from_f<T>(s);
    // the producing conv's bias gradient is the sum of the per-sample sums (fp32, before rounding)
    if (db) atomicAdd(db + blockIdx.x * CVB * V + t, s);
    // ... and, for a temb projection, that linear's bias gradient too (the same sum over every row)
    if (db2) atomicAdd(db2 + blockIdx.x * CVB * V + t, s);
  }
}

// image [N][H][W][C] <-> patches [N][H/p][W/p][(i*p+j)*C + c]
template <typename T>
__global__ void s2d_kernel(const T* __restrict__ x, T* __restrict__ y, int N, int H, int W, int C,
                           int p, int inverse) {
  DP_PDL_ENTRY();
  const int64_t n = (int64_t)N * H * W * C;
  const int h = H / p, w = W / p;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    // i indexes the image layout
    const int c = static_cast<int>(i % C);
    int64_t t = i / C;
    const int xx = static_cast<int>(t % W);
    t /= W;
    const int yy = static_cast<int>(t % H);
    const int b = static_cast<int>(t / H);
    const int64_t j = ((((int64_t)b * h + yy / p) * w + xx / p) * p * p + (yy % p) * p + (xx % p)) * C + c;
    if (inverse)
      y[i] = x[j];
    else
      y[j] = x[i];
  }
}

// ++step; bc = (1 - b1^step, 1 - b2^step)   (one thread; precedes adamw_kernel in the stream)
__global__ void adamw_step_kernel(int* step, float b1, float b2, float* bc) {
  DP_PDL_ENTRY();
  const int s = ++(*step);
  bc[0] = 1.f - powf(b1, static_cast<float>(s));
  bc[1] = 1.f - powf(b2, static_cast<float>(s));
}

// ------------------------------------------------------------------ 16-byte vector variants
// x [rows][2F] = [a | g] -> y [rows][F] = a * gelu(g): one vector of V features per thread
template <typename T>
__global__ void geglu_fwd_vec_kernel(const T* __restrict__ x, T* __restrict__ y, int64_t rows, int F) {
  DP_PDL_ENTRY();
  constexpr int V = VecT<T>::N;
  const int FV = F / V;
  const int64_t n = rows * FV;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / FV;
    const int fv = static_cast<int>(i - r * FV);
    float a[V], g[V];
    load_vec(x + r * 2 * F + fv * V, a);
    load_vec(x + r * 2 * F + F + fv * V, g);
#pragma unroll
    for (int j = 0; j < V; ++j) a[j] *= gelu_erf(g[j]);
    store_vec(y + r * F + fv * V, a);
  }
}
template <typename T>
__global__ void geglu_bwd_vec_kernel(const T* __restrict__ x, const T* __restrict__ dy,
                                     T* __restrict__ dx, int64_t rows, int F) {
  DP_PDL_ENTRY();
  constexpr int V = VecT<T>::N;
  const int FV = F / V;
  const int64_t n = rows * FV;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / FV;
    const int fv = static_cast<int>(i - r * FV);
    float a[V], g[V], d[V], da[V], dg[V];
    load_vec(x + r * 2 * F + fv * V, a);
    load_vec(x + r * 2 * F + F + fv * V, g);
    load_vec(dy + r * F + fv * V, d);
#pragma unroll
    for (int j = 0; j < V; ++j) {
      da[j] = d[j] * gelu_erf(g[j]);
      dg[j] = d[j] * a[j] * gelu_erf_grad(g[j]);
    }
    store_vec(dx + r * 2 * F + fv * V, da);
    store_vec(dx + r * 2 * F + F + fv * V, dg);
  }
}

// GEGLU backward fused with the bias gradient of the projection that produced x (the FF input
// projection ff1): db[0..2F) += column sums of dx = [da | dg]. Block = CVB vectors of the F half x
// 256/CVB row lanes over one row segment (grid (FV/CVB, segments)), two rows' loads in flight per
// thread, one fp32 atomic per column and block. Replaces the separate bias-gradient pass that
// re-read dx (2F columns) from HBM.
template <typename T>
__global__ void __launch_bounds__(256) geglu_bwd_bias_kernel(const T* __restrict__ x, const T* __restrict__ dy,
                                                             T* __restrict__ dx, float* __restrict__ db,
                                                             int64_t rows, int F, int CVB, int64_t seg) {
  DP_PDL_ENTRY();
  constexpr int V = VecT<T>::N;
  const int RL = 256 / CVB;
  const int lv = threadIdx.x % CVB, rl = threadIdx.x / CVB;
  const int cv = blockIdx.x * CVB + lv;
  const int64_t r0 = (int64_t)blockIdx.y * seg;
  const int64_t r1 = min(rows, r0 + seg);
  float sa[V], sg[V];
#pragma unroll
  for (int j = 0; j < V; ++j) sa[j] = sg[j] = 0.f;
  auto row = [&](int64_t r, const float (&a)[V], const float (&g)[V], const float (&d)[V]) {
    float da[V], dg[V];
#pragma unroll
    for (int j = 0; j < V; ++j) {
      da[j] = d[j] * gelu_erf(g[j]);
      dg[j] = d[j] * a[j] * gelu_erf_grad(g[j]);
    }
    store_vec(dx + r * 2 * F + cv * V, da);
    store_vec(dx + r * 2 * F + F + cv * V, dg);
    // the bias gradient sums what the consumer reads: the rounded stored values
#pragma unroll
    for (int j = 0; j < V; ++j) {
      sa[j] += to_f(from_f<T>(da[j]));
      sg[j] += to_f(from_f<T>(dg[j]));
    }
  };
  if (rl < RL) {
    int64_t r = r0 + rl;
    for (; r + RL < r1; r += 2 * RL) {
      float a0[V], g0[V], d0[V], a1[V], g1[V], d1[V];
      load_vec(x + r * 2 * F + cv * V, a0);
      load_vec(x + r * 2 * F + F + cv * V, g0);
      load_vec(dy + r * F + cv * V, d0);
      load_vec(x + (r + RL) * 2 * F + cv * V, a1);
      load_vec(x + (r + RL) * 2 * F + F + cv * V, g1);
      load_vec(dy + (r + RL) * F + cv * V, d1);
      row(r, a0, g0, d0);
      row(r + RL, a1, g1, d1);
    }
    for (; r < r1; r += RL) {
      float a0[V], g0[V], d0[V];
      load_vec(x + r * 2 * F + cv * V, a0);
      load_vec(x + r * 2 * F + F + cv * V, g0);
      load_vec(dy + r * F + cv * V, d0);
      row(r, a0, g0, d0);
    }
  }
  __shared__ float red[2][256 * 8];
  if (rl < RL) {
#pragma unroll
    for (int j = 0; j < V; ++j) {
      red[0][rl * CVB * V + lv * V + j] = sa[j];
      red[1][rl * CVB * V + lv * V + j] = sg[j];
    }
  }
  __syncthreads();
  for (int t = threadIdx.x; t < 2 * CVB * V; t += 256) {
    const int h = t / (CVB * V), u = t - h * (CVB * V);
    float s = 0.f;
    for (int k = 0; k < RL; ++k) s += red[h][k * CVB * V + u];
    atomicAdd(db + h * F + blockIdx.x * CVB * V + u, s);
  }
}

template <typename T>
__global__ void concat_vec_kernel(const T* __restrict__ a, const T* __restrict__ b, T* __restrict__ dst,
                                  int64_t rows, int Ca, int Cb) {
  DP_PDL_ENTRY();
  constexpr int V = VecT<T>::N;
  const int CVa = Ca / V, CV = (Ca + Cb) / V, CVb = Cb / V;
  const int64_t n = rows * CV;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / CV;
    const int cv = static_cast<int>(i - r * CV);
    uint4 u = make_uint4(0, 0, 0, 0);
    if (cv < CVa)
      u = *reinterpret_cast<const uint4*>(a + (r * CVa + cv) * V);
    else if (b)
      u = *reinterpret_cast<const uint4*>(b + (r * CVb + cv - CVa) * V);
    *reinterpret_cast<uint4*>(dst + i * V) = u;
  }
}

template <typename T>
__global__ void split_vec_kernel(const T* __restrict__ src, T* __restrict__ a, T* __restrict__ b,
                                 int64_t rows, int Ca, int Cb, int acc_a, int acc_b) {
  DP_PDL_ENTRY();
  constexpr int V = VecT<T>::N;
  const int CVa = Ca / V, CV = (Ca + Cb) / V, CVb = Cb / V;
  const int64_t n = rows * CV;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / CV;
    const int cv = static_cast<int>(i - r * CV);
    T* o;
    int acc;
    if (cv < CVa) {
      o = a ? a + (r * CVa + cv) * V : nullptr;
      acc = acc_a;
    } else {
      o = b ? b + (r * CVb + cv - CVa) * V : nullptr;
      acc = acc_b;
    }
    if (!o) continue;
    if (acc) {
      float s[V], t[V];
      load_vec(src + i * V, s);
      load_vec(o, t);
#pragma unroll
      for (int j = 0; j < V; ++j) s[j] += t[j];
      store_vec(o, s);
    } else {
      *reinterpret_cast<uint4*>(o) = *reinterpret_cast<const uint4*>(src + i * V);
    }
  }
}

// db[c] += sum_r dy[r][c] with 16-byte loads: block = 32 channel vectors x 8 row lanes
template <typename T>
__global__ void __launch_bounds__(256) bias_grad_vec_kernel(const T* __restrict__ dy, float* __restrict__ db,
                                                            int64_t rows, int C, int seg) {
  DP_PDL_ENTRY();
  constexpr int V = VecT<T>::N;
  const int CV = C / V;
  const int cv = blockIdx.x * 32 + (threadIdx.x & 31);
  const int ry = threadIdx.x >> 5;
  const int64_t r0 = (int64_t)blockIdx.y * seg;
  const int64_t r1 = min(rows, r0 + seg);
  float acc[V];
#pragma unroll
  for (int j = 0; j < V; ++j) acc[j] = 0.f;
  if (cv < CV) {
#pragma unroll 4
    for (int64_t r = r0 + ry; r < r1; r += 8) {
      float f[V];
      load_vec(dy + r * C + cv * V, f);
#pragma unroll
      for (int j = 0; j < V; ++j) acc[j] += f[j];
    }
  }
  __shared__ float red[8][32 * 8 + 1];
#pragma unroll
  for (int j = 0; j < V; ++j) red[ry][(threadIdx.x & 31) * V + j] = acc[j];
  __syncthreads();
  for (int t = threadIdx.x; t < 32 * V; t += 256) {
    const int c = blockIdx.x * 32 * V + t;
    if (c < C) {
      float s = 0.f;
#pragma unroll
      for (int k = 0; k < 8; ++k) s += red[k][t];
      atomicAdd(db + c, s);
    }
  }
}

// db[c] += sum_r dy[r][c], block = CVB channel vectors (all of a row when C <= 256 vectors) x
// 256/CVB row lanes: no idle lanes for C = 320 / 640 / 1280 (the 32-vector blocks above left
// 3/4 of a block idle at C = 320); 4 rows' loads in flight per thread
template <typename T>
__global__ void __launch_bounds__(256) bias_grad_rows_kernel(const T* __restrict__ dy, float* __restrict__ db,
                                                             int64_t rows, int C, int CVB, int seg) {
  DP_PDL_ENTRY();
  constexpr int V = VecT<T>::N;
  const int CV = C / V;
  const int RL = 256 / CVB;
  const int lane_v = threadIdx.x % CVB, rl = threadIdx.x / CVB;
  const int cv = blockIdx.x * CVB + lane_v;
  const int64_t r0 = (int64_t)blockIdx.y * seg;
  const int64_t r1 = min(rows, r0 + seg);
  float acc[V];
#pragma unroll
  for (int j = 0; j < V; ++j) acc[j] = 0.f;
  if (rl < RL && cv < CV) {
    const T* p = dy + cv * V;
    int64_t r = r0 + rl;
    for (; r + 3 * RL < r1; r += 4 * RL) {
      float f[4][V];
#pragma unroll
      for (int u = 0; u < 4; ++u) load_vec(p + (r + u * RL) * C, f[u]);
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int j = 0; j < V; ++j) acc[j] += f[u][j];
    }
    for (; r < r1; r += RL) {
      float f[V];
      load_vec(p + r * C, f);
#pragma unroll
      for (int j = 0; j < V; ++j) acc[j] += f[j];
    }
  }
  __shared__ float red[256 * 8];
  if (rl < RL) {
#pragma unroll
    for (int j = 0; j < V; ++j) red[rl * CVB * V + lane_v * V + j] = acc[j];
  }
  __syncthreads();
  for (int t = threadIdx.x; t < CVB * V; t += 256) {
    const int c = blockIdx.x * CVB * V + t;
    if (c < C) {
      float s = 0.f;
      for (int k = 0; k < RL; ++k) s += red[k * CVB * V + t];
      atomicAdd(db + c, s);
    }
  }
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

template <typename T>
static const T* cp(const void* p) {
  return reinterpret_cast<const T*>(p);
}
template <typename T>
static T* mp(void* p) {
  return reinterpret_cast<T*>(p);
}
#define ST reinterpret_cast<cudaStream_t>(stream)

extern "C" {

int dp_act_fwd(int op, int dtype, const void* x, void* y, int64_t n, dp_stream_t stream) {
  if (n <= 0) return 0;
  if (!aligned16(x) || !aligned16(y)) {
    set_error("dp_act_fwd: pointers must be 16-byte aligned");
    return DP_ERR_ARGS;
  }
  DISPATCH_T(dtype, launch_k(act_fwd_kernel<T>, dim3(ew_grid(n / VecT<T>::N + 1)), dim3(256), 0, ST,
                             op, cp<T>(x), mp<T>(y), n));
  return ew_check("act_fwd");
}

int dp_act_bwd(int op, int dtype, const void* x, const void* dy, void* dx, int64_t n,
               int accumulate, dp_stream_t stream) {
  if (n <= 0) return 0;
  if (!aligned16(x) || !aligned16(dy) || !aligned16(dx)) {
    set_error("dp_act_bwd: pointers must be 16-byte aligned");
    return DP_ERR_ARGS;
  }
  DISPATCH_T(dtype, launch_k(act_bwd_kernel<T>, dim3(ew_grid(n / VecT<T>::N + 1)), dim3(256), 0, ST,
                             op, cp<T>(x), cp<T>(dy), mp<T>(dx), n, accumulate));
  return ew_check("act_bwd");
}

int dp_geglu_fwd(int dtype, const void* x, void* y, int64_t rows, int F, dp_stream_t stream) {
  if (rows <= 0) return 0;
  const int V = dtype == DP_F32 ? 4 : 8;
  if (F % V == 0 && aligned16(x) && aligned16(y)) {
    DISPATCH_T(dtype, launch_k(geglu_fwd_vec_kernel<T>, dim3(ew_grid(rows * F / V)), dim3(256), 0, ST, 
                          cp<T>(x), mp<T>(y), rows, F));
    return ew_check("geglu_fwd");
  }
  DISPATCH_T(dtype, launch_k(geglu_fwd_kernel<T>, dim3(ew_grid(rows * F)), dim3(256), 0, ST, cp<T>(x), mp<T>(y),
                                                                             rows, F));
  return ew_check("geglu_fwd");
}

int dp_geglu_bwd_db(int dtype, const void* x, const void* dy, void* dx, int64_t rows, int F, float* db,
                    dp_stream_t stream) {
  if (rows <= 0) return 0;
  const int V = dtype == DP_F32 ? 4 : 8;
  if (!db) return dp_geglu_bwd(dtype, x, dy, dx, rows, F, stream);
  if (F % V || !aligned16(x) || !aligned16(dy) || !aligned16(dx)) {
    set_error("dp_geglu_bwd_db: F must be a multiple of the 16-byte vector and the rows 16-byte aligned");
    return DP_ERR_ARGS;
  }
  const int FV = F / V;
  int CVB = 1;
  for (int d = 32; d >= 1; --d)
    if (FV % d == 0) {
      CVB = d;
      break;
    }
  // ~2 blocks per SM over (channel blocks x row segments): few atomics per column
  const int64_t want = 2 * kNumSMs / (FV / CVB) > 0 ? 2 * kNumSMs / (FV / CVB) : 1;
  int64_t seg = (rows + want - 1) / want;
  if (seg < 2 * (256 / CVB)) seg = 2 * (256 / CVB);
  dim3 grid(FV / CVB, static_cast<unsigned>((rows + seg - 1) / seg));
  DISPATCH_T(dtype, launch_k(geglu_bwd_bias_kernel<T>, dim3(grid), dim3(256), 0, ST, cp<T>(x), cp<T>(dy),
                             mp<T>(dx), db, rows, F, CVB, seg));
  return ew_check("geglu_bwd_db");
}

int dp_geglu_bwd(int dtype, const void* x, const void* dy, void* dx, int64_t rows, int F,
                 dp_stream_t stream) {
  if (rows <= 0) return 0;
  const int V = dtype == DP_F32 ? 4 : 8;
  if (F % V == 0 && aligned16(x) && aligned16(dy) && aligned16(dx)) {
    DISPATCH_T(dtype, launch_k(geglu_bwd_vec_kernel<T>, dim3(ew_grid(rows * F / V)), dim3(256), 0, ST, 
                          cp<T>(x), cp<T>(dy), mp<T>(dx), rows, F));
    return ew_check("geglu_bwd");
  }
  DISPATCH_T(dtype, launch_k(geglu_bwd_kernel<T>, dim3(ew_grid(rows * F)), dim3(256), 0, ST, 
                        cp<T>(x), cp<T>(dy), mp<T>(dx), rows, F));
  return ew_check("geglu_bwd");
}

int dp_axpby(int dtype, const void* a, const void* b, void* y, int64_t n, float alpha, float beta,
             dp_stream_t stream) {
  if (n <= 0) return 0;
  if (!aligned16(a) || !aligned16(y) || (b && !aligned16(b))) {
    set_error("dp_axpby: pointers must be 16-byte aligned");
    return DP_ERR_ARGS;
  }
  DISPATCH_T(dtype, launch_k(axpby_kernel<T>, dim3(ew_grid(n / VecT<T>::N + 1)), dim3(256), 0, ST,
                             cp<T>(a), cp<T>(b), mp<T>(y), n, alpha, beta));
  return ew_check("axpby");
}

int dp_gate_residual_fwd(int dtype, const void* x, const void* g, int64_t g_ld, const void* h,
                         void* y, int64_t rows, int C, int rows_per_sample, dp_stream_t stream) {
  if (rows <= 0) return 0;
  DISPATCH_T(dtype, launch_k(gate_res_fwd_kernel<T>, dim3(ew_grid(rows * C)), dim3(256), 0, ST, 
                        cp<T>(x), cp<T>(g), g_ld, cp<T>(h), mp<T>(y), rows, C, rows_per_sample));
  return ew_check("gate_residual_fwd");
}

int dp_gate_residual_bwd(int dtype, const void* dy, const void* g, int64_t g_ld, const void* h,
                         void* dh, void* dg, int64_t dg_ld, int B, int C, int rows_per_sample,
                         dp_stream_t stream) {
  if (B <= 0) return 0;
  dim3 grid((C + 31) / 32, B);
  DISPATCH_T(dtype, launch_k(gate_res_bwd_kernel<T>, dim3(grid), dim3(256), 0, ST, 
                        cp<T>(dy), cp<T>(g), g_ld, cp<T>(h), mp<T>(dh), mp<T>(dg), dg_ld, B, C,
                        rows_per_sample));
  return ew_check("gate_residual_bwd");
}

int dp_q_sample(int dtype, const void* x0, const void* noise, const int64_t* t,
                const float* sqrt_ab, const float* sqrt_1mab, void* xt, int64_t n,
                int64_t per_sample, dp_stream_t stream) {
  if (n <= 0) return 0;
  DISPATCH_T(dtype, launch_k(q_sample_kernel<T>, dim3(ew_grid(n)), dim3(256), 0, ST, 
                        cp<T>(x0), cp<T>(noise), t, sqrt_ab, sqrt_1mab, mp<T>(xt), n, per_sample));
  return ew_check("q_sample");
}

int dp_pred_x0(int dtype, const void* xt, const void* eps, const int64_t* t, const float* sqrt_ab,
               const float* sqrt_1mab, void* out, int64_t n, int64_t per_sample,
               dp_stream_t stream) {
  if (n <= 0) return 0;
  DISPATCH_T(dtype, launch_k(pred_x0_kernel<T>, dim3(ew_grid(n)), dim3(256), 0, ST, 
                        cp<T>(xt), cp<T>(eps), t, sqrt_ab, sqrt_1mab, mp<T>(out), n, per_sample));
  return ew_check("pred_x0");
}

int dp_mse(int dtype, const void* pred, const void* target, void* dpred, float* loss_acc,
           int64_t n, float scale, dp_stream_t stream) {
  if (n <= 0) return 0;
  DISPATCH_T(dtype, launch_k(mse_kernel<T>, dim3(ew_grid(n)), dim3(256), 0, ST, cp<T>(pred), cp<T>(target),
                                                                mp<T>(dpred), loss_acc, n, scale));
  return ew_check("mse");
}

int dp_timestep_embed(int dtype, const int64_t* t, void* out, int B, int dim, float max_period,
                      dp_stream_t stream) {
  if (B <= 0) return 0;
  DISPATCH_T(dtype, launch_k(timestep_embed_kernel<T>, dim3(ew_grid((int64_t)B * dim / 2)), dim3(256), 0, ST, 
                        t, mp<T>(out), B, dim, max_period));
  return ew_check("timestep_embed");
}

int dp_embed(int dtype, const int64_t* ids, const void* table, const void* pos, void* out,
             int64_t rows, int L, int C, dp_stream_t stream) {
  if (rows <= 0) return 0;
  DISPATCH_T(dtype, launch_k(embed_kernel<T>, dim3(ew_grid(rows * C)), dim3(256), 0, ST, 
                        ids, cp<T>(table), cp<T>(pos), mp<T>(out), rows, L, C));
  return ew_check("embed");
}

int dp_concat(int dtype, const void* a, const void* b, void* dst, int64_t rows, int Ca, int Cb,
              dp_stream_t stream) {
  if (rows <= 0) return 0;
  const int V = dtype == DP_F32 ? 4 : 8;
  if (Ca % V == 0 && Cb % V == 0 && aligned16(a) && aligned16(dst) && (!b || aligned16(b))) {
    DISPATCH_T(dtype, launch_k(concat_vec_kernel<T>, dim3(ew_grid(rows * (Ca + Cb) / V)), dim3(256), 0, ST, 
                          cp<T>(a), cp<T>(b), mp<T>(dst), rows, Ca, Cb));
    return ew_check("concat");
  }
  if ((Ca + Cb) % V == 0 && aligned16(dst)) {
    DISPATCH_T(dtype, launch_k(concat_rowvec_kernel<T>, dim3(ew_grid(rows * (Ca + Cb) / V)), dim3(256), 0, ST,
                               cp<T>(a), cp<T>(b), mp<T>(dst), rows, Ca, Cb));
    return ew_check("concat");
  }
  DISPATCH_T(dtype, launch_k(concat_kernel<T>, dim3(ew_grid(rows * (Ca + Cb))), dim3(256), 0, ST, 
                        cp<T>(a), cp<T>(b), mp<T>(dst), rows, Ca, Cb));
  return ew_check("concat");
}

int dp_split(int dtype, const void* src, void* a, void* b, int64_t rows, int Ca, int Cb,
             int acc_a, int acc_b, dp_stream_t stream) {
  if (rows <= 0) return 0;
  const int V = dtype == DP_F32 ? 4 : 8;
  if (Ca % V == 0 && Cb % V == 0 && aligned16(src) && (!a || aligned16(a)) && (!b || aligned16(b))) {
    DISPATCH_T(dtype, launch_k(split_vec_kernel<T>, dim3(ew_grid(rows * (Ca + Cb) / V)), dim3(256), 0, ST, 
                          cp<T>(src), mp<T>(a), mp<T>(b), rows, Ca, Cb, acc_a, acc_b));
    return ew_check("split");
  }
  DISPATCH_T(dtype, launch_k(split_kernel<T>, dim3(ew_grid(rows * (Ca + Cb))), dim3(256), 0, ST, 
                        cp<T>(src), mp<T>(a), mp<T>(b), rows, Ca, Cb, acc_a, acc_b));
  return ew_check("split");
}

int dp_upsample2x(int dtype, const void* x, void* y, int N, int H, int W, int C,
                  dp_stream_t stream) {
  if (N <= 0) return 0;
  const int V = dtype == DP_F32 ? 4 : 8;
  if (C % V == 0 && aligned16(x) && aligned16(y)) {
    DISPATCH_T(dtype, launch_k(upsample2x_vec_kernel<T>, dim3(ew_grid((int64_t)N * 4 * H * W * (C / V))), dim3(256),
                               0, ST, cp<T>(x), mp<T>(y), N, H, W, C));
    return ew_check("upsample2x");
  }
  DISPATCH_T(dtype, launch_k(upsample2x_kernel<T>, dim3(ew_grid((int64_t)N * 4 * H * W * C)), dim3(256), 0, ST, 
                        cp<T>(x), mp<T>(y), N, H, W, C));
  return ew_check("upsample2x");
}

int dp_upsample2x_bwd(int dtype, const void* dy, void* dx, int N, int H, int W, int C,
                      dp_stream_t stream) {
  if (N <= 0) return 0;
  const int V = dtype == DP_F32 ? 4 : 8;
  if (C % V == 0 && aligned16(dy) && aligned16(dx)) {
    DISPATCH_T(dtype, launch_k(upsample2x_bwd_vec_kernel<T>, dim3(ew_grid((int64_t)N * H * W * (C / V))), dim3(256),
                               0, ST, cp<T>(dy), mp<T>(dx), N, H, W, C));
    return ew_check("upsample2x_bwd");
  }
  DISPATCH_T(dtype, launch_k(upsample2x_bwd_kernel<T>, dim3(ew_grid((int64_t)N * H * W * C)), dim3(256), 0, ST, 
                        cp<T>(dy), mp<T>(dx), N, H, W, C));
  return ew_check("upsample2x_bwd");
}

int dp_cast(int src_dtype, int dst_dtype, const void* x, void* y, int64_t n, dp_stream_t stream) {
  if (n <= 0) return 0;
  const int g = ew_grid(n);
  if (src_dtype == DP_F32 && dst_dtype == DP_BF16)
    launch_k(cast_kernel<float, __nv_bfloat16>, dim3(g), dim3(256), 0, ST, cp<float>(x), mp<__nv_bfloat16>(y), n);
  else if (src_dtype == DP_BF16 && dst_dtype == DP_F32)
    launch_k(cast_kernel<__nv_bfloat16, float>, dim3(g), dim3(256), 0, ST, cp<__nv_bfloat16>(x), mp<float>(y), n);
  else if (src_dtype == DP_F32)
    launch_k(cast_kernel<float, float>, dim3(g), dim3(256), 0, ST, cp<float>(x), mp<float>(y), n);
  else
    launch_k(cast_kernel<__nv_bfloat16, __nv_bfloat16>, dim3(g), dim3(256), 0, ST, cp<__nv_bfloat16>(x),
                                                                  mp<__nv_bfloat16>(y), n);
  return ew_check("cast");
}

int dp_row_bias_fwd(int dtype, const void* x, const void* e, int64_t e_ld, void* y, int64_t rows,
                    int C, int rows_per_sample, dp_stream_t stream) {
  if (rows <= 0) return 0;
  const int V = dtype == DP_F32 ? 4 : 8;
  if (C % V || !aligned16(x) || !aligned16(y)) {
    set_error("dp_row_bias_fwd: C must be a multiple of the vector width and x/y 16-byte aligned");
    return DP_ERR_ARGS;
  }
  if (e_ld % V == 0 && aligned16(e))
    DISPATCH_T(dtype, launch_k(row_bias_fwd_kernel<T, true>, dim3(ew_grid(rows * C / V)), dim3(256), 0, ST,
                               cp<T>(x), cp<T>(e), e_ld, mp<T>(y), rows, C, rows_per_sample));
  else
    DISPATCH_T(dtype, launch_k(row_bias_fwd_kernel<T, false>, dim3(ew_grid(rows * C / V)), dim3(256), 0, ST,
                               cp<T>(x), cp<T>(e), e_ld, mp<T>(y), rows, C, rows_per_sample));
  return ew_check("row_bias_fwd");
}

int dp_row_bias_bwd_db(int dtype, const void* dy, void* de, int64_t de_ld, int B, int C,
                       int rows_per_sample, float* db, float* db2, dp_stream_t stream) {
  if (B <= 0) return 0;
  const int V = dtype == DP_F32 ? 4 : 8;
  if (C % V == 0 && de_ld % V == 0 && aligned16(dy) && aligned16(de)) {
    const int CV = C / V;
    // channel vectors per block: the largest divisor of CV (<= 256, >= 8 vectors = 128-byte row
    // runs when CV allows) that still gives >= 2 blocks per SM over (channel blocks x samples)
    const int lo = CV < 8 ? CV : 8;
    int CVB = 0;
    for (int d = (CV < 256 ? CV : 256); d >= lo; --d)
      if (CV % d == 0) {
        CVB = d;
        if ((int64_t)(CV / d) * B >= 2 * kNumSMs) break;
      }
    if (CVB == 0)  // no divisor in [lo, 256] (e.g. prime CV > 256): the largest divisor <= 256
      for (int d = (CV < 256 ? CV : 256); d >= 1; --d)
        if (CV % d == 0) {
          CVB = d;
          break;
        }
    dim3 g(CV / CVB, B);
    DISPATCH_T(dtype, launch_k(row_bias_bwd_vec_kernel<T>, dim3(g), dim3(256), 0, ST, cp<T>(dy), mp<T>(de), de_ld,
                               C, rows_per_sample, CVB, db, db2));
    return ew_check("row_bias_bwd");
  }
  dim3 grid((C + 31) / 32, B);
  DISPATCH_T(dtype, launch_k(row_bias_bwd_kernel<T>, dim3(grid), dim3(256), 0, ST, cp<T>(dy), mp<T>(de), de_ld, C,
                                                                   rows_per_sample, db, db2));
  return ew_check("row_bias_bwd");
}

int dp_row_bias_bwd(int dtype, const void* dy, void* de, int64_t de_ld, int B, int C,
                    int rows_per_sample, dp_stream_t stream) {
  return dp_row_bias_bwd_db(dtype, dy, de, de_ld, B, C, rows_per_sample, nullptr, nullptr, stream);
}

int dp_space_to_depth(int dtype, const void* x, void* y, int N, int H, int W, int C, int p,
                      int inverse, dp_stream_t stream) {
  if (N <= 0) return 0;
  if (H % p || W % p) {
    set_error("dp_space_to_depth: H and W must be multiples of p");
    return DP_ERR_ARGS;
  }
  DISPATCH_T(dtype, launch_k(s2d_kernel<T>, dim3(ew_grid((int64_t)N * H * W * C)), dim3(256), 0, ST, 
                        cp<T>(x), mp<T>(y), N, H, W, C, p, inverse));
  return ew_check("space_to_depth");
}

int dp_bias_grad(int dtype, const void* dy, float* db, int64_t rows, int C, dp_stream_t stream) {
  if (rows <= 0) return 0;
  const int V = dtype == DP_F32 ? 4 : 8;
  static const bool old_path = getenv("DP_BIAS_GRAD_OLD") != nullptr;  // A/B experiments
  if (C % V == 0 && aligned16(dy) && !old_path) {
    const int CV = C / V;
    // channel vectors per block: the divisor of CV (<= 256) that keeps the most of 256 threads busy
    int CVB = 0, best = -1;
    for (int d = 1; d <= 256 && d <= CV; ++d)
      if (CV % d == 0 && (256 / d) * d >= best) {
        best = (256 / d) * d;
        CVB = d;
      }
    const int RL = 256 / CVB;
    // ~4 resident blocks per SM, at least 4 rows per row lane
    int64_t seg = (rows + 4 * kNumSMs - 1) / (4 * kNumSMs);
    if (seg < 4 * RL) seg = 4 * RL;
    dim3 grid(CV / CVB, static_cast<unsigned>((rows + seg - 1) / seg));
    DISPATCH_T(dtype, launch_k(bias_grad_rows_kernel<T>, dim3(grid), dim3(256), 0, ST, cp<T>(dy), db, rows, C, CVB,
                               static_cast<int>(seg)));
    return ew_check("bias_grad");
  }
  if (C % V == 0 && aligned16(dy)) {
    // 16-byte vectors: a block covers 32 vectors (256 bf16 channels) x 8 row lanes
    const int CV = C / V;
    int64_t seg = (rows * ((CV + 31) / 32) + 2 * kNumSMs - 1) / (2 * kNumSMs);  // ~2 waves
    seg = seg < 64 ? 64 : seg;
    dim3 grid((CV + 31) / 32, static_cast<unsigned>((rows + seg - 1) / seg));
    DISPATCH_T(dtype, launch_k(bias_grad_vec_kernel<T>, dim3(grid), dim3(256), 0, ST, cp<T>(dy), db, rows, C,
                                                                      static_cast<int>(seg)));
    return ew_check("bias_grad");
  }
  const int seg = 512;
  dim3 grid((C + 31) / 32, static_cast<unsigned>((rows + seg - 1) / seg));
  DISPATCH_T(dtype, launch_k(bias_grad_kernel<T>, dim3(grid), dim3(256), 0, ST, cp<T>(dy), db, rows, C, seg));
  return ew_check("bias_grad");
}

int dp_adamw(float* param, const float* grad, float* exp_avg, float* exp_avg_sq,
             void* param_bf16, int64_t n, float lr, float beta1, float beta2, float eps,
             float weight_decay, int step, float grad_scale, dp_stream_t stream) {
  if (n <= 0) return 0;
  if (!aligned16(param) || !aligned16(grad) || !aligned16(exp_avg) || !aligned16(exp_avg_sq)) {
    set_error("dp_adamw: flat buffers must be 16-byte aligned");
    return DP_ERR_ARGS;
  }
  const float bc1 = 1.f - powf(beta1, static_cast<float>(step));
  const float bc2 = 1.f - powf(beta2, static_cast<float>(step));
  launch_k(adamw_kernel, dim3(ew_grid(n / 4 + 1)), dim3(256), 0, ST, param, grad, exp_avg, exp_avg_sq,
                                                    mp<__nv_bfloat16>(param_bf16), n, lr, beta1,
                                                    beta2, eps, weight_decay, bc1, bc2,
                                                    grad_scale, nullptr, 0);
  return ew_check("adamw");
}

// Chunked AdamW (optimizer overlapped with the backward pass): advance the device step counter
// and bias corrections once per iteration, then update any number of flat slices with them.
int dp_adamw_advance(int* step_dev, float beta1, float beta2, float* bc_dev, dp_stream_t stream) {
  launch_k(adamw_step_kernel, dim3(1), dim3(1), 0, ST, step_dev, beta1, beta2, bc_dev);
  return ew_check("adamw_advance");
}

int dp_adamw_apply(float* param, const float* grad, float* exp_avg, float* exp_avg_sq,
                   void* param_bf16, int64_t n, float lr, float beta1, float beta2, float eps,
                   float weight_decay, const float* bc_dev, float grad_scale, int max_ctas,
                   int zero_grad, dp_stream_t stream) {
  if (n <= 0) return 0;
  if (!aligned16(param) || !aligned16(grad) || !aligned16(exp_avg) || !aligned16(exp_avg_sq)) {
    set_error("dp_adamw_apply: flat buffers must be 16-byte aligned");
    return DP_ERR_ARGS;
  }
  // max_ctas > 0 caps the grid (grid-stride loop): a background update running next to the
  // backward pass must leave thread slots for the persistent GEMM CTAs on every SM
  int grid = ew_grid(n / 4 + 1);
  if (max_ctas > 0 && grid > max_ctas) grid = max_ctas;
  launch_k(adamw_kernel, dim3(grid), dim3(256), 0, ST, param, grad, exp_avg, exp_avg_sq,
                                                    mp<__nv_bfloat16>(param_bf16), n, lr, beta1,
                                                    beta2, eps, weight_decay, 1.f, 1.f, grad_scale,
                                                    bc_dev, zero_grad);
  return ew_check("adamw_apply");
}

int dp_adamw_dev(float* param, const float* grad, float* exp_avg, float* exp_avg_sq,
                 void* param_bf16, int64_t n, float lr, float beta1, float beta2, float eps,
                 float weight_decay, int* step_dev, float* bc_dev, float grad_scale,
                 dp_stream_t stream) {
  if (n <= 0) return 0;
  if (!aligned16(param) || !aligned16(grad) || !aligned16(exp_avg) || !aligned16(exp_avg_sq)) {
    set_error("dp_adamw_dev: flat buffers must be 16-byte aligned");
    return DP_ERR_ARGS;
  }
  launch_k(adamw_step_kernel, dim3(1), dim3(1), 0, ST, step_dev, beta1, beta2, bc_dev);
  launch_k(adamw_kernel, dim3(ew_grid(n / 4 + 1)), dim3(256), 0, ST, param, grad, exp_avg, exp_avg_sq,
                                                    mp<__nv_bfloat16>(param_bf16), n, lr, beta1,
                                                    beta2, eps, weight_decay, 1.f, 1.f, grad_scale,
                                                    bc_dev, 0);
  return ew_check("adamw_dev");
}

}  // extern "C"
