// Convolution lowering helpers: im2col / col2im (generic path for small-channel
// convs and the fp32 configuration), dgrad weight flip, and zero-dilation of
// the output gradient (dgrad of strided convs as a stride-1 conv).
#include <string>
#include "common.cuh"
#include "dpipe.h"

namespace dp {
void set_error(const std::string& s);

template <typename T>
__global__ void im2col_kernel(const T* __restrict__ x, T* __restrict__ cols, int N, int H, int W,
                              int C, int R, int S, int stride, int ph, int pw, int P, int Q,
                              int64_t total) {
  DP_PDL_ENTRY();
  const int64_t ncol = (int64_t)R * S * C;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = i / ncol;
    const int col = static_cast<int>(i - row * ncol);
    const int c = col % C;
    const int tap = col / C;
    const int s = tap % S, r = tap / S;
    const int q = static_cast<int>(row % Q);
    const int64_t t = row / Q;
    const int p = static_cast<int>(t % P);
    const int n = static_cast<int>(t / P);
    const int h = p * stride + r - ph, w = q * stride + s - pw;
    T v = from_f<T>(0.f);
    if (h >= 0 && h < H && w >= 0 && w < W) v = x[(((int64_t)n * H + h) * W + w) * C + c];
    cols[i] = v;
  }
}

// Gather form of col2im (deterministic): each input element sums the columns that read it.
template <typename T>
__global__ void col2im_kernel(const T* __restrict__ cols, T* __restrict__ dx, int N, int H, int W,
                              int C, int R, int S, int stride, int ph, int pw, int P, int Q,
                              int64_t total) {
  DP_PDL_ENTRY();
  const int64_t ncol = (int64_t)R * S * C;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int c = static_cast<int>(i % C);
    int64_t t = i / C;
    const int w = static_cast<int>(t % W);
    t /= W;
    const int h = static_cast<int>(t % H);
    const int n = static_cast<int>(t / H);
    float acc = 0.f;
    for (int r = 0; r < R; ++r) {
      const int hp = h + ph - r;
      if (hp < 0 || hp % stride) continue;
      const int p = hp / stride;
      if (p >= P) continue;
      for (int s = 0; s < S; ++s) {
        const int wq = w + pw - s;
        if (wq < 0 || wq % stride) continue;
        const int q = wq / stride;
        if (q >= Q) continue;
        const int64_t row = ((int64_t)n * P + p) * Q + q;
        acc += to_f<T>(cols[row * ncol + (r * S + s) * C + c]);
      }
    }
    dx[i] = from_f<T>(to_f<T>(dx[i]) + acc);
  }
}

template <typename T>
__global__ void flip_kernel(const T* __restrict__ w, T* __restrict__ wt, int K, int R, int S,
                            int C) {
  DP_PDL_ENTRY();
  const int64_t total = (int64_t)K * R * S * C;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    // i indexes w[k][r][s][c]
    const int c = static_cast<int>(i % C);
    int64_t t = i / C;
    const int s = static_cast<int>(t % S);
    t /= S;
    const int r = static_cast<int>(t % R);
    const int k = static_cast<int>(t / R);
    wt[(((int64_t)c * R + (R - 1 - r)) * S + (S - 1 - s)) * K + k] = w[i];
  }
}

// Tiled flip-transpose (bf16, K % 8 == 0, C % 8 == 0): per tap, a 64 x 64 block of w[k][tap][c]
// is read with 16-byte row loads (coalesced in c), staged in shared memory, and written as
// 16-byte vectors of 8 consecutive k (coalesced in k) to wt[c][flipped tap][k]. The scalar
// flip_kernel above scatters its writes with stride K (one 2-byte store per 128-byte line).
__global__ void __launch_bounds__(256)
    flip_t_kernel(const __nv_bfloat16* __restrict__ w, __nv_bfloat16* __restrict__ wt, int K, int R, int S,
                  int C) {
  DP_PDL_ENTRY();
  __shared__ __nv_bfloat16 tile[64][64 + 8];
  const int c0 = blockIdx.x * 64, k0 = blockIdx.y * 64, tap = blockIdx.z;
  const int RS = R * S;
  const int r = tap / S, s = tap - (tap / S) * S;
  const int ftap = (R - 1 - r) * S + (S - 1 - s);
  for (int i = threadIdx.x; i < 64 * 8; i += 256) {
    const int kk = i >> 3, cv = (i & 7) * 8;
    const int k = k0 + kk, c = c0 + cv;
    uint4 u = make_uint4(0, 0, 0, 0);
    if (k < K && c < C) u = *reinterpret_cast<const uint4*>(w + ((int64_t)k * RS + tap) * C + c);
    *reinterpret_cast<uint4*>(&tile[kk][cv]) = u;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 64 * 8; i += 256) {
    const int cc = i >> 3, kv = (i & 7) * 8;
    const int c = c0 + cc, k = k0 + kv;
    if (c >= C || k >= K) continue;
    __align__(16) __nv_bfloat16 v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = tile[kv + j][cc];
    *reinterpret_cast<uint4*>(wt + ((int64_t)c * RS + ftap) * K + k) = *reinterpret_cast<const uint4*>(v);
  }
}

// Batched refresh of the cached dgrad weight copies (after an optimizer slice): one launch over
// every job's 64x64 tiles instead of one launch per parameter (~150 per step).
struct FlipBatch {
  const __nv_bfloat16* w[DP_FLIP_BATCH_MAX];
  __nv_bfloat16* wt[DP_FLIP_BATCH_MAX];
  int K[DP_FLIP_BATCH_MAX], R[DP_FLIP_BATCH_MAX], S[DP_FLIP_BATCH_MAX], C[DP_FLIP_BATCH_MAX];
  int tile0[DP_FLIP_BATCH_MAX + 1];  // prefix sums of the jobs' tile counts
  int n;
};

__global__ void __launch_bounds__(256) flip_t_batch_kernel(const __grid_constant__ FlipBatch fb) {
  DP_PDL_ENTRY();
  __shared__ __nv_bfloat16 tile[64][64 + 8];
  int j = 0;
  while (j + 1 < fb.n && static_cast<int>(blockIdx.x) >= fb.tile0[j + 1]) ++j;
  const int K = fb.K[j], R = fb.R[j], S = fb.S[j], C = fb.C[j];
  const int ct = (C + 63) / 64, kt = (K + 63) / 64;
  int t = blockIdx.x - fb.tile0[j];
  const int tap = t / (ct * kt);
  t -= tap * ct * kt;
  const int k0 = (t / ct) * 64, c0 = (t - (t / ct) * ct) * 64;
  const __nv_bfloat16* w = fb.w[j];
  __nv_bfloat16* wt = fb.wt[j];
  const int RS = R * S;
  const int r = tap / S, s = tap - (tap / S) * S;
  const int ftap = (R - 1 - r) * S + (S - 1 - s);
  for (int i = threadIdx.x; i < 64 * 8; i += 256) {
    const int kk = i >> 3, cv = (i & 7) * 8;
    const int k = k0 + kk, c = c0 + cv;
    uint4 u = make_uint4(0, 0, 0, 0);
    if (k < K && c < C) u = *reinterpret_cast<const uint4*>(w + ((int64_t)k * RS + tap) * C + c);
    *reinterpret_cast<uint4*>(&tile[kk][cv]) = u;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 64 * 8; i += 256) {
    const int cc = i >> 3, kv = (i & 7) * 8;
    const int c = c0 + cc, k = k0 + kv;
    if (c >= C || k >= K) continue;
    __align__(16) __nv_bfloat16 v[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) v[q] = tile[kv + q][cc];
    *reinterpret_cast<uint4*>(wt + ((int64_t)c * RS + ftap) * K + k) = *reinterpret_cast<const uint4*>(v);
  }
}

template <typename T>
__global__ void dilate_kernel(const T* __restrict__ dy, T* __restrict__ out, int N, int P, int Q,
                              int C, int stride) {
  DP_PDL_ENTRY();
  const int Ho = P * stride, Wo = Q * stride;
  const int64_t total = (int64_t)N * Ho * Wo * C;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int c = static_cast<int>(i % C);
    int64_t t = i / C;
    const int w = static_cast<int>(t % Wo);
    t /= Wo;
    const int h = static_cast<int>(t % Ho);
    const int n = static_cast<int>(t / Ho);
    T v = from_f<T>(0.f);
    if (h % stride == 0 && w % stride == 0)
      v = dy[(((int64_t)n * P + h / stride) * Q + w / stride) * C + c];
    out[i] = v;
  }
}

// bf16, C % 8 == 0: one thread per 16-byte channel vector of the dilated map
__global__ void dilate_vec_kernel(const __nv_bfloat16* __restrict__ dy, __nv_bfloat16* __restrict__ out, int N,
                                  int P, int Q, int C, int stride) {
  DP_PDL_ENTRY();
  const int Ho = P * stride, Wo = Q * stride, CV = C / 8;
  const int64_t total = (int64_t)N * Ho * Wo * CV;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int cv = static_cast<int>(i % CV);
    int64_t t = i / CV;
    const int w = static_cast<int>(t % Wo);
    t /= Wo;
    const int h = static_cast<int>(t % Ho);
    const int n = static_cast<int>(t / Ho);
    uint4 v = make_uint4(0, 0, 0, 0);
    if (h % stride == 0 && w % stride == 0)
      v = *reinterpret_cast<const uint4*>(dy + (((int64_t)n * P + h / stride) * Q + w / stride) * C + cv * 8);
    *reinterpret_cast<uint4*>(out + i * 8) = v;
  }
}

static inline int grid_for(int64_t total) {
  int64_t g = (total + 255) / 256;
  const int64_t cap = (int64_t)kNumSMs * 16;
  return static_cast<int>(g < 1 ? 1 : (g > cap ? cap : g));
}

static int check(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) set_error(std::string(what) + ": " + cudaGetErrorString(e));
  return e;
}

}  // namespace dp

using namespace dp;

extern "C" {

int dp_im2col(int dtype, const void* x, void* cols, int N, int H, int W, int C, int R, int S,
              int stride, int pad_h, int pad_w, int P, int Q, dp_stream_t stream) {
  const int64_t total = (int64_t)N * P * Q * R * S * C;
  if (total == 0) return 0;
  auto st = reinterpret_cast<cudaStream_t>(stream);
  if (dtype == DP_F32)
    launch_k(im2col_kernel<float>, dim3(grid_for(total)), dim3(256), 0, st, 
        (const float*)x, (float*)cols, N, H, W, C, R, S, stride, pad_h, pad_w, P, Q, total);
  else
    launch_k(im2col_kernel<__nv_bfloat16>, dim3(grid_for(total)), dim3(256), 0, st, 
        (const __nv_bfloat16*)x, (__nv_bfloat16*)cols, N, H, W, C, R, S, stride, pad_h, pad_w, P,
        Q, total);
  return check("im2col");
}

int dp_col2im(int dtype, const void* cols, void* dx, int N, int H, int W, int C, int R, int S,
              int stride, int pad_h, int pad_w, int P, int Q, dp_stream_t stream) {
  const int64_t total = (int64_t)N * H * W * C;
  if (total == 0) return 0;
  auto st = reinterpret_cast<cudaStream_t>(stream);
  if (dtype == DP_F32)
    launch_k(col2im_kernel<float>, dim3(grid_for(total)), dim3(256), 0, st, 
        (const float*)cols, (float*)dx, N, H, W, C, R, S, stride, pad_h, pad_w, P, Q, total);
  else
    launch_k(col2im_kernel<__nv_bfloat16>, dim3(grid_for(total)), dim3(256), 0, st, 
        (const __nv_bfloat16*)cols, (__nv_bfloat16*)dx, N, H, W, C, R, S, stride, pad_h, pad_w, P,
        Q, total);
  return check("col2im");
}

int dp_conv_weight_flip(int dtype, const void* w, void* wt, int K, int R, int S, int C,
                        dp_stream_t stream) {
  const int64_t total = (int64_t)K * R * S * C;
  if (total == 0) return 0;
  auto st = reinterpret_cast<cudaStream_t>(stream);
  if (dtype != DP_F32 && K % 8 == 0 && C % 8 == 0) {
    dim3 grid((C + 63) / 64, (K + 63) / 64, R * S);
    launch_k(flip_t_kernel, dim3(grid), dim3(256), 0, st, (const __nv_bfloat16*)w, (__nv_bfloat16*)wt, K, R, S, C);
  } else if (dtype == DP_F32)
    launch_k(flip_kernel<float>, dim3(grid_for(total)), dim3(256), 0, st, (const float*)w, (float*)wt, K, R, S, C);
  else
    launch_k(flip_kernel<__nv_bfloat16>, dim3(grid_for(total)), dim3(256), 0, st, 
        (const __nv_bfloat16*)w, (__nv_bfloat16*)wt, K, R, S, C);
  return check("conv_weight_flip");
}

int dp_conv_weight_flip_batch(const DpFlipJob* jobs, int n, dp_stream_t stream) {
  auto st = reinterpret_cast<cudaStream_t>(stream);
  for (int base = 0; base < n; base += DP_FLIP_BATCH_MAX) {
    FlipBatch fb{};
    fb.n = n - base < DP_FLIP_BATCH_MAX ? n - base : DP_FLIP_BATCH_MAX;
    int tiles = 0;
    for (int i = 0; i < fb.n; ++i) {
      const DpFlipJob& jb = jobs[base + i];
      if (jb.K % 8 || jb.C % 8 || (reinterpret_cast<uintptr_t>(jb.w) | reinterpret_cast<uintptr_t>(jb.wt)) % 16) {
        dp::set_error("dp_conv_weight_flip_batch: bf16 jobs with K % 8 == 0, C % 8 == 0, 16-byte aligned");
        return DP_ERR_ARGS;
      }
      fb.w[i] = static_cast<const __nv_bfloat16*>(jb.w);
      fb.wt[i] = static_cast<__nv_bfloat16*>(jb.wt);
      fb.K[i] = jb.K;
      fb.R[i] = jb.R;
      fb.S[i] = jb.S;
      fb.C[i] = jb.C;
      fb.tile0[i] = tiles;
      tiles += ((jb.C + 63) / 64) * ((jb.K + 63) / 64) * jb.R * jb.S;
    }
    fb.tile0[fb.n] = tiles;
    if (tiles == 0) continue;
    launch_k(flip_t_batch_kernel, dim3(tiles), dim3(256), 0, st, fb);
  }
  return check("conv_weight_flip_batch");
}

int dp_dilate(int dtype, const void* dy, void* out, int N, int P, int Q, int C, int stride,
              dp_stream_t stream) {
  const int64_t total = (int64_t)N * P * stride * Q * stride * C;
  if (total == 0) return 0;
  auto st = reinterpret_cast<cudaStream_t>(stream);
  if (dtype == DP_F32)
    launch_k(dilate_kernel<float>, dim3(grid_for(total)), dim3(256), 0, st, (const float*)dy, (float*)out, N, P, Q,
                                                           C, stride);
  else if (C % 8 == 0 && (reinterpret_cast<uintptr_t>(dy) | reinterpret_cast<uintptr_t>(out)) % 16 == 0)
    launch_k(dilate_vec_kernel, dim3(grid_for(total / 8)), dim3(256), 0, st, (const __nv_bfloat16*)dy,
             (__nv_bfloat16*)out, N, P, Q, C, stride);
  else
    launch_k(dilate_kernel<__nv_bfloat16>, dim3(grid_for(total)), dim3(256), 0, st, 
        (const __nv_bfloat16*)dy, (__nv_bfloat16*)out, N, P, Q, C, stride);
  return check("dilate");
}

}  // extern "C"
