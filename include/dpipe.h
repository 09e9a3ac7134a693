/*
 * dpipe.h — C ABI of libdpipe.so, the sm_100a kernel library behind the
 * pipelined diffusion-training executor (paper_2405_01248_b200).
 *
 * The reference (arXiv 2405.01248, /root/reference) ships only the offline
 * planner `pipefill`; its back-end engine ("PyTorch 2.0.1 and CUDA 11.7 with
 * 20k LoC in Python") is not in the reference tree. The entry
 * points below are the compute operators that back-end called through
 * PyTorch/cuDNN/cuBLAS for the stage forward/backward (PAPER.md:259-266,
 * Fig. 6 step 6) and the frozen-encoder fills.
 * Each one replaces a library op of that engine:
 *
 *   dp_gemm            torch.nn.functional.linear / torch.bmm (cuBLAS)
 *   dp_conv_fwd        torch.nn.functional.conv2d forward (cuDNN implicit GEMM)
 *   dp_conv_wgrad      conv2d weight gradient (cuDNN wgrad)
 *   dp_im2col/col2im   generic conv lowering (small-channel convs, fp32 path)
 *   dp_group_norm_*    torch.nn.GroupNorm(+SiLU) fwd/bwd
 *   dp_layer_norm_*    torch.nn.LayerNorm fwd/bwd
 *   dp_softmax_*       row softmax fwd/bwd (attention)
 *   dp_eltwise         GEGLU / GELU / SiLU / add / scale / diffusion q_sample / MSE
 *   dp_adamw           torch.optim.AdamW (multi-tensor, fp32 master weights)
 *
 * Conventions: plain device pointers, element strides, explicit cudaStream_t.
 * The caller (PyTorch's caching allocator) owns every buffer; no entry point
 * allocates, frees or synchronizes. Every entry returns 0 on success or a
 * nonzero error code (cudaError_t, or DP_ERR_* for argument errors);
 * dp_last_error() returns a message for the last failure on this thread.
 */
#ifndef DPIPE_H_
#define DPIPE_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* dp_stream_t; /* == cudaStream_t */

enum { DP_F32 = 0, DP_BF16 = 1 };
enum { DP_OUT_STORE = 0, DP_OUT_ATOMIC_ADD = 1 };
enum { DP_ERR_ARGS = 1001, DP_ERR_UNSUPPORTED = 1002, DP_ERR_DRIVER = 1003 };

/* D[z](m,n) = alpha * sum_k A[z](m,k) * B[z](n,k)  (+ bias[n]) (+ Res[z](m,n))
 * z = z1 + batch1 * z2.  A is "K-major" when A(m,k) = A[m*a_ld + k] and
 * "MN-major" when A(m,k) = A[k*a_ld + m]; same for B with n. Strides in
 * elements. out_mode DP_OUT_ATOMIC_ADD adds into an fp32 D (split-K and
 * gradient accumulation). dtype selects the tensor-core bf16 path (tcgen05,
 * fp32 accumulate) or the fp32 path. */
typedef struct DpGemmArgs {
  int M, N, K;
  int batch1, batch2;
  int dtype;
  const void* A;
  int64_t a_ld, a_bs1, a_bs2;
  int a_mn_major;
  const void* B;
  int64_t b_ld, b_bs1, b_bs2;
  int b_mn_major;
  void* D;
  int d_dtype;
  int64_t d_ld, d_bs1, d_bs2;
  int out_mode;
  const float* bias;
  const void* Res; /* same dtype and strides convention as D */
  int64_t r_ld, r_bs1, r_bs2;
  float alpha;
  int split_k; /* 0 = heuristic */
} DpGemmArgs;

/* 2-D convolution over NHWC activations with weights [K][R][S][C].
 * Output y is NHWC [N][P][Q][K]. pad_h/pad_w are the top/left paddings;
 * the bottom/right padding is implied by P, Q (zero outside the input). */
typedef struct DpConvArgs {
  int dtype;
  int N, H, W, C;
  int K, R, S;
  int stride, pad_h, pad_w;
  int P, Q;
  const void* x;
  const void* w;
  void* y;
  const float* bias;
  const void* Res; /* optional residual, same layout as y */
  float alpha;
  int out_mode;
  int split_k;
} DpConvArgs;

int dp_gemm(const DpGemmArgs* args, dp_stream_t stream);
/* y = conv(x, w) (+bias) (+Res); bf16 tensor-core implicit GEMM, needs C % 64 == 0 */
int dp_conv_fwd(const DpConvArgs* args, dp_stream_t stream);
/* w-grad: y is dW fp32 [K][R][S][C] (accumulated), x the layer input, w := dy [N][P][Q][K] */
int dp_conv_wgrad(const DpConvArgs* args, dp_stream_t stream);

/* cols[(n*P+p)*Q+q][(r*S+s)*C+c] = x[n][p*stride+r-pad_h][q*stride+s-pad_w][c] (0 outside) */
int dp_im2col(int dtype, const void* x, void* cols, int N, int H, int W, int C, int R, int S,
              int stride, int pad_h, int pad_w, int P, int Q, dp_stream_t stream);
/* dx[...] (+)= scatter-add of cols (the adjoint of im2col); dx must be zeroed by caller */
int dp_col2im(int dtype, const void* cols, void* dx, int N, int H, int W, int C, int R, int S,
              int stride, int pad_h, int pad_w, int P, int Q, dp_stream_t stream);
/* wt[c][R-1-r][S-1-s][k] = w[k][r][s][c] (dgrad-as-conv weights) */
int dp_conv_weight_flip(int dtype, const void* w, void* wt, int K, int R, int S, int C,
                        dp_stream_t stream);
/* out[n][p*stride][q*stride][c] = dy[n][p][q][c]; other positions 0. out: [N][P*stride][Q*stride][C] */
int dp_dilate(int dtype, const void* dy, void* out, int N, int P, int Q, int C, int stride,
              dp_stream_t stream);

const char* dp_last_error(void);
int dp_version(void);

#ifdef __cplusplus
}
#endif
#endif /* DPIPE_H_ */
