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
enum { DP_ACT_NONE = 0, DP_ACT_GELU = 1, DP_ACT_GELU_TANH = 2, DP_ACT_SILU = 3 };

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
  /* optional fp32 workspace (caller-owned, 16-byte aligned). When a bf16 STORE GEMM covers
     too few tiles to fill the SMs, the kernel accumulates split-K partials into it with fp32
     atomics and a finish kernel applies bias/residual and writes D. dp_gemm_workspace()
     returns the bytes that enable this (0: not needed); with a smaller or NULL workspace the
     GEMM runs unsplit. */
  float* workspace;
  int64_t workspace_bytes;
  /* optional GEGLU epilogues (bf16, K-major operands, no residual / batch):
     geglu_mode 1 (forward of the FF input projection, N = 2F): B rows [0, F) produce a and [F, 2F) g of
       the pre-activation D = [a | g] (stored as usual, it is the backward's input); geglu_out[m][f] =
       a * gelu_erf(g) (row stride geglu_ld) is written by the same epilogue;
     geglu_mode 2 (input gradient of the FF output projection, N = F): the GEMM result is dy = dL/dy of
       the GEGLU output; with h = geglu_out ([M][2F] pre-activation, row stride geglu_ld) the epilogue
       writes D[m][f] = dy * gelu(g) and D[m][F + f] = dy * a * gelu'(g) (D is [M][2F], row stride d_ld);
     geglu_mode 3 (GELU activation epilogue, bf16 K-major store, N % 128 == 0, no residual / batch):
       D = gelu_erf(A B^T + bias) (geglu_out unused).
     0: off. */
  void* geglu_out;
  int64_t geglu_ld;
  int geglu_mode;
} DpGemmArgs;

/* 2-D convolution over NHWC activations with weights [K][R][S][C].
 * Output y is NHWC [N][P][Q][K]. pad_h/pad_w are the top/left paddings;
 * the bottom/right padding is implied by P, Q (zero outside the input). */
#define DP_GN_SLOTS 16
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
  float* workspace; /* as DpGemmArgs::workspace (conv fwd / dgrad) */
  int64_t workspace_bytes;
  /* conv fwd, bf16: GroupNorm statistics of the output for its consumer (gn_groups groups, K / gn_groups a
     power of two in [4, 32], P*Q % 32 == 0): gn_sums[slot][n][g] = partial {sum, sum of squares} over the
     stored (bf16) values in DP_GN_SLOTS copies (spreads the reductions), zeroed and accumulated by the
     launch; read by dp_group_norm_fwd_sums. NULL: off. */
  float* gn_sums;
  int gn_groups;
} DpConvArgs;

/* Multi-head attention over strided [B][N][heads*head_dim] activations (q, k, v may be
   column slices of one fused qkv / kv tensor). Strides in elements: *_ld between tokens,
   *_bs between batch entries. lse (optional) receives [B][heads][N] log2-domain
   log-sum-exp (m + log2 l) of the scaled scores. */
typedef struct DpAttnArgs {
  int dtype;
  int B, N, Nk, heads, head_dim;
  const void* q;
  const void* k;
  const void* v;
  void* o;
  int64_t q_ld, q_bs, kv_ld, kv_bs, o_ld, o_bs;
  float scale;
  float* lse;
  int causal; /* forward only: key j > query i masked (N == Nk; CLIP's causal text encoder) */
} DpAttnArgs;

int dp_gemm(const DpGemmArgs* args, dp_stream_t stream);
/* bytes of fp32 workspace that let dp_gemm / dp_conv_fwd / dp_conv_dgrad split K over all SMs
   for an under-filled launch (0 = the launch fills the machine unsplit); host-only query */
int64_t dp_gemm_workspace(const DpGemmArgs* args);
int64_t dp_conv_fwd_workspace(const DpConvArgs* args);
int64_t dp_conv_dgrad_workspace(const DpConvArgs* args);
/* fused attention forward (tcgen05 S = QK^T and O = PV, online softmax from TMEM);
   bf16, head_dim 64; args->causal masks key j > query i (N == Nk; no backward) */
int dp_flash_attn_fwd(const DpAttnArgs* args, dp_stream_t stream);
/* fused attention backward (recomputes P from args->lse): dq (token stride dq_ld), dk/dv
   (token stride dkv_ld) for the o written by dp_flash_attn_fwd (non-causal); workspace holds
   B*heads*N + B*N*heads*64 floats (the dQ accumulator is unused when Nk <= 128: dQ is stored
   directly) */
/* bytes of fp32 workspace dp_flash_attn_bwd needs for these args (D, dQ accumulator and, when the
   query tiles are split across CTAs, the dK/dV accumulators) */
int64_t dp_flash_attn_bwd_workspace(const DpAttnArgs* args);
int dp_flash_attn_bwd(const DpAttnArgs* args, const void* dout, int64_t do_ld, void* dq,
                      int64_t dq_ld, void* dk, void* dv, int64_t dkv_ld, float* workspace,
                      dp_stream_t stream);
/* y = conv(x, w) (+bias) (+Res); bf16 tensor-core implicit GEMM, needs C % 64 == 0 */
int dp_conv_fwd(const DpConvArgs* args, dp_stream_t stream);
/* input gradient of a stride-1 conv, weights read tap-flipped in place (no transposed copy):
   N,H,W,C describe dx (= args->y), P,Q describe dy (= args->x), w the forward weights
   [K][R][S][C], pad_h/pad_w the forward paddings; needs C % 64 == 0 and K % 64 == 0 */
int dp_conv_dgrad(const DpConvArgs* args, dp_stream_t stream);
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
/* Batched dgrad weight-copy refresh (bf16): for every job, wt[c][R-1-r][S-1-s][k] = w[k][r][s][c]
   (dp_conv_weight_flip's layout), all jobs in one launch per DP_FLIP_BATCH_MAX jobs. */
#define DP_FLIP_BATCH_MAX 48
typedef struct DpFlipJob {
  const void* w;
  void* wt;
  int K, R, S, C;
} DpFlipJob;
int dp_conv_weight_flip_batch(const DpFlipJob* jobs, int n, dp_stream_t stream);
int dp_dilate(int dtype, const void* dy, void* out, int N, int P, int Q, int C, int stride,
              dp_stream_t stream);


/* ---- elementwise (eltwise.cu); dtype DP_F32 / DP_BF16, n in elements ---- */
/* y = act(x); dx (+)= dy * act'(x). 16-byte aligned pointers. */
int dp_act_fwd(int op, int dtype, const void* x, void* y, int64_t n, dp_stream_t stream);
int dp_act_bwd(int op, int dtype, const void* x, const void* dy, void* dx, int64_t n,
               int accumulate, dp_stream_t stream);
/* x [rows][2F] = [a | g] -> y [rows][F] = a * gelu(g)   (SD GEGLU feed-forward) */
int dp_geglu_fwd(int dtype, const void* x, void* y, int64_t rows, int F, dp_stream_t stream);
int dp_geglu_bwd(int dtype, const void* x, const void* dy, void* dx, int64_t rows, int F,
                 dp_stream_t stream);
/* GEGLU backward fused with the producing projection's bias gradient: db[0..2F) += column sums of
   dx (fp32 accumulate; db NULL -> dp_geglu_bwd) */
int dp_geglu_bwd_db(int dtype, const void* x, const void* dy, void* dx, int64_t rows, int F, float* db,
                    dp_stream_t stream);
/* y = alpha*a + beta*b  (b may be NULL) */
int dp_axpby(int dtype, const void* a, const void* b, void* y, int64_t n, float alpha, float beta,
             dp_stream_t stream);
/* adaLN-Zero gated residual: y[r] = x[r] + g[r/rps] * h[r]; backward gives dh and dg[B][C] */
int dp_gate_residual_fwd(int dtype, const void* x, const void* g, int64_t g_ld, const void* h,
                         void* y, int64_t rows, int C, int rows_per_sample, dp_stream_t stream);
int dp_gate_residual_bwd(int dtype, const void* dy, const void* g, int64_t g_ld, const void* h,
                         void* dh, void* dg, int64_t dg_ld, int B, int C, int rows_per_sample,
                         dp_stream_t stream);
/* x_t = sqrt_ab[t] x0 + sqrt_1mab[t] noise ; x0_hat = (x_t - sqrt_1mab[t] eps) / sqrt_ab[t] */
int dp_q_sample(int dtype, const void* x0, const void* noise, const int64_t* t,
                const float* sqrt_ab, const float* sqrt_1mab, void* xt, int64_t n,
                int64_t per_sample, dp_stream_t stream);
int dp_pred_x0(int dtype, const void* xt, const void* eps, const int64_t* t, const float* sqrt_ab,
               const float* sqrt_1mab, void* out, int64_t n, int64_t per_sample,
               dp_stream_t stream);
/* *loss_acc += scale * sum (pred - target)^2 ; dpred = 2 scale (pred - target) (dpred may be NULL) */
int dp_mse(int dtype, const void* pred, const void* target, void* dpred, float* loss_acc,
           int64_t n, float scale, dp_stream_t stream);
/* sinusoidal embedding [B][dim], cos half first */
int dp_timestep_embed(int dtype, const int64_t* t, void* out, int B, int dim, float max_period,
                      dp_stream_t stream);
/* out[r] = table[ids[r]] (+ pos[r % L]) */
int dp_embed(int dtype, const int64_t* ids, const void* table, const void* pos, void* out,
             int64_t rows, int L, int C, dp_stream_t stream);
/* channel concat of row-major [rows][Ca] and [rows][Cb] (b NULL -> zeros) and its adjoint */
int dp_concat(int dtype, const void* a, const void* b, void* dst, int64_t rows, int Ca, int Cb,
              dp_stream_t stream);
int dp_split(int dtype, const void* src, void* a, void* b, int64_t rows, int Ca, int Cb,
             int acc_a, int acc_b, dp_stream_t stream);
/* NHWC nearest 2x upsample and its adjoint (sum of the 4 copies) */
int dp_upsample2x(int dtype, const void* x, void* y, int N, int H, int W, int C,
                  dp_stream_t stream);
int dp_upsample2x_bwd(int dtype, const void* dy, void* dx, int N, int H, int W, int C,
                      dp_stream_t stream);
/* per-sample channel bias: y[r] = x[r] + e[r / rows_per_sample]; de[b] = sum of dy over sample b */
int dp_row_bias_fwd(int dtype, const void* x, const void* e, int64_t e_ld, void* y, int64_t rows,
                    int C, int rows_per_sample, dp_stream_t stream);
int dp_row_bias_bwd(int dtype, const void* dy, void* de, int64_t de_ld, int B, int C,
                    int rows_per_sample, dp_stream_t stream);
/* as dp_row_bias_bwd, and db[c] += sum over all rows of dy (the bias gradient of the layer that
   produced x, e.g. a ResBlock's first conv) and db2[c] += the same sum (the bias gradient of the layer
   that produced e, e.g. the temb projection: sum_b de[b]) from the same per-sample sums; fp32, NULL -> none */
int dp_row_bias_bwd_db(int dtype, const void* dy, void* de, int64_t de_ld, int B, int C,
                       int rows_per_sample, float* db, float* db2, dp_stream_t stream);
/* NHWC image [N][H][W][C] <-> patches [N][H/p][W/p][p*p*C] (DiT patchify/unpatchify);
   H, W, C describe the image side in both directions */
int dp_space_to_depth(int dtype, const void* x, void* y, int N, int H, int W, int C, int p,
                      int inverse, dp_stream_t stream);
/* db[c] += sum_r dy[r][c]  (bias gradient, fp32 accumulate) */
int dp_bias_grad(int dtype, const void* dy, float* db, int64_t rows, int C, dp_stream_t stream);
int dp_cast(int src_dtype, int dst_dtype, const void* x, void* y, int64_t n, dp_stream_t stream);
/* AdamW (torch.optim.AdamW semantics) over a flat fp32 master buffer; optionally refreshes the
   bf16 compute copy. grad_scale multiplies the gradient first. */
int dp_adamw(float* param, const float* grad, float* exp_avg, float* exp_avg_sq,
             void* param_bf16, int64_t n, float lr, float beta1, float beta2, float eps,
             float weight_decay, int step, float grad_scale, dp_stream_t stream);

/* same update with the step counter on the device (*step_dev is incremented first; bc_dev
   receives the two bias corrections) so that a captured CUDA graph can replay it */
/* chunked AdamW: advance the device step counter / bias corrections once per iteration, then
   update flat slices (e.g. layer by layer while the backward pass still runs) */
int dp_adamw_advance(int* step_dev, float beta1, float beta2, float* bc_dev, dp_stream_t stream);
int dp_adamw_apply(float* param, const float* grad, float* exp_avg, float* exp_avg_sq,
                   void* param_bf16, int64_t n, float lr, float beta1, float beta2, float eps,
                   float weight_decay, const float* bc_dev, float grad_scale, int max_ctas,
                   int zero_grad, dp_stream_t stream);
int dp_adamw_dev(float* param, const float* grad, float* exp_avg, float* exp_avg_sq,
                 void* param_bf16, int64_t n, float lr, float beta1, float beta2, float eps,
                 float weight_decay, int* step_dev, float* bc_dev, float grad_scale,
                 dp_stream_t stream);

/* ---- normalisation and softmax (norm.cu) ---- */
/* GroupNorm(+SiLU) over NHWC [N][HW][C]; gamma/beta fp32 (NULL = no affine); mean/rstd fp32
   [N][G] saved for backward; workspace of dp_group_norm_workspace() bytes. */
size_t dp_group_norm_workspace(int N, int HW, int G);
int dp_group_norm_fwd(int dtype, const void* x, const float* gamma, const float* beta, void* y,
                      float* mean, float* rstd, int N, int HW, int C, int G, float eps, int silu,
                      float* workspace, dp_stream_t stream);
/* GroupNorm(+SiLU) forward from statistics the producer accumulated (DpConvArgs::gn_sums): one pass over x */
int dp_group_norm_fwd_sums(int dtype, const void* x, const float* gamma, const float* beta, void* y,
                           float* mean, float* rstd, int N, int HW, int C, int G, float eps, int silu,
                           const float* sums, dp_stream_t stream);
/* dx (+)= ..., dgamma/dbeta fp32 accumulated (may be NULL) */
int dp_group_norm_bwd(int dtype, const void* x, const void* dy, const float* gamma,
                      const float* beta, const float* mean, const float* rstd, void* dx,
                      float* dgamma, float* dbeta, int N, int HW, int C, int G, int silu,
                      int accumulate, float* workspace, dp_stream_t stream);
/* LayerNorm over rows of C (C <= 2048). Either per-channel affine gamma/beta (fp32) or per-sample
   adaLN modulation y = xhat*(1+mod[b][scale_off+c]) + mod[b][shift_off+c], b = row/rows_per_sample */
/* T5-style RMSNorm forward (frozen encoders): y = x * rsqrt(mean(x^2) + eps) * gamma, rows of C */
int dp_rms_norm_fwd(int dtype, const void* x, const float* gamma, void* y, int64_t rows, int C,
                    float eps, dp_stream_t stream);
int dp_layer_norm_fwd(int dtype, const void* x, const float* gamma, const float* beta,
                      const void* mod, int64_t mod_ld, int shift_off, int scale_off,
                      int rows_per_sample, void* y, float* mean, float* rstd, int64_t rows, int C,
                      float eps, dp_stream_t stream);
int dp_layer_norm_bwd(int dtype, const void* x, const void* dy, const float* gamma,
                      const void* mod, int64_t mod_ld, int shift_off, int scale_off,
                      int rows_per_sample, const float* mean, const float* rstd, void* dx,
                      float* dgamma, float* dbeta, void* dmod, int64_t dmod_ld, int64_t rows,
                      int C, int accumulate, dp_stream_t stream);
/* P = softmax(scale * S) over rows of fp32 scores, row stride ld for S and P
   (causal: col j masked when j > row % Lq) */
int dp_softmax_fwd(int dtype, const float* S, void* P, int64_t rows, int cols, int ld,
                   float scale, int causal, int Lq, dp_stream_t stream);
/* dS = scale * P * (dP - rowsum(dP * P)), row stride ld for P, dP, dS */
int dp_softmax_bwd(int dtype, const void* P, const float* dP, void* dS, int64_t rows, int cols,
                   int ld, float scale, dp_stream_t stream);

/* Launch timing (bench roofline pass): a pool of >= n CUDA events, recorded by index on a stream;
   elapsed milliseconds between two recorded events (-1 on error). */
int dp_timing_events(int n);
int dp_timing_record(int i, dp_stream_t stream);
float dp_timing_elapsed(int i, int j);

const char* dp_last_error(void);
int dp_version(void);

#ifdef __cplusplus
}
#endif
#endif /* DPIPE_H_ */
