// Fused multi-head attention forward for sm_100a (head dim 64), K4 in SURVEY §2.4.
//
// One CTA = one 128-query tile of one (batch, head); 4 warps, thread t owns query row t.
//   * TMA loads Q once and streams 128-key K/V tiles (K and V double-buffered) from the strided
//     [B, N, heads*64] activations (fused qkv / kv tensors, no copies);
//   * thread 0 issues tcgen05.mma: S = Q K^T into TMEM (128 fp32 columns), and O += P V_j into TMEM
//     (64 columns) with P read from TMEM (64 columns of bf16 pairs, the MMA's A operand);
//   * all 128 threads run the online softmax on their S row straight from TMEM (tcgen05.ld) with
//     packed f32x2 math (FFMA2 / FADD2, three-input FMNMX), part of the exponentials on the FMA
//     pipe (ex2_poly2), write P = exp2(S*scale*log2e - m) as bf16 pairs back into TMEM (no
//     shared-memory round trip); the running max moves only past a threshold, so the O rescale in
//     TMEM is rare (FA4-style lazy correction);
//   * epilogue: O / l (TMEM -> registers) staged through shared memory and written by one TMA
//     tensor store, log-sum-exp saved for the backward pass.
// Two CTAs fit per SM (81 KB shared memory, 256 TMEM columns each), so one CTA's softmax
// overlaps the other's MMAs. Keys beyond N_k (cross-attention, 77 tokens) are masked.
#include <cstdlib>
#include <type_traits>
#include <string>
#include <cudaTypedefs.h>
#include "common.cuh"
#include "dpipe.h"

namespace dp {
void set_error(const std::string& s);

namespace fa {

constexpr int BQ = 128, BKV = 128, HD = 64;
constexpr uint32_t TILE_BYTES = BQ * HD * 2;  // 16 KB: Q, K or V tile (128 rows x 128 B)

struct Params {
  int N, Nk, heads;
  float scale_log2;  // softmax scale * log2(e)
  float* lse;        // [B][heads][N] (log2 domain: m + log2(l))
  int causal;        // key j > query i masked (N == Nk)
};

DP_DEV float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// 2^x for x <= 0 on the FMA pipe (degree-3 minimax on [-0.5, 0.5], max rel. error 7.5e-5, far below
// bf16's 3.9e-3): round-to-nearest by the 1.5*2^23 magic add, the polynomial on the fraction as packed
// f32x2 FMAs, the integer part shifted into the exponent field. x is clamped at -126 (2^-126 ~ 0).
// The forward softmax is bound by MUFU.EX2 (16 / clk / SM against 128-wide tensor MMAs), so a share of
// the exponentials is computed here instead (the FA4 split of the exp work between MUFU and FMA).
DP_DEV float2 ex2_poly2(float2 x) {
  x.x = fmaxf(x.x, -126.f);  // round(x) >= -126: p in [0.7, 1.42] keeps a biased exponent >= 0
  x.y = fmaxf(x.y, -126.f);
  const float2 magic = make_float2(12582912.f, 12582912.f);
  const float2 t = __fadd2_rn(x, magic);
  const float2 xi = __fadd2_rn(t, make_float2(-12582912.f, -12582912.f));
  const float2 f = __fadd2_rn(x, make_float2(-xi.x, -xi.y));
  float2 pp = __ffma2_rn(make_float2(0.05517167f, 0.05517167f), f, make_float2(0.24261114f, 0.24261114f));
  pp = __ffma2_rn(pp, f, make_float2(0.69326097f, 0.69326097f));
  pp = __ffma2_rn(pp, f, make_float2(0.99992806f, 0.99992806f));
  return make_float2(__int_as_float(__float_as_int(pp.x) + (__float_as_int(t.x) << 23)),
                     __int_as_float(__float_as_int(pp.y) + (__float_as_int(t.y) << 23)));
}

DP_DEV float max3f(float a, float b, float c) {
  float d;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
  return d;
}

DP_DEV void tma_load_4d_(const CUtensorMap* map, uint64_t* bar, void* dst, int c0, int c1, int c2,
                         int c3) {
  tma_load_4d(map, bar, dst, c0, c1, c2, c3);
}

// EMU: pairs (of the 16 per 32-key chunk) whose exponentials run on the FMA pipe (ex2_poly2)
template <int EMU>
__global__ void __launch_bounds__(128, 2)
    fa_fwd_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                  const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmO,
                  const Params p) {
  DP_PDL_ENTRY();
  extern __shared__ uint8_t smem_raw[];
  // 1024-byte alignment by an offset from the __shared__ array (not an integer round trip), so the
  // compiler keeps the shared address space: LDS/STS instead of generic LD/ST on the LSU path
  const uint32_t pad = (1024u - (smem_u32(smem_raw) & 1023u)) & 1023u;
  uint8_t* smem = smem_raw + pad;
  uint8_t* sQ = smem;
  uint8_t* sK = sQ + TILE_BYTES;          // 2 buffers
  uint8_t* sV = sK + 2 * TILE_BYTES;      // 2 buffers
  // barriers in the alignment slack when it has room, else after the tiles (5 tiles + 1 KB requested)
  uint64_t* bar = reinterpret_cast<uint64_t*>(pad >= 64 ? smem_raw : sV + 2 * TILE_BYTES);
  uint64_t* bar_q = bar;
  uint64_t* bar_k = bar + 1;  // [2]
  uint64_t* bar_v = bar + 3;  // [2]
  uint64_t* bar_s = bar + 5;
  uint64_t* bar_o = bar + 6;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 7);

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int qt = blockIdx.x, h = blockIdx.y, b = blockIdx.z;
  const int q0 = qt * BQ;
  int ntiles = (p.Nk + BKV - 1) / BKV;
  if (p.causal) ntiles = min(ntiles, (q0 + BQ - 1) / BKV + 1);  // tiles past the diagonal are masked

  if (tid == 0) {
    tma_prefetch(&tmQ);
    tma_prefetch(&tmK);
    tma_prefetch(&tmV);
    for (int i = 0; i < 7; ++i) mbar_init(&bar[i], 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc<256>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t t_s = tmem;          // S: columns [0, 128)
  const uint32_t t_o = tmem + 128;    // O: columns [128, 192)
  const uint32_t t_p = tmem + 192;    // P (bf16 pairs, 128 keys): columns [192, 256), A operand of PV
  const uint32_t lane_off = static_cast<uint32_t>(warp * 32) << 16;
  const uint32_t idesc_s = idesc_bf16_f32(BQ, BKV, 0, 0);
  const uint32_t idesc_o = idesc_bf16_f32(BQ, HD, 0, 1);

  // Pipeline per key tile j (one MMA-issuing thread, in-order tensor pipe):
  //   once P(j) is in shared memory, PV(j) (accumulating into O in TMEM) and S(j+1) are issued back
  //   to back; the wait for S(j+1) covers PV(j), so P and O are free for softmax(j+1).
  //   K and V are double-buffered (V(j+1) streams in while tile j's softmax runs).
  auto issue_s = [&](int j) {
    const int kb = j & 1;
    mbar_wait(&bar_k[kb], (j >> 1) & 1);
    tc_fence_after();
    const uint32_t qa = smem_u32(sQ), ka = smem_u32(sK + kb * TILE_BYTES);
#pragma unroll
    for (int k = 0; k < HD / 16; ++k)
      tc_mma_bf16(t_s, smem_desc_sw128(qa + k * 32, 16, 1024), smem_desc_sw128(ka + k * 32, 16, 1024),
                  idesc_s, k > 0 ? 1u : 0u);
    tc_commit(bar_s);
  };
  if (tid == 0) {
    mbar_expect_tx(bar_q, TILE_BYTES);
    tma_load_4d_(&tmQ, bar_q, sQ, 0, q0, h, b);
    for (int t = 0; t < 2 && t < ntiles; ++t) {
      mbar_expect_tx(&bar_k[t], TILE_BYTES);
      tma_load_4d_(&tmK, &bar_k[t], sK + t * TILE_BYTES, 0, t * BKV, h, b);
      mbar_expect_tx(&bar_v[t], TILE_BYTES);
      tma_load_4d_(&tmV, &bar_v[t], sV + t * TILE_BYTES, 0, t * BKV, h, b);
    }
    mbar_wait(bar_q, 0);
    issue_s(0);
  }

  // O accumulates across key tiles in TMEM (PV(j) with accumulate = j > 0). The running max is
  // raised only when a row's max grows by more than RESCALE_T (log2 units, a factor of 256): P then
  // stays <= 256 (exact enough in bf16, fp32 row sums), and the O rescale (TMEM -> registers ->
  // TMEM) is skipped on most tiles instead of folding a register accumulator every tile.
  constexpr float RESCALE_T = 8.f;
  float m_run = -INFINITY, l_run = 0.f;
  const int row = tid;  // query row inside the tile

  for (int j = 0; j < ntiles; ++j) {
    mbar_wait(bar_s, j & 1);  // S(j) done, and (in-order) PV(j-1) too
    tc_fence_after();
    const int valid = p.causal ? min(min(BKV, p.Nk - j * BKV), q0 + row - j * BKV + 1)
                               : min(BKV, p.Nk - j * BKV);
    // the row's 128 scores leave TMEM under one wait
    uint32_t sv[BKV];
#pragma unroll
    for (int c = 0; c < BKV / 32; ++c)
      tmem_ld_32x32(t_s + lane_off + c * 32, *reinterpret_cast<uint32_t(*)[32]>(&sv[c * 32]));
    tmem_ld_wait();
    // full tiles (every row of the warp sees all 128 keys: the common case) run a copy of the
    // softmax without the per-element key mask
    float m_use, alpha, lsum = 0.f;
    float2 ls2[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
    auto softmax_tile = [&](auto full_t) {
      constexpr bool FULL = decltype(full_t)::value;
      float mx = -INFINITY;
      if constexpr (FULL) {
        // four independent FMNMX3 chains (one or two softmax warps per SMSP: latency, not issue, bound)
        float m4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
        for (int i = 0; i < BKV; i += 2)
          m4[(i / 2) & 3] = max3f(m4[(i / 2) & 3], __uint_as_float(sv[i]), __uint_as_float(sv[i + 1]));
        mx = max3f(m4[0], m4[1], fmaxf(m4[2], m4[3]));
      } else {
#pragma unroll
        for (int i = 0; i < BKV; ++i)
          if (i < valid) mx = fmaxf(mx, __uint_as_float(sv[i]));
      }
      const float m_cand = fmaxf(m_run, mx * p.scale_log2);
      if (m_cand - m_run > RESCALE_T) {
        m_use = m_cand;
        alpha = ex2(m_run - m_cand);  // 0 on the first tile
      } else {
        m_use = m_run;
        alpha = 1.f;
      }
      // P = exp2(s*scale - m) -> bf16 pairs -> TMEM (the A operand of PV: no shared-memory round trip);
      // PV(j-1) has read it (complete before S(j)).
      // Packed f32x2 arithmetic (FFMA2 / FADD2) halves the FMA-pipe instructions per score.
      const float2 sc2 = make_float2(p.scale_log2, p.scale_log2), nm2 = make_float2(-m_use, -m_use);
      uint32_t pk[32];  // 64 keys of P as bf16 pairs (one TMEM store per 64 keys)
#pragma unroll
      for (int c = 0; c < BKV / 32; ++c) {
        float pv[32];
#pragma unroll
        for (int i = 0; i < 32; i += 2) {
          const float2 x = __ffma2_rn(make_float2(__uint_as_float(sv[c * 32 + i]), __uint_as_float(sv[c * 32 + i + 1])),
                                      sc2, nm2);
          float2 e;
          // emulated pairs spread over the chunk (every 16/EMU-th pair) so MUFU and FMA work interleave
          if (EMU > 0 && ((i / 2) % (16 / (EMU > 0 ? EMU : 1))) == (16 / (EMU > 0 ? EMU : 1)) - 1) {
            e = ex2_poly2(x);
          } else {
            e.x = ex2(x.x);
            e.y = ex2(x.y);
          }
          if constexpr (!FULL) {
            e.x = (c * 32 + i < valid) ? e.x : 0.f;
            e.y = (c * 32 + i + 1 < valid) ? e.y : 0.f;
          }
          pv[i] = e.x;
          pv[i + 1] = e.y;
          ls2[(i / 2) & 3] = __fadd2_rn(ls2[(i / 2) & 3], e);
        }
#pragma unroll
        for (int i = 0; i < 16; ++i) pk[(c & 1) * 16 + i] = pack_bf16x2(pv[2 * i], pv[2 * i + 1]);
        if (c & 1) tmem_st_32x32(t_p + lane_off + (c >> 1) * 32, pk);  // keys 64*(c>>1) .. +64
      }
    };
    if (__all_sync(0xffffffffu, valid >= BKV))
      softmax_tile(std::true_type{});
    else
      softmax_tile(std::false_type{});
    lsum = (ls2[0].x + ls2[0].y) + (ls2[1].x + ls2[1].y) + ((ls2[2].x + ls2[2].y) + (ls2[3].x + ls2[3].y));
    // rescale O (holding PV(0..j-1), complete before S(j)) where the max moved;
    // warp-collective TMEM access, so a warp rescales when any of its rows needs it
    if (j > 0 && __any_sync(0xffffffffu, alpha != 1.f)) {
#pragma unroll
      for (int c = 0; c < HD / 32; ++c) {
        uint32_t ov[32];
        tmem_ld_32x32(t_o + lane_off + c * 32, ov);
        tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < 32; i += 2) {
          const float2 r = __fmul2_rn(make_float2(__uint_as_float(ov[i]), __uint_as_float(ov[i + 1])),
                                      make_float2(alpha, alpha));
          ov[i] = __float_as_uint(r.x);
          ov[i + 1] = __float_as_uint(r.y);
        }
        tmem_st_32x32(t_o + lane_off + c * 32, ov);
      }
      tmem_st_wait();
    }
    tmem_st_wait();
    tc_fence_before();
    __syncthreads();  // P(j) in TMEM; S(j) read and O rescaled in TMEM by every thread
    if (tid == 0) {
      tc_fence_after();
      const int vb = j & 1;
      mbar_wait(&bar_v[vb], (j >> 1) & 1);
      tc_fence_after();
      const uint32_t va = smem_u32(sV + vb * TILE_BYTES);
#pragma unroll
      for (int k = 0; k < BKV / 16; ++k) {
        const uint64_t bd = smem_desc_sw128(va + k * 2048, 8192, 1024);
        tc_mma_bf16_ts(t_o, t_p + k * 8, bd, idesc_o, (j > 0 || k > 0) ? 1u : 0u);  // 16 keys = 8 columns
      }
      tc_commit(bar_o);
      // S(j+1) behind PV(j): the wait for S(j+1) then also covers PV(j) (in-order tensor pipe), so
      // P and O are free for the next softmax without a second barrier. Measured at 32x5x1024^2
      // against S(j+1) ahead of PV(j) (+ a PV wait before the P store): 86 vs 91 us, and against an
      // S(j+1) issued before softmax(j) through a per-warp "S consumed" barrier: 92 us.
      if (j + 1 < ntiles) {
        issue_s(j + 1);
        // S(j) finished: K buffer j&1 is free for tile j+2
        if (j + 2 < ntiles) {
          mbar_expect_tx(&bar_k[j & 1], TILE_BYTES);
          tma_load_4d_(&tmK, &bar_k[j & 1], sK + (j & 1) * TILE_BYTES, 0, (j + 2) * BKV, h, b);
        }
      }
    }
    l_run = l_run * alpha + lsum;
    m_run = m_use;
    if (tid == 0 && j + 1 < ntiles && j >= 1) {
      // V(j+1) into buffer (j+1)&1 (V(j-1) there was consumed by PV(j-1), complete before S(j))
      mbar_expect_tx(&bar_v[(j + 1) & 1], TILE_BYTES);
      tma_load_4d_(&tmV, &bar_v[(j + 1) & 1], sV + ((j + 1) & 1) * TILE_BYTES, 0, (j + 1) * BKV, h, b);
    }
  }
  // the last PV, then O / l -> shared (SWIZZLE_128B rows of 64 bf16) -> one TMA store
  mbar_wait(bar_o, (ntiles - 1) & 1);
  tc_fence_after();
  const float inv = l_run > 0.f ? 1.f / l_run : 0.f;
  uint8_t* so = sQ;  // Q is free: the last S MMA completed before the last PV
#pragma unroll
  for (int c = 0; c < HD / 32; ++c) {
    uint32_t ov[32];
    tmem_ld_32x32(t_o + lane_off + c * 32, ov);
    tmem_ld_wait();
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      uint4 u;
      u.x = pack_bf16x2(__uint_as_float(ov[q * 8 + 0]) * inv, __uint_as_float(ov[q * 8 + 1]) * inv);
      u.y = pack_bf16x2(__uint_as_float(ov[q * 8 + 2]) * inv, __uint_as_float(ov[q * 8 + 3]) * inv);
      u.z = pack_bf16x2(__uint_as_float(ov[q * 8 + 4]) * inv, __uint_as_float(ov[q * 8 + 5]) * inv);
      u.w = pack_bf16x2(__uint_as_float(ov[q * 8 + 6]) * inv, __uint_as_float(ov[q * 8 + 7]) * inv);
      const int chunk = c * 4 + q;
      *reinterpret_cast<uint4*>(so + row * 128 + ((chunk ^ (row & 7)) * 16)) = u;
    }
  }
  if (p.lse && q0 + row < p.N)
    p.lse[((int64_t)b * p.heads + h) * p.N + q0 + row] = m_run + log2f(l_run);
  fence_async_shared();
  __syncthreads();
  if (tid == 0) {
    tma_store_4d(&tmO, so, 0, q0, h, b);
    bulk_commit();
    bulk_wait_all();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<256>(tmem);
  }
}

constexpr size_t SMEM = 1024 + 5 * TILE_BYTES;

// ------------------------------------------------------------------ backward
// D[b][h][n] = sum_d dO[b][n][h*64+d] * O[b][n][h*64+d]: rows taken in memory order (b, n, h), eight
// threads per 128-byte row (16-byte loads), shuffle reduction inside the 8-lane group
__global__ void __launch_bounds__(256) fa_bwd_prep_kernel(const __nv_bfloat16* __restrict__ o,
                                                          const __nv_bfloat16* __restrict__ dout,
                                                          float* __restrict__ Dv, int B, int N, int heads,
                                                          int64_t o_ld, int64_t do_ld, float* __restrict__ dq_zero,
                                                          float* __restrict__ dkv_zero, int64_t dkv_rows) {
  DP_PDL_ENTRY();
  const int sub = threadIdx.x & 7;
  const int64_t total = (int64_t)B * N * heads;
  const float4 z4 = make_float4(0.f, 0.f, 0.f, 0.f);
  // the fp32 dQ (and split dK / dV) accumulators the backward kernel reduce-adds into are zeroed here,
  // 64-float rows, 8 floats per thread (no separate memset node between the PDL kernels)
  if (dkv_zero)
    for (int64_t r = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 3; r < dkv_rows;
         r += ((int64_t)gridDim.x * blockDim.x) >> 3) {
      float4* d = reinterpret_cast<float4*>(dkv_zero + r * HD + sub * 8);
      d[0] = z4;
      d[1] = z4;
    }
  for (int64_t r = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 3; r < total;
       r += ((int64_t)gridDim.x * blockDim.x) >> 3) {
    if (dq_zero) {  // row r = (b, n, h) of [B][N][heads][64]: the same index order as the loop
      float4* d = reinterpret_cast<float4*>(dq_zero + r * HD + sub * 8);
      d[0] = z4;
      d[1] = z4;
    }
    const int h = static_cast<int>(r % heads);
    const int64_t bn = r / heads;
    const int n = static_cast<int>(bn % N);
    const int b = static_cast<int>(bn / N);
    const uint4 a = *reinterpret_cast<const uint4*>(o + ((int64_t)b * N + n) * o_ld + h * HD + sub * 8);
    const uint4 c = *reinterpret_cast<const uint4*>(dout + ((int64_t)b * N + n) * do_ld + h * HD + sub * 8);
    const __nv_bfloat162* a2 = reinterpret_cast<const __nv_bfloat162*>(&a);
    const __nv_bfloat162* c2 = reinterpret_cast<const __nv_bfloat162*>(&c);
    float s = 0.f;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float2 fa = __bfloat1622float2(a2[j]), fc = __bfloat1622float2(c2[j]);
      s = fmaf(fa.x, fc.x, fmaf(fa.y, fc.y, s));
    }
    s += __shfl_xor_sync(0xffffffffu, s, 1);
    s += __shfl_xor_sync(0xffffffffu, s, 2);
    s += __shfl_xor_sync(0xffffffffu, s, 4);
    if (sub == 0) Dv[((int64_t)b * heads + h) * N + n] = s;
  }
}

// out[b][n][h*64+d] (bf16, token stride out_ld) = alpha * acc[b][n][h][d] (fp32, dense): 8 elements
// per thread (two 16-byte loads, one 16-byte store)
__global__ void fa_dq_cast_kernel(const float* __restrict__ acc, __nv_bfloat16* __restrict__ out,
                                  int64_t rows, int C, int64_t out_ld, float alpha) {
  DP_PDL_ENTRY();
  const int cv = C / 8;
  const int64_t n = rows * cv;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / cv;
    const int c = static_cast<int>(i - r * cv) * 8;
    const float4 u = reinterpret_cast<const float4*>(acc)[2 * i];
    const float4 v = reinterpret_cast<const float4*>(acc)[2 * i + 1];
    uint4 o;
    o.x = pack_bf16x2(alpha * u.x, alpha * u.y);
    o.y = pack_bf16x2(alpha * u.z, alpha * u.w);
    o.z = pack_bf16x2(alpha * v.x, alpha * v.y);
    o.w = pack_bf16x2(alpha * v.z, alpha * v.w);
    *reinterpret_cast<uint4*>(out + r * out_ld + c) = o;
  }}

struct BwdParams {
  int N, Nk, heads;
  float scale_log2;   // softmax scale * log2(e)
  float scale;        // softmax scale (dS -> dS_raw)
  const float* lse;   // [B][heads][N]
  const float* Dv;    // [B][heads][N]
  float* dq_acc;      // [B][N][heads][64] fp32, zero-initialised (reduced into by TMA: tmDQ)
  int qsplit;         // CTAs per key tile (query tiles split between them)
  int dq_direct;      // one key tile (Nk <= 128): each dQ tile has one producer -> scaled bf16 written
                      // by a TMA store through tmDQ (no fp32 accumulator, memset or cast pass)
  float* dkv_acc;     // qsplit > 1: [2][B][Nk][heads][64] fp32 dK (unscaled), dV, zero-initialised
};

// One CTA = one 128-key tile of one (batch, head); thread t owns key row t (S^T, dP^T rows).
// Per 128-query tile: S^T = K Q^T, dP^T = V dO^T (TMEM); P^T = exp2(S^T*sl - lse) -> TMEM (bf16,
// the A operand of dV += P^T dO), dS^T = P^T (dP^T - D) -> shared (bf16, K-major over queries);
// dK += dS^T Q (TMEM accumulators across query tiles), dQ_i = dS K (TMEM) -> staged, TMA reduce-add.
constexpr uint32_t BWD_SMEM_TILES = 10;  // K, V, Q[3], dO[3], dS^T (2)
constexpr int NQB = 3;                   // Q / dO buffers: tile li+1 is loaded a full tile ahead

__global__ void __launch_bounds__(256, 1)
    fa_bwd_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                  const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmDO,
                  const __grid_constant__ CUtensorMap tmDK, const __grid_constant__ CUtensorMap tmDV,
                  const __grid_constant__ CUtensorMap tmDQ, const BwdParams p) {
  DP_PDL_ENTRY();
  extern __shared__ uint8_t smem_raw[];
  // 1024-byte alignment by an offset from the __shared__ array (not an integer round trip), so the
  // compiler keeps the shared address space: LDS/STS instead of generic LD/ST on the LSU path
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sK = smem;
  uint8_t* sV = sK + TILE_BYTES;
  uint8_t* sQ = sV + TILE_BYTES;          // [NQB]
  uint8_t* sDO = sQ + NQB * TILE_BYTES;   // [NQB]
  uint8_t* sDST = sDO + NQB * TILE_BYTES; // 2 blocks (queries 0-63, 64-127)
  // dQ_i staging (128 query rows x 64 fp32, 256-byte rows): one TMA reduce-add per query tile
  // instead of 2048 per-thread vector atomics (those saturated the LSU queue, lg_throttle)
  float* sDQ = reinterpret_cast<float*>(sDST + 2 * TILE_BYTES);
  float* sLse = sDQ + BQ * HD;                                     // [2][128]
  float* sD = sLse + 256;                                          // [2][128]
  uint64_t* bar = reinterpret_cast<uint64_t*>(sD + 256);
  uint64_t* bar_kv = bar;
  uint64_t* bar_q = bar + 1;   // [NQB]
  uint64_t* bar_sp = bar + 1 + NQB;
  uint64_t* bar_acc = bar + 2 + NQB;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 3 + NQB);

  // 8 warps: warps w and w+4 share TMEM lanes 32*(w%4).. (key rows) and split the 128 query
  // columns of every S^T / dP^T tile (and the 64 dQ / dK / dV columns) between them
  const int tid = threadIdx.x;
  const int warp = tid >> 5;
  const int row = tid & 127;   // key row (TMEM lane) of this thread
  const int half = tid >> 7;   // column half
  const int kt = blockIdx.x / p.qsplit, h = blockIdx.y, b = blockIdx.z;
  const int k0 = kt * BKV;
  const int nq = (p.N + BQ - 1) / BQ;
  // query tiles [i0, i1) of this CTA (split when there are too few key tiles to fill the SMs)
  const int per = (nq + p.qsplit - 1) / p.qsplit;
  const int i0 = (blockIdx.x % p.qsplit) * per;
  const int i1 = min(nq, i0 + per);
  const int64_t bh = (int64_t)b * p.heads + h;

  if (tid == 0) {
    tma_prefetch(&tmQ);
    tma_prefetch(&tmK);
    tma_prefetch(&tmV);
    tma_prefetch(&tmDO);
    for (int i = 0; i < 3 + NQB; ++i) mbar_init(&bar[i], 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t t_st = tmem, t_dpt = tmem + 128, t_dv = tmem + 256, t_dk = tmem + 320, t_dq = tmem + 384;
  const uint32_t t_p = tmem + 448;  // P^T of the tile in flight, bf16 pairs (64 columns = 128 queries)
  const uint32_t lane_off = static_cast<uint32_t>((warp & 3) * 32) << 16;

  auto load_q = [&](int i, int buf) {
    mbar_expect_tx(&bar_q[buf], 2 * TILE_BYTES);
    tma_load_4d(&tmQ, &bar_q[buf], sQ + buf * TILE_BYTES, 0, i * BQ, h, b);
    tma_load_4d(&tmDO, &bar_q[buf], sDO + buf * TILE_BYTES, 0, i * BQ, h, b);
  };
  if (tid == 0) {
    mbar_expect_tx(bar_kv, 2 * TILE_BYTES);
    tma_load_4d(&tmK, bar_kv, sK, 0, k0, h, b);
    tma_load_4d(&tmV, bar_kv, sV, 0, k0, h, b);
    for (int t = 0; t < NQB && i0 + t < i1; ++t) load_q(i0 + t, t);
  }
  // lse / D of the first query tile (rows >= N: lse = +inf -> P = 0)
  auto load_rows = [&](int i, int buf) {
    if (half) return;
    const int q = i * BQ + row;
    sLse[buf * 128 + row] = q < p.N ? p.lse[bh * p.N + q] : INFINITY;
    sD[buf * 128 + row] = q < p.N ? p.Dv[bh * p.N + q] : 0.f;
  };
  load_rows(i0, 0);
  const uint32_t id_sq = idesc_bf16_f32(BKV, BQ, 0, 0);  // S^T / dP^T: M=keys, N=queries, K=64
  const uint32_t id_acc = idesc_bf16_f32(BKV, HD, 0, 1); // dV / dK: M=keys, N=64, K=queries (dV: A in TMEM)
  const uint32_t id_dq = idesc_bf16_f32(BQ, HD, 1, 1);   // dQ: M=queries (A MN-major), N=64
  const bool key_valid = k0 + row < p.Nk;

  // Pipeline (one issuing thread, in-order tensor pipe): at the end of tile li's softmax thread 0
  // issues S^T / dP^T of tile li+1 FIRST and then tile li's accumulator MMAs (dV, dK += ..., dQ_li),
  // so the next softmax starts after 512 MMA cycles and runs while the accumulators (768 cycles)
  // drain; it waits for them only before it overwrites P^T / dS^T in shared memory, and then drains
  // dQ_li from TMEM (a tile late). The previous order (accumulators, then the next S^T / dP^T, and
  // every warp waiting for the accumulators before the next tile) left the softmax warps idle a
  // third of the kernel (ncu: the bar_acc wait was the top stall).
  auto issue_sdp = [&](int li) {  // li: tile index local to this CTA
    const int qb = li % NQB;
    if (li == 0) mbar_wait(bar_kv, 0);
    mbar_wait(&bar_q[qb], (li / NQB) & 1);
    tc_fence_after();
    const uint32_t ka = smem_u32(sK), va = smem_u32(sV);
    const uint32_t qa = smem_u32(sQ + qb * TILE_BYTES), da = smem_u32(sDO + qb * TILE_BYTES);
#pragma unroll
    for (int k = 0; k < HD / 16; ++k) {
      tc_mma_bf16(t_st, smem_desc_sw128(ka + k * 32, 16, 1024), smem_desc_sw128(qa + k * 32, 16, 1024),
                  id_sq, k > 0 ? 1u : 0u);
      tc_mma_bf16(t_dpt, smem_desc_sw128(va + k * 32, 16, 1024), smem_desc_sw128(da + k * 32, 16, 1024),
                  id_sq, k > 0 ? 1u : 0u);
    }
    tc_commit(bar_sp);
  };
  auto issue_acc = [&](int li) {
    const int qb = li % NQB;
    const uint32_t dsa = smem_u32(sDST), ka = smem_u32(sK);
    const uint32_t qa = smem_u32(sQ + qb * TILE_BYTES), da = smem_u32(sDO + qb * TILE_BYTES);
#pragma unroll
    for (int k = 0; k < BQ / 16; ++k) {
      const uint32_t aoff = (k >> 2) * TILE_BYTES + (k & 3) * 32;  // K-major over queries
      // dV += P^T dO    (A = P^T from TMEM: 16 queries = 8 columns; B(n=d, k=q) = dO[q][d]: MN-major)
      tc_mma_bf16_ts(t_dv, t_p + k * 8, smem_desc_sw128(da + k * 2048, 8192, 1024), id_acc,
                     (li > 0 || k > 0) ? 1u : 0u);
      // dK += dS^T Q    (B(n=d, k=q) = Q[q][d]: MN-major)
      tc_mma_bf16(t_dk, smem_desc_sw128(dsa + aoff, 16, 1024), smem_desc_sw128(qa + k * 2048, 8192, 1024),
                  id_acc, (li > 0 || k > 0) ? 1u : 0u);
    }
#pragma unroll
    for (int k = 0; k < BKV / 16; ++k) {
      // dQ_i = dS K: A(m=q, k=key) = dS^T[key][q] (MN-major, 64-query chunks 16 KB apart),
      //              B(n=d, k=key) = K[key][d] (MN-major)
      tc_mma_bf16(t_dq, smem_desc_sw128(dsa + k * 2048, TILE_BYTES, 1024),
                  smem_desc_sw128(ka + k * 2048, 8192, 1024), id_dq, k > 0 ? 1u : 0u);
    }
    tc_commit(bar_acc);
  };
  // dQ of query tile `i` (TMEM, complete) -> the staging buffer: half-buffer `half` holds 128 rows x
  // 32 fp32 (128 B) in the SWIZZLE_128B layout of tmDQ's box (16-byte chunk k of row r at k ^ (r & 7))
  auto drain_dq = [&]() {
    uint32_t v[32];
    tmem_ld_32x32(t_dq + lane_off + half * 32, v);
    tmem_ld_wait();
    if (p.dq_direct) {
      // bf16 tile of 128-byte rows (64 dims): this half's 4 chunks, SWIZZLE_128B like tmQ
      uint8_t* dst = reinterpret_cast<uint8_t*>(sDQ) + row * 128;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        uint4 u;
        u.x = pack_bf16x2(p.scale * __uint_as_float(v[k * 8 + 0]), p.scale * __uint_as_float(v[k * 8 + 1]));
        u.y = pack_bf16x2(p.scale * __uint_as_float(v[k * 8 + 2]), p.scale * __uint_as_float(v[k * 8 + 3]));
        u.z = pack_bf16x2(p.scale * __uint_as_float(v[k * 8 + 4]), p.scale * __uint_as_float(v[k * 8 + 5]));
        u.w = pack_bf16x2(p.scale * __uint_as_float(v[k * 8 + 6]), p.scale * __uint_as_float(v[k * 8 + 7]));
        *reinterpret_cast<uint4*>(dst + (((half * 4 + k) ^ (row & 7)) * 16)) = u;
      }
    } else {
      uint8_t* dst = reinterpret_cast<uint8_t*>(sDQ) + half * (BQ * 128) + row * 128;
#pragma unroll
      for (int k = 0; k < 8; ++k)
        *reinterpret_cast<float4*>(dst + ((k ^ (row & 7)) * 16)) =
            make_float4(__uint_as_float(v[k * 4]), __uint_as_float(v[k * 4 + 1]), __uint_as_float(v[k * 4 + 2]),
                        __uint_as_float(v[k * 4 + 3]));
    }
  };
  auto emit_dq = [&](int i) {  // thread 0: the staged dQ of query tile i -> global
    if (p.dq_direct) {
      tma_store_4d(&tmDQ, sDQ, 0, i * BQ, h, b);
    } else {
      tma_reduce_add_4d(&tmDQ, sDQ, h * HD, i * BQ, b, 0);
      tma_reduce_add_4d(&tmDQ, reinterpret_cast<uint8_t*>(sDQ) + BQ * 128, h * HD + 32, i * BQ, b, 0);
    }
    bulk_commit();
  };
  if (tid == 0) issue_sdp(0);
  // lse / D rows of the tile after next, loaded a tile ahead of their shared-memory store so the
  // global load latency is not exposed inside the loop
  float nxt_lse = INFINITY, nxt_d = 0.f;
  auto fetch_rows = [&](int i) {
    if (half || i >= i1) return;
    const int q = i * BQ + row;
    nxt_lse = q < p.N ? p.lse[bh * p.N + q] : INFINITY;
    nxt_d = q < p.N ? p.Dv[bh * p.N + q] : 0.f;
  };
  fetch_rows(i0 + 1);
  __syncthreads();  // sLse/sD of the first tile

  for (int i = i0; i < i1; ++i) {
    const int li = i - i0;
    const int qb = li & 1;
    mbar_wait(bar_sp, li & 1);
    tc_fence_after();
    const float* lse = sLse + qb * 128;
    const float* Dq = sD + qb * 128;
    uint32_t sva[2][32], dva[2][32];  // both 32-query chunks of this half, one TMEM wait
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      tmem_ld_32x32(t_st + lane_off + (half * 2 + u) * 32, sva[u]);
      tmem_ld_32x32(t_dpt + lane_off + (half * 2 + u) * 32, dva[u]);
    }
    tmem_ld_wait();
    // P^T and dS^T of this thread's 64 queries, packed to bf16 in registers until the previous
    // tile's accumulator MMAs have released the shared-memory operands
    uint32_t ppk[2][16], dpk[2][16];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int c = half * 2 + u;
#pragma unroll
      for (int j = 0; j < 32; j += 2) {
        const int q = c * 32 + j;
        const float2 x = __ffma2_rn(make_float2(__uint_as_float(sva[u][j]), __uint_as_float(sva[u][j + 1])),
                                    make_float2(p.scale_log2, p.scale_log2), make_float2(-lse[q], -lse[q + 1]));
        const float p0 = key_valid ? ex2(x.x) : 0.f, p1 = key_valid ? ex2(x.y) : 0.f;
        const float2 ds = __fmul2_rn(make_float2(p0, p1),
                                     __fadd2_rn(make_float2(__uint_as_float(dva[u][j]), __uint_as_float(dva[u][j + 1])),
                                                make_float2(-Dq[q], -Dq[q + 1])));
        ppk[u][j / 2] = pack_bf16x2(p0, p1);
        dpk[u][j / 2] = pack_bf16x2(ds.x, ds.y);
      }
    }
    if (li > 0) {
      mbar_wait(bar_acc, (li - 1) & 1);  // tile li-1's dV / dK / dQ MMAs done (they read P^T / sDST)
      tc_fence_after();
      if (tid == 0) {
        // the Q/dO buffer of tile li-1 is free: tile li+2 goes there (tile li+1 arrived a tile ago)
        if (i + 2 < i1) load_q(i + 2, (li + 2) % NQB);
        bulk_wait_read<0>();  // the staged dQ of tile li-2 has been read
      }
      __syncthreads();
      drain_dq();
    }
    // P^T -> TMEM (this thread's key row, its 64 queries = 32 columns), dS^T -> shared memory
    tmem_st_32x32(t_p + lane_off + half * 32, *reinterpret_cast<uint32_t(*)[32]>(&ppk[0][0]));
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int c = half * 2 + u;
      const int blk = c >> 1;
#pragma unroll
      for (int q4 = 0; q4 < 4; ++q4) {
        const int chunk = (c & 1) * 4 + q4;
        const int off = blk * TILE_BYTES + row * 128 + ((chunk ^ (row & 7)) * 16);
        *reinterpret_cast<uint4*>(sDST + off) =
            make_uint4(dpk[u][q4 * 4], dpk[u][q4 * 4 + 1], dpk[u][q4 * 4 + 2], dpk[u][q4 * 4 + 3]);
      }
    }
    tmem_st_wait();
    if (!half && i + 1 < i1) {  // rows of tile i+1 (loaded a tile ago) -> the other buffer
      sLse[(qb ^ 1) * 128 + row] = nxt_lse;
      sD[(qb ^ 1) * 128 + row] = nxt_d;
    }
    fetch_rows(i + 2);
    fence_async_shared();
    tc_fence_before();
    __syncthreads();  // P^T / dS^T (and dQ of tile li-1) staged; S^T / dP^T of tile li read
    if (tid == 0) {
      tc_fence_after();
      if (li > 0) emit_dq(i - 1);
      if (i + 1 < i1) issue_sdp(li + 1);
      issue_acc(li);
    }
  }
  // the last tile's accumulators, then its dQ
  if (i1 > i0) {
    mbar_wait(bar_acc, (i1 - 1 - i0) & 1);
    tc_fence_after();
    if (tid == 0) bulk_wait_read<0>();
    __syncthreads();
    drain_dq();
    fence_async_shared();
    __syncthreads();
    if (tid == 0) {
      emit_dq(i1 - 1);
      bulk_wait_all();
    }
  }
  tc_fence_after();
  if (p.qsplit > 1) {
    // partial dK / dV over this CTA's query tiles -> fp32 atomics (scale and bf16 cast afterwards)
    const int c = half;
    uint32_t vk[32], vv[32];
    tmem_ld_32x32(t_dk + lane_off + c * 32, vk);
    tmem_ld_32x32(t_dv + lane_off + c * 32, vv);
    tmem_ld_wait();
    if (key_valid) {
      const int64_t off = (((int64_t)b * p.Nk + k0 + row) * p.heads + h) * HD + c * 32;
      const int64_t plane = (int64_t)gridDim.z * p.Nk * p.heads * HD;
#pragma unroll
      for (int j = 0; j < 32; j += 4) {
        atomicAdd(reinterpret_cast<float4*>(p.dkv_acc + off + j),
                  make_float4(__uint_as_float(vk[j]), __uint_as_float(vk[j + 1]), __uint_as_float(vk[j + 2]),
                              __uint_as_float(vk[j + 3])));
        atomicAdd(reinterpret_cast<float4*>(p.dkv_acc + plane + off + j),
                  make_float4(__uint_as_float(vv[j]), __uint_as_float(vv[j + 1]), __uint_as_float(vv[j + 2]),
                              __uint_as_float(vv[j + 3])));
      }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
      tc_fence_after();
      tmem_dealloc<512>(tmem);
    }
    return;
  }
  // dK (scaled), dV -> bf16 -> shared (reuse the Q buffers) -> TMA stores (thread = key row)
  uint8_t* sdk = sQ;
  uint8_t* sdv = sQ + TILE_BYTES;
  {
    const int c = half;
    uint32_t vk[32], vv[32];
    tmem_ld_32x32(t_dk + lane_off + c * 32, vk);
    tmem_ld_32x32(t_dv + lane_off + c * 32, vv);
    tmem_ld_wait();
#pragma unroll
    for (int q4 = 0; q4 < 4; ++q4) {
      const int chunk = c * 4 + q4;
      const int off = row * 128 + ((chunk ^ (row & 7)) * 16);
      uint4 u;
      u.x = pack_bf16x2(p.scale * __uint_as_float(vk[q4 * 8 + 0]), p.scale * __uint_as_float(vk[q4 * 8 + 1]));
      u.y = pack_bf16x2(p.scale * __uint_as_float(vk[q4 * 8 + 2]), p.scale * __uint_as_float(vk[q4 * 8 + 3]));
      u.z = pack_bf16x2(p.scale * __uint_as_float(vk[q4 * 8 + 4]), p.scale * __uint_as_float(vk[q4 * 8 + 5]));
      u.w = pack_bf16x2(p.scale * __uint_as_float(vk[q4 * 8 + 6]), p.scale * __uint_as_float(vk[q4 * 8 + 7]));
      *reinterpret_cast<uint4*>(sdk + off) = u;
      u.x = pack_bf16x2(__uint_as_float(vv[q4 * 8 + 0]), __uint_as_float(vv[q4 * 8 + 1]));
      u.y = pack_bf16x2(__uint_as_float(vv[q4 * 8 + 2]), __uint_as_float(vv[q4 * 8 + 3]));
      u.z = pack_bf16x2(__uint_as_float(vv[q4 * 8 + 4]), __uint_as_float(vv[q4 * 8 + 5]));
      u.w = pack_bf16x2(__uint_as_float(vv[q4 * 8 + 6]), __uint_as_float(vv[q4 * 8 + 7]));
      *reinterpret_cast<uint4*>(sdv + off) = u;
    }
  }
  fence_async_shared();
  __syncthreads();
  if (tid == 0) {
    tma_store_4d(&tmDK, sdk, 0, k0, h, b);
    tma_store_4d(&tmDV, sdv, 0, k0, h, b);
    bulk_commit();
    bulk_wait_all();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

constexpr size_t BWD_SMEM = 1024 + BWD_SMEM_TILES * TILE_BYTES + BQ * HD * 4 + 4 * 256 * 4 + 64;

}  // namespace fa

PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder();

// 4-D bf16 map over a [B][N][heads*64] view: dims {64, N, heads, B}, box {64, 128, 1, 1}.
static int fa_map(CUtensorMap* map, const void* base, int N, int heads, int B, int64_t ld,
                  int64_t bstride) {
  auto fn = tensor_map_encoder();
  if (!fn) {
    set_error("cuTensorMapEncodeTiled unavailable");
    return DP_ERR_DRIVER;
  }
  if (reinterpret_cast<uintptr_t>(base) % 16 || (ld * 2) % 16 || (bstride * 2) % 16) {
    set_error("flash attention: 16-byte aligned base and strides required");
    return DP_ERR_ARGS;
  }
  cuuint64_t gdim[4] = {64, (cuuint64_t)N, (cuuint64_t)heads, (cuuint64_t)B};
  cuuint64_t gstr[3] = {(cuuint64_t)(ld * 2), 128, (cuuint64_t)(bstride * 2)};
  cuuint32_t box[4] = {64, 128, 1, 1};
  cuuint32_t es[4] = {1, 1, 1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(base), gdim, gstr, box,
                  es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("flash attention: cuTensorMapEncodeTiled failed");
    return DP_ERR_DRIVER;
  }
  return 0;
}

}  // namespace dp

extern "C" int dp_flash_attn_fwd(const DpAttnArgs* a, dp_stream_t stream) {
  using namespace dp;
  if (a->head_dim != 64 || a->dtype != DP_BF16) {
    set_error("dp_flash_attn_fwd: bf16, head_dim 64 only");
    return DP_ERR_UNSUPPORTED;
  }
  if (a->causal && a->N != a->Nk) {
    set_error("dp_flash_attn_fwd: causal masking needs N == Nk");
    return DP_ERR_ARGS;
  }
  if (a->B <= 0 || a->N <= 0 || a->Nk <= 0) return 0;
  CUtensorMap mq, mk, mv, mo;
  if (int e = fa_map(&mq, a->q, a->N, a->heads, a->B, a->q_ld, a->q_bs)) return e;
  if (int e = fa_map(&mk, a->k, a->Nk, a->heads, a->B, a->kv_ld, a->kv_bs)) return e;
  if (int e = fa_map(&mv, a->v, a->Nk, a->heads, a->B, a->kv_ld, a->kv_bs)) return e;
  if (int e = fa_map(&mo, a->o, a->N, a->heads, a->B, a->o_ld, a->o_bs)) return e;
  // share of the softmax exponentials emulated on the FMA pipe: EMU of every 16 pairs (DP_FA_EMU:
  // experiments; 0, 1, 2, 4 or 8)
  static const int emu = [] {
    const char* e = getenv("DP_FA_EMU");
    const int v = e ? atoi(e) : 4;
    return (v == 0 || v == 1 || v == 2 || v == 4 || v == 8) ? v : 4;
  }();
  auto kern = emu == 0 ? fa::fa_fwd_kernel<0> : emu == 1 ? fa::fa_fwd_kernel<1> : emu == 2 ? fa::fa_fwd_kernel<2>
            : emu == 8 ? fa::fa_fwd_kernel<8> : fa::fa_fwd_kernel<4>;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(fa::SMEM));
    if (e != cudaSuccess) {
      set_error(std::string("flash attention attr: ") + cudaGetErrorString(e));
      return e;
    }
    attr = true;
  }
  fa::Params p{a->N, a->Nk, a->heads, a->scale * 1.4426950408889634f, a->lse, a->causal};
  dim3 grid((a->N + fa::BQ - 1) / fa::BQ, a->heads, a->B);
  launch_k(kern, dim3(grid), dim3(128), fa::SMEM, reinterpret_cast<cudaStream_t>(stream), mq, mk, mv,
           mo, p);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error(std::string("flash attention launch: ") + cudaGetErrorString(e));
    return e;
  }
  return 0;
}

// query-tile split of the backward: key-tile CTAs x heads x batch below two per SM -> give each key tile
// several CTAs (each a contiguous range of query tiles, dK/dV reduced with fp32 atomics)
static int fa_bwd_qsplit(const DpAttnArgs* a) {
  using namespace dp;
  const long long nkt = (a->Nk + fa::BKV - 1) / fa::BKV;
  const int nq = (a->N + fa::BQ - 1) / fa::BQ;
  const long long ctas = nkt * a->heads * a->B;
  static const int forced = [] {
    const char* e = getenv("DP_FA_QSPLIT");  // experiments only
    return e ? atoi(e) : 0;
  }();
  if (forced > 0) return forced <= nq ? forced : nq;
  if (ctas >= 2LL * 148 || nq < 2) return 1;
  int q = static_cast<int>((2LL * 148 + ctas - 1) / ctas);
  if (q > nq) q = nq;
  const int per = (nq + q - 1) / q;
  return (nq + per - 1) / per;  // no empty splits
}

extern "C" int64_t dp_flash_attn_bwd_workspace(const DpAttnArgs* a) {
  const int64_t C = (int64_t)a->heads * 64;
  int64_t floats = (int64_t)a->B * a->heads * a->N + (int64_t)a->B * a->N * C;
  if (fa_bwd_qsplit(a) > 1) floats += 2 * (int64_t)a->B * a->Nk * C;
  return floats * 4;
}

extern "C" int dp_flash_attn_bwd(const DpAttnArgs* a, const void* dout, int64_t do_ld, void* dq,
                                 int64_t dq_ld, void* dk, void* dv, int64_t dkv_ld, float* workspace,
                                 dp_stream_t stream) {
  using namespace dp;
  if (a->head_dim != 64 || a->dtype != DP_BF16 || a->causal) {
    set_error("dp_flash_attn_bwd: bf16, head_dim 64, non-causal only");
    return DP_ERR_UNSUPPORTED;
  }
  if (a->B <= 0 || a->N <= 0 || a->Nk <= 0) return 0;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const int C = a->heads * 64;
  const int64_t rows = (int64_t)a->B * a->N;
  float* Dv = workspace;                                   // [B][heads][N]
  float* dq_acc = workspace + (int64_t)a->B * a->heads * a->N;  // [B][N][heads][64]
  const bool dq_direct = a->Nk <= fa::BKV;
  const int qsplit = fa_bwd_qsplit(a);
  float* dkv_acc = dq_acc + rows * C;  // [2][B][Nk][heads][64] (split only)
  const int64_t kv_rows = (int64_t)a->B * a->Nk;
  // accumulators zeroed by the prep kernel (16-byte stores) when aligned, else by memsets
  const bool zero_in_prep = (reinterpret_cast<uintptr_t>(dq_acc) & 15) == 0;
  if (!zero_in_prep) {
    if (!dq_direct) cudaMemsetAsync(dq_acc, 0, sizeof(float) * rows * C, st);
    if (qsplit > 1) cudaMemsetAsync(dkv_acc, 0, sizeof(float) * 2 * kv_rows * C, st);
  }
  {
    const int64_t total = (int64_t)a->B * a->heads * a->N;
    int gp = static_cast<int>((total * 8 + 255) / 256);
    if (gp > 148 * 8) gp = 148 * 8;
    launch_k(fa::fa_bwd_prep_kernel, dim3(gp), dim3(256), 0, st,
        reinterpret_cast<const __nv_bfloat16*>(a->o), reinterpret_cast<const __nv_bfloat16*>(dout), Dv, a->B,
        a->N, a->heads, a->o_ld, do_ld, (dq_direct || !zero_in_prep) ? nullptr : dq_acc,
        (qsplit > 1 && zero_in_prep) ? dkv_acc : nullptr,
        2 * kv_rows * a->heads);
  }
  CUtensorMap mq, mk, mv, mdo, mdk, mdv;
  if (int e = fa_map(&mq, a->q, a->N, a->heads, a->B, a->q_ld, a->q_bs)) return e;
  if (int e = fa_map(&mk, a->k, a->Nk, a->heads, a->B, a->kv_ld, a->kv_bs)) return e;
  if (int e = fa_map(&mv, a->v, a->Nk, a->heads, a->B, a->kv_ld, a->kv_bs)) return e;
  if (int e = fa_map(&mdo, dout, a->N, a->heads, a->B, do_ld, a->N * do_ld)) return e;
  if (int e = fa_map(&mdk, dk, a->Nk, a->heads, a->B, dkv_ld, a->Nk * dkv_ld)) return e;
  if (int e = fa_map(&mdv, dv, a->Nk, a->heads, a->B, dkv_ld, a->Nk * dkv_ld)) return e;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(fa::fa_bwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(fa::BWD_SMEM));
    if (e != cudaSuccess) {
      set_error(std::string("flash attention bwd attr: ") + cudaGetErrorString(e));
      return e;
    }
    attr = true;
  }
  // dq_acc [B][N][C] fp32: dims {C, N, B, 1}, box {32, 128, 1, 1} (128-byte rows, SWIZZLE_128B);
  // dq_direct: the bf16 dq itself, mapped like q
  CUtensorMap mdq;
  if (dq_direct) {
    if (int e = fa_map(&mdq, dq, a->N, a->heads, a->B, dq_ld, a->N * dq_ld)) return e;
  } else {
    auto fn = tensor_map_encoder();
    cuuint64_t gdim[4] = {(cuuint64_t)C, (cuuint64_t)a->N, (cuuint64_t)a->B, 1};
    cuuint64_t gstr[3] = {(cuuint64_t)C * 4, (cuuint64_t)a->N * C * 4, (cuuint64_t)a->B * a->N * C * 4};
    cuuint32_t box[4] = {32, 128, 1, 1};
    cuuint32_t es[4] = {1, 1, 1, 1};
    if (!fn || fn(&mdq, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, dq_acc, gdim, gstr, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
      set_error("flash attention bwd: dQ tensor map encode failed");
      return DP_ERR_DRIVER;
    }
  }
  fa::BwdParams p{a->N, a->Nk, a->heads, a->scale * 1.4426950408889634f, a->scale, a->lse, Dv, dq_acc,
                  qsplit, dq_direct ? 1 : 0, dkv_acc};
  dim3 grid((a->Nk + fa::BKV - 1) / fa::BKV * qsplit, a->heads, a->B);
  launch_k(fa::fa_bwd_kernel, dim3(grid), dim3(256), fa::BWD_SMEM, st, mq, mk, mv, mdo, mdk, mdv, mdq, p);
  if (qsplit > 1) {
    const int64_t nk2 = kv_rows * C / 8;
    int gk = static_cast<int>((nk2 + 255) / 256);
    if (gk > 148 * 8) gk = 148 * 8;
    launch_k(fa::fa_dq_cast_kernel, dim3(gk), dim3(256), 0, st, dkv_acc, reinterpret_cast<__nv_bfloat16*>(dk),
             kv_rows, C, dkv_ld, a->scale);
    launch_k(fa::fa_dq_cast_kernel, dim3(gk), dim3(256), 0, st, dkv_acc + kv_rows * C,
             reinterpret_cast<__nv_bfloat16*>(dv), kv_rows, C, dkv_ld, 1.0f);
  }
  if (!dq_direct) {
    const int64_t n2 = rows * C / 8;
    int g = static_cast<int>((n2 + 255) / 256);
    if (g > 148 * 8) g = 148 * 8;
    launch_k(fa::fa_dq_cast_kernel, dim3(g), dim3(256), 0, st, dq_acc, reinterpret_cast<__nv_bfloat16*>(dq), rows,
             C, dq_ld, a->scale);
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error(std::string("flash attention bwd launch: ") + cudaGetErrorString(e));
    return e;
  }
  return 0;
}
