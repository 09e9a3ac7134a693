// Tensor-core GEMM / implicit-GEMM convolution for sm_100a (tcgen05 + TMEM + TMA),
// plus the fp32 SIMT GEMM used by the fp32 (parity) configuration.
//
// One persistent, warp-specialised kernel serves every contraction of the
// training step:
//   warp 0 (1 thread)   TMA producer: fills a STAGES-deep smem ring (A 128x64, B BNx64)
//   warp 1 (1 thread)   MMA issuer: 4 x tcgen05.mma (128 x BN x 16) per k-block into TMEM
//   warp 2              TMEM allocator (2 accumulator buffers of BN fp32 columns)
//   warps 4-11          epilogue, two warps per TMEM lane quadrant (even / odd 32-column chunks):
//                       tcgen05.ld -> alpha/bias/residual -> bf16 TMA tensor store, or fp32 atomic
//                       accumulate (split-K, gradient accumulation)
// Operand "modes" only change how the producer addresses global memory:
//   A_KMAJ / B_KMAJ     row-major [rows][K]                      (linear fwd, QK^T)
//   A_MNMAJ / B_MNMAJ   [K][rows]                                (dgrad/wgrad, P.V)
//   A_CONV              NHWC activations, implicit im2col: one 4-D TMA box per
//                       (tap, 64-channel block); padding comes from TMA OOB zero fill,
//                       stride-2 from TMA element strides
//   A_WG_DY / B_WG_X    conv weight gradient: K runs over 64-pixel tiles of dY / shifted X
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <mutex>
#include <string>
#include <cudaTypedefs.h>
#include "common.cuh"
#include "dpipe.h"

namespace dp {

thread_local std::string g_last_error;
void set_error(const std::string& s) { g_last_error = s; }

enum { A_KMAJ = 0, A_MNMAJ = 1, A_CONV = 2, A_WG_DY = 3, A_WG_X = 4 };
enum { B_KMAJ = 0, B_MNMAJ = 1, B_WG_X = 2, B_DGRAD = 3, B_WG_DY = 4 };

struct TcParams {
  int M, N;
  int num_kb;
  int tiles_m, tiles_n, batch1, nbatch, splits, kb_per_split;
  int a_mode, b_mode;
  int P, Q;        // output spatial dims (conv modes)
  int tw, th, tn;  // pixel box (128 pixels for A_CONV, 64 for the wgrad modes)
  int stride, pad_h, pad_w, S, cblk, C;
  int Rf;          // filter height (B_DGRAD flips taps)
  int stream_k;    // 1: contiguous k-iteration ranges per CTA (fp32 atomic outputs)
  int d_tma;       // 1: bf16 output written by TMA tensor stores (tmD)
  int halo;        // 1: 3x3 stride-1 conv with one input strip per filter row (TcCfg HALO)
  int geglu, F;    // GEGLU epilogues: 1 = forward (N = 2F, tile = [a cols | g cols] of one BN/2-wide
                   // output range), 2 = backward through the FF output projection's dgrad (N = F)
  const void* gh;  // geglu 2: the pre-activation h = [a | g], bf16 [M][2F], row stride gh_ld
  int64_t gh_ld;
  float* gn_sums;  // GroupNorm statistics epilogue (GEG == 3): [samples][G][2] {sum, sum of squares}
  int gn_lg, gn_hw, gn_G;  // log2(channels per group), output pixels per sample, groups
  void* D;
  int64_t d_ld, d_bs1, d_bs2;
  int d_f32, out_mode, vec_ok;
  const float* bias;
  const void* R;
  int64_t r_ld, r_bs1, r_bs2;
  float alpha;
};

constexpr int BM = 128;
constexpr int BK = 64;
// warps 0-3: TMA producer, MMA issuer, TMEM allocator, idle; warps 4-11: epilogue (two per TMEM lane
// quadrant), each with two 2 KB bf16 staging buffers for the TMA stores
constexpr int EPI_WARPS = 8;
constexpr int GEMM_THREADS = 32 * (4 + EPI_WARPS);
constexpr int EPI_SMEM = EPI_WARPS * 2 * 32 * 64;
constexpr uint32_t A_STAGE_BYTES = BM * BK * 2;

// HALO (3x3 stride-1 convs whose 128-pixel tiles lie in one image row): a stage holds ONE input
// strip of 130 pixels x 64 channels for a filter row r and the three taps s = 0..2 read it as
// row-shifted views (UMMA descriptor base offset), with the three matching weight blocks: the
// A operand crosses L2 -> SM once per filter row instead of once per tap.
constexpr int HALO_ROWS = BM + 2;
constexpr uint32_t HALO_A_BYTES = HALO_ROWS * BK * 2;   // bytes the halo TMA box delivers
template <int BN, int CG, bool HALO = false>
struct TcCfg {
  static constexpr int BNL = BN / CG;  // B columns staged per CTA (a CTA pair splits N)
  static constexpr uint32_t B_SUB = BNL * BK * 2;
  static constexpr uint32_t B_STAGE_BYTES = (HALO ? 3 : 1) * B_SUB;
  static constexpr uint32_t A_BYTES = HALO ? ((HALO_A_BYTES + 1023) / 1024) * 1024 : A_STAGE_BYTES;
  static constexpr uint32_t A_TX = HALO ? HALO_A_BYTES : A_STAGE_BYTES;
  // as many 64-deep k-stages as fit next to the epilogue staging buffers
  static constexpr int STAGES_FIT = (225 * 1024 - EPI_SMEM) / (A_BYTES + B_STAGE_BYTES);
  static constexpr int STAGES = STAGES_FIT > 8 ? 8 : STAGES_FIT;
  // BN > 256 (320: U-Net 320/640-channel layers): two N = BN/2 MMAs per k-step into adjacent TMEM
  // column ranges, one accumulator buffer (the epilogue is exposed once per long-K tile); each CTA
  // of a pair stages BNL/2 rows of B for each half
  static constexpr int NH = BN > 256 ? 2 : 1;
  static constexpr uint32_t B_HALF = B_SUB / NH;
  static constexpr int NACC = 2 * BN <= 512 ? 2 : 1;
  static constexpr int TMEM_COLS = (NACC * BN <= 128) ? 128 : (NACC * BN <= 256 ? 256 : 512);
  static constexpr size_t SMEM = 1024 + STAGES * (A_BYTES + B_STAGE_BYTES) + EPI_SMEM + 256;
};

DP_DEV void pixel_origin(int pix0, int P, int Q, int& n, int& h, int& w) {
  const int pq = P * Q;
  n = pix0 / pq;
  const int rem = pix0 - n * pq;
  h = rem / Q;
  w = rem - h * Q;
}

template <int BN>
DP_DEV void epilogue_store(const TcParams& p, int row, int n, int z1, int z2, const uint32_t (&v)[32]) {
  float f[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) f[i] = __uint_as_float(v[i]);
  if (p.alpha != 1.f) {
#pragma unroll
    for (int i = 0; i < 32; ++i) f[i] *= p.alpha;
  }
  const int nvalid = min(32, p.N - n);
  if (p.bias) {
    if (nvalid == 32 && (reinterpret_cast<uintptr_t>(p.bias + n) & 15) == 0) {
      // 8 x 16-byte loads (the 32 scalar loads per chunk were warp-uniform but 32 instructions)
#pragma unroll
      for (int i = 0; i < 32; i += 4) {
        const float4 b4 = __ldg(reinterpret_cast<const float4*>(p.bias + n + i));
        f[i] += b4.x;
        f[i + 1] += b4.y;
        f[i + 2] += b4.z;
        f[i + 3] += b4.w;
      }
    } else if (nvalid == 32) {
#pragma unroll
      for (int i = 0; i < 32; ++i) f[i] += __ldg(p.bias + n + i);
    } else {
#pragma unroll
      for (int i = 0; i < 32; ++i)
        if (i < nvalid) f[i] += __ldg(p.bias + n + i);
    }
  }
  if (p.R) {
    const int64_t roff = z1 * p.r_bs1 + z2 * p.r_bs2 + (int64_t)row * p.r_ld + n;
    if (p.d_f32) {
      const float* r = reinterpret_cast<const float*>(p.R) + roff;
#pragma unroll
      for (int i = 0; i < 32; ++i)
        if (i < nvalid) f[i] += r[i];
    } else {
      const __nv_bfloat16* r = reinterpret_cast<const __nv_bfloat16*>(p.R) + roff;
      if (nvalid == 32 && p.vec_ok) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          uint4 u = *reinterpret_cast<const uint4*>(r + q * 8);
          const __nv_bfloat16* b = reinterpret_cast<const __nv_bfloat16*>(&u);
#pragma unroll
          for (int i = 0; i < 8; ++i) f[q * 8 + i] += __bfloat162float(b[i]);
        }
      } else {
  #pragma unroll
      for (int i = 0; i < 32; ++i)
        if (i < nvalid) f[i] += __bfloat162float(r[i]);
      }
    }
  }
  const int64_t doff = z1 * p.d_bs1 + z2 * p.d_bs2 + (int64_t)row * p.d_ld + n;
  if (p.d_f32) {
    float* d = reinterpret_cast<float*>(p.D) + doff;
    if (p.out_mode == DP_OUT_ATOMIC_ADD) {
      if (nvalid == 32 && p.vec_ok) {
#pragma unroll
        for (int q = 0; q < 8; ++q)
          atomicAdd(reinterpret_cast<float4*>(d + 4 * q),
                    make_float4(f[4 * q], f[4 * q + 1], f[4 * q + 2], f[4 * q + 3]));
      } else {
#pragma unroll
        for (int i = 0; i < 32; ++i)
          if (i < nvalid) atomicAdd(d + i, f[i]);
      }
    } else {
      if (nvalid == 32 && p.vec_ok) {
#pragma unroll
        for (int q = 0; q < 8; ++q)
          *reinterpret_cast<float4*>(d + 4 * q) =
              make_float4(f[4 * q], f[4 * q + 1], f[4 * q + 2], f[4 * q + 3]);
      } else {
#pragma unroll
        for (int i = 0; i < 32; ++i)
          if (i < nvalid) d[i] = f[i];
      }
    }
  } else {
    __nv_bfloat16* d = reinterpret_cast<__nv_bfloat16*>(p.D) + doff;
    if (nvalid == 32 && p.vec_ok) {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        uint4 u;
        u.x = pack_bf16x2(f[q * 8 + 0], f[q * 8 + 1]);
        u.y = pack_bf16x2(f[q * 8 + 2], f[q * 8 + 3]);
        u.z = pack_bf16x2(f[q * 8 + 4], f[q * 8 + 5]);
        u.w = pack_bf16x2(f[q * 8 + 6], f[q * 8 + 7]);
        *reinterpret_cast<uint4*>(d + q * 8) = u;
      }
    } else {
#pragma unroll
      for (int i = 0; i < 32; ++i)
        if (i < nvalid) d[i] = __float2bfloat16_rn(f[i]);
    }
  }
}

// ---------------------------------------------------------------- work decomposition
// Shared by the producer, MMA and epilogue roles (each walks the same sequence).
//  * tiled mode: items = tiles x splits, CTA b takes items b, b+G, ...; tiles are rastered
//    in bands of GM m-tiles (n fastest inside a band) so the CTAs of one wave share A
//    tiles and a band's B tiles stay L2 resident.
//  * stream-K mode (fp32 atomic outputs only): the tiles x num_kb k-iterations are cut
//    into gridDim.x equal contiguous ranges; a range may cover parts of several tiles and
//    each part is reduced with fp32 atomics (perfect wave balance for skinny wgrads).
struct Work {
  int m_blk, n_blk, z1, z2, kb0, kb1;
};
constexpr int GM = 8;

DP_DEV void tile_coords(const TcParams& p, int t, Work& w) {
  const int per_batch = p.tiles_m * p.tiles_n;
  const int z = t / per_batch;
  t -= z * per_batch;
  const int band_items = GM * p.tiles_n;
  const int band = t / band_items;
  const int within = t - band * band_items;
  const int gm = min(GM, p.tiles_m - band * GM);
  w.m_blk = band * GM + within % gm;
  w.n_blk = within / gm;
  w.z1 = z % p.batch1;
  w.z2 = z / p.batch1;
}

struct WorkIter {
  int cursor, end, unit, units;
  DP_DEV void init(const TcParams& p, int cg) {
    unit = blockIdx.x / cg;   // one work unit per CTA pair (cg = 2) or per CTA
    units = gridDim.x / cg;
    if (p.stream_k) {
      const long long tot = (long long)p.tiles_m * p.tiles_n * p.nbatch * p.num_kb;
      cursor = static_cast<int>(tot * unit / units);
      end = static_cast<int>(tot * (unit + 1) / units);
    } else {
      cursor = unit;
      end = p.tiles_m * p.tiles_n * p.nbatch * p.splits;
    }
  }
  DP_DEV bool next(const TcParams& p, Work& w) {
    if (cursor >= end) return false;
    if (p.stream_k) {
      const int t = cursor / p.num_kb;
      w.kb0 = cursor - t * p.num_kb;
      w.kb1 = min(p.num_kb, w.kb0 + (end - cursor));
      tile_coords(p, t, w);
      cursor += w.kb1 - w.kb0;
    } else {
      const int tiles = p.tiles_m * p.tiles_n * p.nbatch;
      const int split = cursor / tiles;
      tile_coords(p, cursor - split * tiles, w);
      w.kb0 = split * p.kb_per_split;
      w.kb1 = min(p.num_kb, w.kb0 + p.kb_per_split);
      cursor += units;
    }
    return true;
  }
};

// Epilogue of one 32x32 chunk through shared memory and a TMA tensor store (bf16 outputs):
// lane = row; the 64-byte row is written in the SWIZZLE_64B layout the D map expects
// (16-byte chunk index XOR ((row >> 1) & 3)), which also spreads the 32 lanes over all banks.
DP_DEV void stage_row_bf16(uint8_t* buf, int lane, const float (&f)[32]) {
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    uint4 u;
    u.x = pack_bf16x2(f[q * 8 + 0], f[q * 8 + 1]);
    u.y = pack_bf16x2(f[q * 8 + 2], f[q * 8 + 3]);
    u.z = pack_bf16x2(f[q * 8 + 4], f[q * 8 + 5]);
    u.w = pack_bf16x2(f[q * 8 + 6], f[q * 8 + 7]);
    const int qs = q ^ ((lane >> 1) & 3);
    // st.shared (not a generic store): the staging buffer is known to be shared memory
    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(smem_u32(buf + lane * 64 + qs * 16)),
                 "r"(u.x), "r"(u.y), "r"(u.z), "r"(u.w)
                 : "memory");
  }
}

// GroupNorm statistics of one 32 x 32 output chunk (GEG == 3 conv launches): the bf16-rounded values (what
// the consumer reads) summed per group of 2^lg consecutive channels inside each lane's row by a fixed
// tree, reduced over the warp's 32 rows (one sample: P*Q % 32 == 0), one atomic pair per group and chunk.
// The GroupNorm that follows then reads x once (dp_group_norm_fwd_sums) instead of twice.
DP_DEV void gn_stats_chunk(const TcParams& p, const float (&f)[32], int row, int row0, int n, int lane) {
  if (row0 >= p.M) return;  // warp-uniform
  const bool live = row < p.M;
  float s1[16], q1[16];
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    const float a = live ? __bfloat162float(__float2bfloat16_rn(f[2 * j])) : 0.f;
    const float b = live ? __bfloat162float(__float2bfloat16_rn(f[2 * j + 1])) : 0.f;
    s1[j] = a + b;
    q1[j] = fmaf(a, a, b * b);
  }
  // pairwise tree up to 2^lg channels per group: s1 holds groups of 2, then 4, 8, 16, 32
#pragma unroll
  for (int lvl = 1; lvl < 5; ++lvl) {
    if (lvl >= p.gn_lg) break;  // uniform
#pragma unroll
    for (int j = 0; j < (16 >> lvl); ++j) {
      s1[j] = s1[2 * j] + s1[2 * j + 1];
      q1[j] = q1[2 * j] + q1[2 * j + 1];
    }
  }
  const int m = 32 >> p.gn_lg;  // groups in this chunk
  const int sample = row0 / p.gn_hw;
  // DP_GN_SLOTS copies of the table (CTA b adds into copy b % slots): thousands of tiles add into the
  // same few (sample, group) entries, and same-address reductions serialise in L2
  const int slot = blockIdx.x % DP_GN_SLOTS;
  float* out = p.gn_sums + (((int64_t)slot * (p.M / p.gn_hw) + sample) * p.gn_G + (n >> p.gn_lg)) * 2;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    if (j >= m) break;
    float a = s1[j], b = q1[j];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      a += __shfl_xor_sync(0xffffffffu, a, o);
      b += __shfl_xor_sync(0xffffffffu, b, o);
    }
    if (lane == 0) atomicAdd(reinterpret_cast<float2*>(out + 2 * j), make_float2(a, b));
  }
}

// fp32 half chunk (16 columns, 64-byte row) in the SWIZZLE_64B layout of the 16 x 32 reduce box
DP_DEV void stage_row_f32(uint8_t* buf, int lane, const float (&f)[32], int hh) {
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int qs = q ^ ((lane >> 1) & 3);
    asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(smem_u32(buf + lane * 64 + qs * 16)),
                 "f"(f[hh * 16 + q * 4 + 0]), "f"(f[hh * 16 + q * 4 + 1]), "f"(f[hh * 16 + q * 4 + 2]),
                 "f"(f[hh * 16 + q * 4 + 3])
                 : "memory");
  }
}

template <int BN>
DP_DEV void epilogue_math(const TcParams& p, int row, int n, int z1, int z2, const uint32_t (&v)[32],
                          float (&f)[32], const uint4 (&rpre)[4], bool use_pre) {
#pragma unroll
  for (int i = 0; i < 32; ++i) f[i] = __uint_as_float(v[i]);
  if (p.alpha != 1.f) {
#pragma unroll
    for (int i = 0; i < 32; ++i) f[i] *= p.alpha;
  }
  const int nvalid = min(32, p.N - n);
  if (p.bias) {
    if (nvalid == 32 && (reinterpret_cast<uintptr_t>(p.bias + n) & 15) == 0) {
      // 8 x 16-byte loads (the 32 scalar loads per chunk were warp-uniform but 32 instructions)
#pragma unroll
      for (int i = 0; i < 32; i += 4) {
        const float4 b4 = __ldg(reinterpret_cast<const float4*>(p.bias + n + i));
        f[i] += b4.x;
        f[i + 1] += b4.y;
        f[i + 2] += b4.z;
        f[i + 3] += b4.w;
      }
    } else if (nvalid == 32) {
#pragma unroll
      for (int i = 0; i < 32; ++i) f[i] += __ldg(p.bias + n + i);
    } else {
#pragma unroll
      for (int i = 0; i < 32; ++i)
        if (i < nvalid) f[i] += __ldg(p.bias + n + i);
    }
  }
  if (use_pre) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const __nv_bfloat16* b = reinterpret_cast<const __nv_bfloat16*>(&rpre[q]);
#pragma unroll
      for (int i = 0; i < 8; ++i) f[q * 8 + i] += __bfloat162float(b[i]);
    }
  } else if (p.R && row < p.M) {
    const int64_t roff = z1 * p.r_bs1 + z2 * p.r_bs2 + (int64_t)row * p.r_ld + n;
    const __nv_bfloat16* r = reinterpret_cast<const __nv_bfloat16*>(p.R) + roff;
    if (nvalid == 32 && p.vec_ok) {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        uint4 u = *reinterpret_cast<const uint4*>(r + q * 8);
        const __nv_bfloat16* b = reinterpret_cast<const __nv_bfloat16*>(&u);
#pragma unroll
        for (int i = 0; i < 8; ++i) f[q * 8 + i] += __bfloat162float(b[i]);
      }
    } else {
#pragma unroll
      for (int i = 0; i < 32; ++i)
        if (i < nvalid) f[i] += __bfloat162float(r[i]);
    }
  }
}

constexpr int EPI_STAGE_BYTES = 32 * 64;  // one 32 x 32 bf16 chunk

// GEG: GEGLU epilogue instantiations (0 = none, 1 = FF input projection forward, 2 = FF output projection
// input gradient); kept out of the other instantiations so their epilogue registers stay as they were
template <int BN, int CG, bool HALO, bool RES, int GEG = 0>
__global__ void __launch_bounds__(GEMM_THREADS, 1)
    tc_gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   const __grid_constant__ CUtensorMap tmD, const __grid_constant__ CUtensorMap tmD2,
                   const TcParams p) {
  using Cfg = TcCfg<BN, CG, HALO>;
  constexpr int STAGES = Cfg::STAGES;
  constexpr int BNL = Cfg::BNL;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * Cfg::A_BYTES;
  uint8_t* sE = sB + STAGES * Cfg::B_STAGE_BYTES;            // 4 warps x 2 x 2 KB, 1 KB aligned
  uint64_t* full = reinterpret_cast<uint64_t*>(sE + 2 * EPI_WARPS * EPI_STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  // warp index through a shuffle from lane 0: the compiler then knows it is warp-uniform, so the role
  // branches below are uniform and the producer / MMA bookkeeping lives in uniform registers (no
  // per-instruction uniformity waterfall around every UTMALDG / UTCHMMA)
  const int warp = __shfl_sync(0xffffffffu, static_cast<int>(threadIdx.x >> 5), 0);
  const int lane = threadIdx.x & 31;
  // CTA pair (cta_group::2): rank 0 (leader) issues the M=256 MMAs; each CTA stages its own
  // 128 rows of A and half of B's N columns, and owns its 128 rows of the accumulator.
  const int crank = CG == 2 ? static_cast<int>(cluster_ctarank()) : 0;
  const bool leader = crank == 0;
  if (threadIdx.x == 0) {
    tma_prefetch(&tmA);
    tma_prefetch(&tmB);
    if (p.d_tma) tma_prefetch(&tmD);
    if constexpr (GEG == 1) tma_prefetch(&tmD2);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], EPI_WARPS * CG);  // one arrival per epilogue warp of each CTA
    }
    fence_barrier_init();
  }
  if (warp == 2) {
    if constexpr (CG == 2)
      tmem_alloc_2sm<Cfg::TMEM_COLS>(tmem_slot);
    else
      tmem_alloc<Cfg::TMEM_COLS>(tmem_slot);
  }
  tc_fence_before();
  if constexpr (CG == 2)
    cluster_sync();
  else
    __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  // Programmatic dependent launch: everything above (barrier init, TMEM allocation, descriptor
  // prefetch) overlaps the tail of the previous kernel in the stream; no global memory is read
  // or written before the previous grid has completed and flushed.
  DP_PDL_ENTRY();

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer (every CTA)
    // The whole warp walks the work list (lane 0 issues). Per-tile invariants (weight-gradient
    // channel / tap of every 64-column box) are computed once per tile and the per-k-block
    // coordinates (conv tap + channel block, pixel tile) advance incrementally: the divisions the
    // producer used to do per k-block (~330 instructions) had made it, not the tensor core, the
    // bound of the conv wgrad mainloop.
    const bool issuer = lane == 0;
    int stage = 0;
    uint32_t phase = 0;
    WorkIter it;
    it.init(p, CG);
    Work wk;
    const bool wg = p.a_mode == A_WG_DY || p.a_mode == A_WG_X;
    while (it.next(p, wk)) {
      const int z1 = wk.z1, z2 = wk.z2;
      const int m0 = wk.m_blk * (BM * CG) + crank * BM;
      const int n0 = wk.n_blk * BN + crank * BNL;
      int cn = 0, ch = 0, cw = 0;
      if (p.a_mode == A_CONV) {
        pixel_origin(m0, p.P, p.Q, cn, ch, cw);
        ch = ch * p.stride - p.pad_h;
        cw = cw * p.stride - p.pad_w;
      }
      // weight-gradient window boxes: (channel, filter row, filter column) of each 64-wide box of the
      // x operand (B for B_WG_X: columns n0 + 64 j; A for A_WG_X: rows m0 + 64 j)
      constexpr int NXB = (BNL / 64) > 2 ? (BNL / 64) : 2;
      int xci[NXB], xrr[NXB], xss[NXB];
      if (p.b_mode == B_WG_X || p.a_mode == A_WG_X) {
        const int base = p.a_mode == A_WG_X ? m0 : n0;
#pragma unroll
        for (int j = 0; j < NXB; ++j) {
          const int nn = base + 64 * j;
          const int tap = nn / p.C;
          xci[j] = nn - tap * p.C;
          xrr[j] = tap / p.S;
          xss[j] = tap - xrr[j] * p.S;
        }
      }
      // k-block counters: (filter row, filter column, channel block) for the conv modes, pixel tile
      // origin for the weight-gradient modes
      int kr = 0, ks = 0, kc = 0, pn = 0, ph = 0, pw = 0;
      if (p.a_mode == A_CONV) {
        const int per_r = HALO ? p.cblk : p.S * p.cblk;
        kr = wk.kb0 / per_r;
        const int rem = wk.kb0 - kr * per_r;
        ks = HALO ? 0 : rem / p.cblk;
        kc = rem - ks * p.cblk;
      } else if (wg) {
        pixel_origin(wk.kb0 * BK, p.P, p.Q, pn, ph, pw);
      }
      for (int kb = wk.kb0; kb < wk.kb1; ++kb) {
        mbar_wait(&empty[stage], phase ^ 1);
        if (leader && issuer) mbar_expect_tx(&full[stage], CG * (Cfg::A_TX + Cfg::B_STAGE_BYTES));
        uint8_t* a_dst = sA + stage * Cfg::A_BYTES;
        uint8_t* b_dst = sB + stage * Cfg::B_STAGE_BYTES;
        uint64_t* fb = &full[stage];
        auto load = [&](const CUtensorMap* m, void* dst, int c0, int c1, int c2, int c3) {
          if (!issuer) return;
          if constexpr (CG == 2)
            tma_load_4d_2sm(m, fb, dst, c0, c1, c2, c3);
          else
            tma_load_4d(m, fb, dst, c0, c1, c2, c3);
        };
        if constexpr (HALO) {
          // kb = (filter row r, 64-channel block): one 130-pixel strip, three tap weight blocks
          load(&tmA, a_dst, kc * BK, cw, ch + kr, cn);
#pragma unroll
          for (int ss = 0; ss < 3; ++ss)
            load(&tmB, b_dst + ss * Cfg::B_SUB, ((kr * 3 + ss) * p.cblk + kc) * BK, n0, z1, z2);
        } else {
          switch (p.a_mode) {
            case A_KMAJ:
              load(&tmA, a_dst, kb * BK, m0, z1, z2);
              break;
            case A_MNMAJ:
              load(&tmA, a_dst, m0, kb * BK, z1, z2);
              load(&tmA, a_dst + 8192, m0 + 64, kb * BK, z1, z2);
              break;
            case A_CONV:
              load(&tmA, a_dst, kc * BK, cw + ks, ch + kr, cn);
              break;
            case A_WG_X: {  // rows = (tap, channel): shifted input windows, MN-major
              const int hin = ph * p.stride - p.pad_h, win = pw * p.stride - p.pad_w;
#pragma unroll
              for (int j = 0; j < 2; ++j) load(&tmA, a_dst + j * 8192, xci[j], win + xss[j], hin + xrr[j], pn);
              break;
            }
            default:  // A_WG_DY
              load(&tmA, a_dst, m0, pw, ph, pn);
              load(&tmA, a_dst + 8192, m0 + 64, pw, ph, pn);
              break;
          }
          switch (p.b_mode) {
            case B_KMAJ:
              if constexpr (GEG == 1) {
                // [a rows | g rows] of output range n_blk*BN/2: a pair's CTAs hold one half each,
                // a single CTA stacks both (two BN/2-row boxes)
                const int na = wk.n_blk * (BN / 2);
                if constexpr (CG == 2) {
                  load(&tmB, b_dst, kb * BK, crank ? p.F + na : na, z1, z2);
                } else {
                  load(&tmB, b_dst, kb * BK, na, z1, z2);
                  load(&tmB, b_dst + (BN / 2) * BK * 2, kb * BK, p.F + na, z1, z2);
                }
              } else if constexpr (Cfg::NH == 2) {
                const int nt = wk.n_blk * BN + crank * (BNL / 2);
                load(&tmB, b_dst, kb * BK, nt, z1, z2);
                load(&tmB, b_dst + Cfg::B_HALF, kb * BK, nt + BN / 2, z1, z2);
              } else {
                load(&tmB, b_dst, kb * BK, n0, z1, z2);
              }
              break;
            case B_MNMAJ:
#pragma unroll
              for (int j = 0; j < BNL / 64; ++j) load(&tmB, b_dst + j * 8192, n0 + 64 * j, kb * BK, z1, z2);
              break;
            case B_DGRAD:
              // B(n = input channel c, k = (tap, filter kk)) = w[kk][R-1-r][S-1-s][c]: the conv
              // weights [K][R][S][C] read tap-flipped in place (no transposed copy)
#pragma unroll
              for (int j = 0; j < BNL / 64; ++j)
                load(&tmB, b_dst + j * 8192, n0 + 64 * j, p.S - 1 - ks, p.Rf - 1 - kr, kc * BK);
              break;
            case B_WG_DY:  // dy [pixels][K] MN-major (swapped weight gradient)
#pragma unroll
              for (int j = 0; j < BNL / 64; ++j) load(&tmB, b_dst + j * 8192, n0 + 64 * j, pw, ph, pn);
              break;
            default: {  // B_WG_X
              const int hin = ph * p.stride - p.pad_h, win = pw * p.stride - p.pad_w;
#pragma unroll
              for (int j = 0; j < BNL / 64; ++j) load(&tmB, b_dst + j * 8192, xci[j], win + xss[j], hin + xrr[j], pn);
              break;
            }
          }
        }
        __syncwarp();
        if (p.a_mode == A_CONV) {
          if (++kc == p.cblk) {
            kc = 0;
            if (HALO || ++ks == p.S) {
              ks = 0;
              ++kr;
            }
          }
        } else if (wg) {
          pw += p.tw;
          if (pw >= p.Q) {
            pw = 0;
            ph += p.th;
            if (ph >= p.P) {
              ph = 0;
              pn += p.tn;
            }
          }
        }
        if (++stage == STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else if (warp == 1 && leader) {
    // ------------------------------------------------------------ MMA issuer (leader CTA)
    // warp-wide bookkeeping (uniform registers), lane 0 issues the MMAs and commits
    const int a_mn = (p.a_mode == A_MNMAJ || p.a_mode == A_WG_DY || p.a_mode == A_WG_X) ? 1 : 0;
    const int b_mn = (p.b_mode != B_KMAJ) ? 1 : 0;
    const uint32_t idesc = idesc_bf16_f32(BM * CG, BN / Cfg::NH, a_mn, b_mn);
    const bool issuer = lane == 0;
    int stage = 0;
    uint32_t phase = 0;
    int acc = 0;
    uint32_t acc_phase = 0;
    WorkIter it;
    it.init(p, CG);
    Work wk;
    while (it.next(p, wk)) {
      mbar_wait(&tempty[acc], acc_phase ^ 1);
      tc_fence_after();
      const uint32_t d_tmem = tmem_base + acc * BN;
      for (int kb = wk.kb0; kb < wk.kb1; ++kb) {
        mbar_wait(&full[stage], phase);
        tc_fence_after();
        const uint32_t a_addr = smem_u32(sA + stage * Cfg::A_BYTES);
        const uint32_t b_addr = smem_u32(sB + stage * Cfg::B_STAGE_BYTES);
        if constexpr (HALO) {
#pragma unroll
          for (int ss = 0; ss < 3; ++ss)
#pragma unroll
            for (int j = 0; j < BK / 16; ++j) {
              // tap ss = the strip shifted by ss pixel rows (128 B): start address mid swizzle atom
              const uint64_t adesc = smem_desc_sw128(a_addr + ss * 128 + j * 32, 16, 1024);  // no base offset: the
              // SWIZZLE_128B phase follows the absolute smem address (TMA wrote the strip the same
              // way), so a row-shifted start is consistent as is (tests/test_gemm_gpu.py::halo)
              const uint64_t bdesc = smem_desc_sw128(b_addr + ss * Cfg::B_SUB + j * 32, 16, 1024);
              const uint32_t accum = (kb > wk.kb0 || ss > 0 || j > 0) ? 1u : 0u;
              if (!issuer) {
              } else if constexpr (CG == 2)
                tc_mma_bf16_2sm(d_tmem, adesc, bdesc, idesc, accum);
              else
                tc_mma_bf16(d_tmem, adesc, bdesc, idesc, accum);
            }
        } else if constexpr (Cfg::NH == 2) {
#pragma unroll
          for (int j = 0; j < BK / 16; ++j)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const uint64_t adesc = smem_desc_sw128(a_addr + j * 32, 16, 1024);
              const uint64_t bdesc = smem_desc_sw128(b_addr + h * Cfg::B_HALF + j * 32, 16, 1024);
              const uint32_t accum = (kb > wk.kb0 || j > 0) ? 1u : 0u;
              if (!issuer) {
              } else if constexpr (CG == 2)
                tc_mma_bf16_2sm(d_tmem + h * (BN / 2), adesc, bdesc, idesc, accum);
              else
                tc_mma_bf16(d_tmem + h * (BN / 2), adesc, bdesc, idesc, accum);
            }
        } else
#pragma unroll
        for (int j = 0; j < BK / 16; ++j) {
          const uint64_t adesc = a_mn ? smem_desc_sw128(a_addr + j * 2048, 8192, 1024)
                                      : smem_desc_sw128(a_addr + j * 32, 16, 1024);
          const uint64_t bdesc = b_mn ? smem_desc_sw128(b_addr + j * 2048, 8192, 1024)
                                      : smem_desc_sw128(b_addr + j * 32, 16, 1024);
          const uint32_t accum = (kb > wk.kb0 || j > 0) ? 1u : 0u;
          if (!issuer) {
          } else if constexpr (CG == 2)
            tc_mma_bf16_2sm(d_tmem, adesc, bdesc, idesc, accum);
          else
            tc_mma_bf16(d_tmem, adesc, bdesc, idesc, accum);
        }
        if (!issuer) {
        } else if constexpr (CG == 2)
          tc_commit_2sm_mc(&empty[stage]);
        else
          tc_commit(&empty[stage]);
        __syncwarp();
        if (++stage == STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
      if (!issuer) {
      } else if constexpr (CG == 2)
        tc_commit_2sm_mc(&tfull[acc]);
      else
        tc_commit(&tfull[acc]);
      __syncwarp();
      if (++acc == Cfg::NACC) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
  } else if (warp >= 4) {
    // ------------------------------------------------------------ epilogue (every CTA)
    const int wq = warp & 3;            // TMEM lane quadrant (rows wq*32 .. +32 of the tile)
    const int half = (warp - 4) >> 2;   // chunk parity this warp stores
    int acc = 0;
    uint32_t acc_phase = 0;
    uint8_t* ebuf = sE + (warp - 4) * 2 * EPI_STAGE_BYTES;
    int chunk_seq = 0;
    const uint32_t tempty_leader0 = CG == 2 ? mapa_shared(smem_u32(&tempty[0]), 0) : 0;
    WorkIter it;
    it.init(p, CG);
    Work wk;
    // bf16 residual (TMA-store path): each lane's 64-byte row segments are fetched two chunks
    // ahead, the first two before the accumulator is ready, so their DRAM latency overlaps the
    // MMAs and the previous chunks instead of stalling every chunk
    const bool rpre_on = RES && p.R != nullptr && p.vec_ok && !p.d_f32 && p.d_tma;
    auto rload = [&](const Work& w, int row, int c, uint4 (&dst)[4]) {
      const int n = w.n_blk * BN + c * 32;
      if (rpre_on && row < p.M && c < BN / 32 && n + 32 <= p.N) {
        const __nv_bfloat16* rb = reinterpret_cast<const __nv_bfloat16*>(p.R) + w.z1 * p.r_bs1 +
                                  w.z2 * p.r_bs2 + (int64_t)row * p.r_ld + n;
#pragma unroll
        for (int q = 0; q < 4; ++q) dst[q] = *reinterpret_cast<const uint4*>(rb + q * 8);
      }
    };
    while (it.next(p, wk)) {
      const int row0 = wk.m_blk * (BM * CG) + crank * BM + wq * 32;
      const int row = row0 + lane;
      uint4 r1[4], r2[4];
      if constexpr (RES) {
        rload(wk, row, half, r1);
        rload(wk, row, half + 2, r2);
      }
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      // two warps per TMEM lane quadrant split the accumulator's 32-column chunks (even / odd):
      // the epilogue (TMEM load, bias / residual, bf16 staging, TMA store per chunk) is latency
      // bound per warp and had bounded short-K GEMMs with one warp per quadrant
      const int nch = GEG == 1 ? 0 : min(BN / 32, (p.N - wk.n_blk * BN + 31) / 32);  // warp-uniform
      const uint32_t tbase = tmem_base + (static_cast<uint32_t>(wq * 32) << 16) + acc * BN;
      if constexpr (GEG == 1) {
        // chunk pair (a cols c, g cols c + BN/64): bias, bf16 rounding (the stored pre-activation, which
        // the backward reads), y = a * gelu_erf(g) from the rounded values, three TMA stores
#pragma unroll 1
        for (int c = half; c < BN / 64; c += 2) {
          const int na = wk.n_blk * (BN / 2) + c * 32;
          uint32_t va[32], vg[32];
          tmem_ld_32x32(tbase + c * 32, va);
          tmem_ld_32x32(tbase + BN / 2 + c * 32, vg);
          tmem_ld_wait_dep(va);
          tmem_ld_wait_dep(vg);
          // a and g rows: bias, bf16 rounding, staged and stored (the stored pre-activation is what the
          // backward reads); y is then computed from the staged bf16 rows (same inputs as the unfused
          // geglu kernel) and stored once the first staging buffer has been read by its TMA store
          auto stage_pre = [&](const uint32_t (&v)[32], const float* bias, int col) -> uint8_t* {
            uint8_t* buf = ebuf + (chunk_seq & 1) * EPI_STAGE_BYTES;
            if (chunk_seq >= 2) {
              if (lane == 0) bulk_wait_read<1>();
              __syncwarp();
            }
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const float4 b0 = __ldg(reinterpret_cast<const float4*>(bias + q * 8));
              const float4 b1 = __ldg(reinterpret_cast<const float4*>(bias + q * 8 + 4));
              uint4 u;
              u.x = pack_bf16x2(__uint_as_float(v[q * 8 + 0]) + b0.x, __uint_as_float(v[q * 8 + 1]) + b0.y);
              u.y = pack_bf16x2(__uint_as_float(v[q * 8 + 2]) + b0.z, __uint_as_float(v[q * 8 + 3]) + b0.w);
              u.z = pack_bf16x2(__uint_as_float(v[q * 8 + 4]) + b1.x, __uint_as_float(v[q * 8 + 5]) + b1.y);
              u.w = pack_bf16x2(__uint_as_float(v[q * 8 + 6]) + b1.z, __uint_as_float(v[q * 8 + 7]) + b1.w);
              const int qs = q ^ ((lane >> 1) & 3);
              asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(smem_u32(buf + lane * 64 + qs * 16)),
                           "r"(u.x), "r"(u.y), "r"(u.z), "r"(u.w)
                           : "memory");
            }
            fence_async_shared();
            __syncwarp();
            if (lane == 0 && row0 < p.M) {
              tma_store_4d(&tmD, buf, col, row0, 0, 0);
              bulk_commit();
            }
            ++chunk_seq;
            return buf;
          };
          const uint8_t* ba = stage_pre(va, p.bias + na, na);
          const uint8_t* bg = stage_pre(vg, p.bias + p.F + na, p.F + na);
          uint32_t yp[16];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int qs = q ^ ((lane >> 1) & 3);
            uint4 ua, ug;
            asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                         : "=r"(ua.x), "=r"(ua.y), "=r"(ua.z), "=r"(ua.w)
                         : "r"(smem_u32(ba + lane * 64 + qs * 16)));
            asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                         : "=r"(ug.x), "=r"(ug.y), "=r"(ug.z), "=r"(ug.w)
                         : "r"(smem_u32(bg + lane * 64 + qs * 16)));
            const uint32_t* pa = &ua.x;
            const uint32_t* pg = &ug.x;
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const float2 fa = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(pa + i));
              const float2 fg = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(pg + i));
              yp[q * 4 + i] = pack_bf16x2(fa.x * (0.5f * fg.x * (1.f + erff(fg.x * 0.70710678118654752f))),
                                          fa.y * (0.5f * fg.y * (1.f + erff(fg.y * 0.70710678118654752f))));
            }
          }
          {
            uint8_t* buf = ebuf + (chunk_seq & 1) * EPI_STAGE_BYTES;  // = the a buffer: wait for its store
            if (lane == 0) bulk_wait_read<1>();
            __syncwarp();
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const int qs = q ^ ((lane >> 1) & 3);
              asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(smem_u32(buf + lane * 64 + qs * 16)),
                           "r"(yp[q * 4]), "r"(yp[q * 4 + 1]), "r"(yp[q * 4 + 2]), "r"(yp[q * 4 + 3])
                           : "memory");
            }
            fence_async_shared();
            __syncwarp();
            if (lane == 0 && row0 < p.M) {
              tma_store_4d(&tmD2, buf, na, row0, 0, 0);
              bulk_commit();
            }
            ++chunk_seq;
          }
        }
      }
#pragma unroll 1
      for (int c = half; c < nch; c += 2) {
        const int n = wk.n_blk * BN + c * 32;
        uint32_t v[32];
        tmem_ld_32x32(tbase + c * 32, v);
        uint4 rc[4];
        if constexpr (RES) {
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            rc[q] = r1[q];
            r1[q] = r2[q];
          }
          rload(wk, row, c + 4, r2);
        }
        // GEGLU backward: this chunk's a / g rows of h are loaded while the TMEM load is in flight
        uint4 ua[4], ug[4];
        if constexpr (GEG == 2) {
          const __nv_bfloat16* hr = reinterpret_cast<const __nv_bfloat16*>(p.gh) + (int64_t)row * p.gh_ld + n;
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            ua[q] = row < p.M ? *reinterpret_cast<const uint4*>(hr + q * 8) : make_uint4(0, 0, 0, 0);
            ug[q] = row < p.M ? *reinterpret_cast<const uint4*>(hr + p.F + q * 8) : make_uint4(0, 0, 0, 0);
          }
        }
        tmem_ld_wait_dep(v);
        const bool use_pre = rpre_on && row < p.M && n + 32 <= p.N;
        if constexpr (GEG == 2) {
          // dy (rounded to bf16, as the unfused dgrad stores it) -> da = dy * gelu(g), dg = dy * a * gelu'(g)
          // from h's a / g rows of this chunk; two TMA stores into dh = [da | dg]
          float da[32], dg[32];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const __nv_bfloat16* pa = reinterpret_cast<const __nv_bfloat16*>(&ua[q]);
            const __nv_bfloat16* pg = reinterpret_cast<const __nv_bfloat16*>(&ug[q]);
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              const float d = __bfloat162float(__float2bfloat16_rn(__uint_as_float(v[q * 8 + i])));
              const float a = __bfloat162float(pa[i]), g = __bfloat162float(pg[i]);
              const float cdf = 0.5f * (1.f + erff(g * 0.70710678118654752f));
              const float pdf = 0.39894228040143268f * __expf(-0.5f * g * g);
              da[q * 8 + i] = d * (g * cdf);
              dg[q * 8 + i] = d * a * (cdf + g * pdf);
            }
          }
          auto put = [&](const float (&f)[32], int col) {
            uint8_t* buf = ebuf + (chunk_seq & 1) * EPI_STAGE_BYTES;
            if (chunk_seq >= 2) {
              if (lane == 0) bulk_wait_read<1>();
              __syncwarp();
            }
            stage_row_bf16(buf, lane, f);
            fence_async_shared();
            __syncwarp();
            if (lane == 0 && row0 < p.M) {
              tma_store_4d(&tmD, buf, col, row0, 0, 0);
              bulk_commit();
            }
            ++chunk_seq;
          };
          put(da, n);
          put(dg, p.F + n);
        } else if (p.d_tma == 3) {
          // transposed fp32 reduce (swapped weight gradient: D rows are the contiguous dimension of the
          // output): stage [16 columns][32 rows] with lane = row, one TMA reduce-add per 16 columns
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {
            uint8_t* buf = ebuf + (chunk_seq & 1) * EPI_STAGE_BYTES;
            if (chunk_seq >= 2) {
              if (lane == 0) bulk_wait_read<1>();
              __syncwarp();
            }
#pragma unroll
            for (int i = 0; i < 16; ++i)
              asm volatile("st.shared.f32 [%0], %1;" ::"r"(smem_u32(buf + i * 128 + lane * 4)),
                           "f"(__uint_as_float(v[hh * 16 + i]) * p.alpha)
                           : "memory");
            fence_async_shared();
            __syncwarp();
            if (lane == 0 && row0 < p.M) {
              tma_reduce_add_4d(&tmD, buf, row0, n + 16 * hh, wk.z1, wk.z2);
              bulk_commit();
            }
            ++chunk_seq;
          }
        } else if (p.d_tma == 2) {
          float f[32];
#pragma unroll
          for (int i = 0; i < 32; ++i) f[i] = __uint_as_float(v[i]) * p.alpha;
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {
            uint8_t* buf = ebuf + (chunk_seq & 1) * EPI_STAGE_BYTES;
            if (chunk_seq >= 2) {
              if (lane == 0) bulk_wait_read<1>();
              __syncwarp();
            }
            stage_row_f32(buf, lane, f, hh);
            fence_async_shared();
            __syncwarp();
            if (lane == 0 && row0 < p.M) {
              tma_reduce_add_4d(&tmD, buf, n + 16 * hh, row0, wk.z1, wk.z2);
              bulk_commit();
            }
            ++chunk_seq;
          }
        } else if (p.d_tma) {
          float f[32];
          epilogue_math<BN>(p, row, n, wk.z1, wk.z2, v, f, rc, use_pre);
          if constexpr (GEG == 3) gn_stats_chunk(p, f, row, row0, n, lane);
          if constexpr (GEG == 4) {  // GELU (erf) of the biased result: the frozen text encoders' MLP fc1
#pragma unroll
            for (int i = 0; i < 32; ++i) f[i] = 0.5f * f[i] * (1.f + erff(f[i] * 0.70710678118654752f));
          }
          uint8_t* buf = ebuf + (chunk_seq & 1) * EPI_STAGE_BYTES;
          if (chunk_seq >= 2) {
            if (lane == 0) bulk_wait_read<1>();
            __syncwarp();
          }
          stage_row_bf16(buf, lane, f);
          fence_async_shared();
          __syncwarp();
          if (lane == 0 && row0 < p.M) {
            tma_store_4d(&tmD, buf, n, row0, wk.z1, wk.z2);
            bulk_commit();
          }
          ++chunk_seq;
        } else if (row < p.M) {
          epilogue_store<BN>(p, row, n, wk.z1, wk.z2, v);
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if constexpr (CG == 2)
          mbar_arrive_cluster(tempty_leader0 + acc * 8);
        else
          mbar_arrive(&tempty[acc]);
      }
      if (++acc == Cfg::NACC) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
    if (p.d_tma && lane == 0) bulk_wait_all();
  }
  tc_fence_before();
  if constexpr (CG == 2)
    cluster_sync();
  else
    __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    if constexpr (CG == 2)
      tmem_dealloc_2sm<Cfg::TMEM_COLS>(tmem_base);
    else
      tmem_dealloc<Cfg::TMEM_COLS>(tmem_base);
  }
}

// ====================================================================== host side

static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  // The encoder is a driver call that validates the global address against the CURRENT context.
  // A thread whose first CUDA work is one of our launches (autograd's device worker thread: torch
  // skips cudaSetDevice when the device index already matches) has no context bound yet and the
  // encoder would fail with CUDA_ERROR_INVALID_CONTEXT; cudaFree(0) binds the primary context.
  thread_local bool bound = false;
  if (!bound) {
    cudaFree(nullptr);
    bound = true;
  }
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void* ptr = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
  });
  return fn;
}

PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() { return encode_fn(); }

// 4-D bf16 map. dims innermost-first; strides in ELEMENTS for dims 1..3.
static int make_map(CUtensorMap* map, const void* base, const uint64_t dims[4],
                    const int64_t strides_el[3], const uint32_t box[4], const uint32_t estr[4],
                    CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_128B, int esize = 2) {
  auto fn = encode_fn();
  if (!fn) {
    set_error("cuTensorMapEncodeTiled unavailable");
    return DP_ERR_DRIVER;
  }
  cuuint64_t gdim[4];
  cuuint64_t gstr[3];
  for (int i = 0; i < 4; ++i) gdim[i] = dims[i] ? dims[i] : 1;
  for (int i = 0; i < 3; ++i) {
    int64_t s = strides_el[i] * esize;
    if (gdim[i + 1] == 1 && (s <= 0 || s % 16)) {
      // degenerate dimension: any legal stride works
      s = 16;
    }
    if (s <= 0 || s % 16) {
      set_error("TMA stride not a positive multiple of 16 bytes");
      return DP_ERR_UNSUPPORTED;
    }
    gstr[i] = static_cast<cuuint64_t>(s);
  }
  if (reinterpret_cast<uintptr_t>(base) % 16) {
    set_error("TMA base pointer not 16-byte aligned");
    return DP_ERR_UNSUPPORTED;
  }
  cuuint32_t bx[4], es[4];
  for (int i = 0; i < 4; ++i) {
    bx[i] = box[i];
    es[i] = estr[i];
  }
  // Encoded maps are cached per host thread: the caching allocator hands the same addresses back every
  // iteration, so after the first step almost every launch finds its (address, geometry) maps here
  // instead of re-encoding three descriptors per GEMM on the host's critical path.
  struct Key {
    const void* base;
    cuuint64_t gdim[4], gstr[3];
    cuuint32_t bx[4], es[4];
    int swz, esize;
  };
  struct Slot {
    Key k;
    CUtensorMap m;
    bool used;
  };
  constexpr int kSlots = 8192;
  thread_local Slot* cache = nullptr;
  if (!cache) cache = new Slot[kSlots]();
  Key k{};
  k.base = base;
  for (int i = 0; i < 4; ++i) {
    k.gdim[i] = gdim[i];
    k.bx[i] = bx[i];
    k.es[i] = es[i];
  }
  for (int i = 0; i < 3; ++i) k.gstr[i] = gstr[i];
  k.swz = static_cast<int>(swz);
  k.esize = esize;
  uint64_t hsh = 1469598103934665603ull;
  const unsigned char* kb = reinterpret_cast<const unsigned char*>(&k);
  for (size_t i = 0; i < sizeof(Key); ++i) hsh = (hsh ^ kb[i]) * 1099511628211ull;
  Slot& slot = cache[hsh & (kSlots - 1)];
  if (slot.used && memcmp(&slot.k, &k, sizeof(Key)) == 0) {
    *map = slot.m;
    return 0;
  }
  CUresult r = fn(map, esize == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4,
                  const_cast<void*>(base), gdim, gstr,
                  bx, es, CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r == CUDA_SUCCESS) {
    slot.k = k;
    slot.m = *map;
    slot.used = true;
  }
  if (r != CUDA_SUCCESS) {
    char buf[256];
    snprintf(buf, sizeof(buf),
             "cuTensorMapEncodeTiled failed (%d): dims %llu,%llu,%llu,%llu box %u,%u,%u,%u", (int)r,
             (unsigned long long)gdim[0], (unsigned long long)gdim[1],
             (unsigned long long)gdim[2], (unsigned long long)gdim[3], bx[0], bx[1], bx[2], bx[3]);
    set_error(buf);
    return DP_ERR_DRIVER;
  }
  return 0;
}

static bool halo_enabled() {
  static const bool on = [] {
    const char* e = getenv("DP_HALO");
    return e ? atoi(e) != 0 : true;
  }();
  return on;
}

template <int BN, int CG, bool HALO = false, bool RES = false, int GEG = 0>
static int launch_tc(const CUtensorMap& ma, const CUtensorMap& mb, const CUtensorMap& md,
                     TcParams p, int max_ctas, cudaStream_t st, const CUtensorMap* md2 = nullptr) {
  using Cfg = TcCfg<BN, CG, HALO>;
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(tc_gemm_kernel<BN, CG, HALO, RES, GEG>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(Cfg::SMEM));
    if (e != cudaSuccess) {
      set_error(std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(e));
      return e;
    }
    attr_set = true;
  }
  const long long units = p.stream_k ? (long long)p.tiles_m * p.tiles_n * p.nbatch * p.num_kb
                                     : (long long)p.tiles_m * p.tiles_n * p.splits * p.nbatch;
  const int max_units = max_ctas / CG;
  const int grid = CG * static_cast<int>(units < max_units ? units : max_units);
  if (grid <= 0) return 0;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(GEMM_THREADS);
  cfg.dynamicSmemBytes = Cfg::SMEM;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CG;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  cudaError_t e = cudaLaunchKernelEx(&cfg, tc_gemm_kernel<BN, CG, HALO, RES, GEG>, ma, mb, md, md2 ? *md2 : md, p);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error(std::string("tc_gemm launch: ") + cudaGetErrorString(e));
    return e;
  }
  return 0;
}

// CTA pairs (cta_group::2, M = 256 per pair) halve the per-SM shared-memory traffic of B;
// used when the 256-row tiling wastes no more rows than the 128-row one and each CTA's half
// of the B tile is a legal TMA box (64-column multiples for MN-major B).
static int env_int(const char* name) {
  const char* v = getenv(name);
  return v ? atoi(v) : 0;
}

// Measured (tools/tile_sweep.py): pairs help long-K GEMMs, single CTAs win for short K
// (K <= 512: 32768x320x320 327 vs 273 TF/s, 32768x2560x320 672 vs 596 TF/s).
static int decide_cg(int M, int bn, bool b_mn_major, int K) {
  static const int forced = env_int("DP_FORCE_CG");  // experiments only
  if (forced == 1) return 1;
  if (M < 256) return 1;
  if (!forced && K <= 512) return 1;
  if (forced == 2 && !(b_mn_major && (bn / 2) % 64)) return 2;
  if (b_mn_major && (bn / 2) % 64) return 1;
  const long long r1 = (long long)((M + 127) / 128) * 128, r2 = (long long)((M + 255) / 256) * 256;
  return r2 <= r1 ? 2 : 1;
}

// Tile width: minimise padded columns plus a per-tile overhead, e.g. N=320 -> 2 x 160,
// N=2880 -> 13 x 224, N=1280 -> 5 x 256. MN-major B operands are loaded in 64-column TMA
// boxes, so they only use multiples of 64.
static int pick_bn(int N, bool b_mn_major) {
  static const int forced = env_int("DP_FORCE_BN");  // experiments only
  if (forced && (!b_mn_major || forced % 64 == 0)) return forced;
  static const int kAll[] = {64, 96, 128, 160, 192, 224, 256};
  static const int kMn[] = {64, 128, 192, 256};
  const int* cand = b_mn_major ? kMn : kAll;
  const int ncand = b_mn_major ? 4 : 7;
  int best = 64;
  long best_cost = -1;
  for (int i = 0; i < ncand; ++i) {
    const int bn = cand[i];
    const long tiles = (N + bn - 1) / bn;
    const long cost = tiles * bn + 24 * tiles;
    if (best_cost < 0 || cost < best_cost || (cost == best_cost && bn > best)) {
      best = bn;
      best_cost = cost;
    }
  }
  return best;
}

// BN = 320 (two N = 160 MMAs per k-step, one accumulator buffer) for N = 320 / 640 / 960 with
// K-major B, CTA pairs and long K: B traffic per MMA cycle drops from (16 + 10) KB / 320 cycles
// (BN 160) to (16 + 20) KB / 640 cycles per SM; the single accumulator exposes the epilogue once
// per tile, which long K (>= 16 k-blocks) amortises.
static int widen_bn(int bn, int cg, bool b_mn, int N, int num_kb) {
  static const int off = env_int("DP_NO_BN320");  // experiments only
  if (off || cg != 2 || b_mn || num_kb < 16) return bn;
  if (N == 320 || N == 640 || N == 960) return 320;
  return bn;
}

// Tile choice for bf16 STORE GEMMs (linears): a wave-aware cost over (BN, CTA pair) candidates,
//   cost = waves(units, SMs / cg) * (num_kb * max(2*BN MMA cycles, L2 bytes per k-block / 80 B/clk)
//          + 2500 [+1500 for the single-accumulator BN 320])
// (fitted on the device-time sweep tools/tile_sweep2.py: e.g. 2048x1280x1280 prefers 128 single-CTA
// 128x160 tiles in one wave over 40 pair tiles of 256x256; 8192^3 keeps pairs of 256).
static void choose_tile(int M, int N, int K, bool b_mn, int& bn_out, int& cg_out) {
  static const int forced_bn = env_int("DP_FORCE_BN"), forced_cg = env_int("DP_FORCE_CG");
  // sustainable L2 -> SM operand feed per SM (bytes per clock) in the cost model (DP_TILE_FEED: experiments)
  static const double feed = env_int("DP_TILE_FEED") > 0 ? env_int("DP_TILE_FEED") : 64.0;
  const int num_kb = (K + BK - 1) / BK;
  double best = -1.0;
  for (int cg = 1; cg <= 2; ++cg) {
    if (cg == 2 && (M < 256 || num_kb <= 8)) continue;  // short K: pairs measured slower
    if (forced_cg && cg != forced_cg) continue;
    for (int bn = 64; bn <= 320; bn += 32) {
      if (bn == 288) continue;
      if (b_mn && bn % 64) continue;
      if (b_mn && cg == 2 && (bn / 2) % 64) continue;
      if (bn == 320 && (cg != 2 || b_mn || num_kb < 16)) continue;
      if (forced_bn && bn != forced_bn) continue;
      const long long units = (long long)((M + 128 * cg - 1) / (128 * cg)) * ((N + bn - 1) / bn);
      const long long per_wave = kNumSMs / cg;
      const long long waves = (units + per_wave - 1) / per_wave;
      const double l2 = (16384.0 + (bn / cg) * 128.0) / feed;
      const double per_kb = (2.0 * bn > l2) ? 2.0 * bn : l2;
      const double cost = waves * (num_kb * per_kb + 2500.0 + (bn > 256 ? 1500.0 : 0.0));
      if (best < 0 || cost < best * 0.999 || (cost <= best * 1.001 && bn > bn_out)) {
        best = cost;
        bn_out = bn;
        cg_out = cg;
      }
    }
  }
}

// bf16 STORE outputs with TMA-legal strides are written by tensor stores (box 32 x 32,
// SWIZZLE_64B); fp32 / atomic outputs keep the direct per-thread path.
// fp32 ATOMIC_ADD outputs (weight gradients, split-K partials) are added by TMA reduce-add of 32 x 16
// fp32 boxes staged in shared memory (d_tma = 2): bulk L2 reductions instead of one red.v4 per lane
// and 16 bytes.
static int make_dmap(CUtensorMap* md, TcParams& p, int M, int N, int b1, int b2) {
  static const int no_red = env_int("DP_NO_TMA_REDUCE");  // experiments: per-thread atomics
  p.d_tma = 0;
  if (!p.vec_ok) return 0;
  const bool red = p.d_f32 && p.out_mode == DP_OUT_ATOMIC_ADD && !no_red;
  if (!red && (p.d_f32 || p.out_mode != DP_OUT_STORE)) return 0;
  const uint64_t d[4] = {(uint64_t)N, (uint64_t)M, (uint64_t)b1, (uint64_t)b2};
  const int64_t s[3] = {p.d_ld, b1 > 1 ? p.d_bs1 : (int64_t)M * p.d_ld,
                        b2 > 1 ? p.d_bs2 : (int64_t)M * p.d_ld * b1};
  const uint32_t box[4] = {red ? 16u : 32u, 32, 1, 1};
  const uint32_t ones[4] = {1, 1, 1, 1};
  if (make_map(md, p.D, d, s, box, ones, CU_TENSOR_MAP_SWIZZLE_64B, red ? 4 : 2) == 0) p.d_tma = red ? 2 : 1;
  return 0;
}

template <int CG, bool RES>
static int launch_cg_r(int bn, const CUtensorMap& ma, const CUtensorMap& mb, const CUtensorMap& md,
                       TcParams& p, cudaStream_t st) {
  switch (bn) {
    case 64: return launch_tc<64, CG, false, RES>(ma, mb, md, p, kNumSMs, st);
    case 96: return launch_tc<96, CG, false, RES>(ma, mb, md, p, kNumSMs, st);
    case 128: return launch_tc<128, CG, false, RES>(ma, mb, md, p, kNumSMs, st);
    case 160: return launch_tc<160, CG, false, RES>(ma, mb, md, p, kNumSMs, st);
    case 192: return launch_tc<192, CG, false, RES>(ma, mb, md, p, kNumSMs, st);
    case 224: return launch_tc<224, CG, false, RES>(ma, mb, md, p, kNumSMs, st);
    case 320:
      if constexpr (CG == 2) return launch_tc<320, 2, false, RES>(ma, mb, md, p, kNumSMs, st);
      [[fallthrough]];
    default: return launch_tc<256, CG, false, RES>(ma, mb, md, p, kNumSMs, st);
  }
}

template <int CG>
static int launch_cg(int bn, const CUtensorMap& ma, const CUtensorMap& mb, const CUtensorMap& md,
                     TcParams& p, cudaStream_t st) {
  // bf16 residual epilogue through TMA stores: the instantiation with residual prefetch
  if (!p.halo && p.R && !p.d_f32 && p.vec_ok && p.d_tma) return launch_cg_r<CG, true>(bn, ma, mb, md, p, st);
  if (!p.halo) return launch_cg_r<CG, false>(bn, ma, mb, md, p, st);
  if (p.halo) {
    switch (bn) {
      case 128: return launch_tc<128, CG, true>(ma, mb, md, p, kNumSMs, st);
      case 160: return launch_tc<160, CG, true>(ma, mb, md, p, kNumSMs, st);
      case 192: return launch_tc<192, CG, true>(ma, mb, md, p, kNumSMs, st);
      default: return launch_tc<256, CG, true>(ma, mb, md, p, kNumSMs, st);
    }
  }
  switch (bn) {
    case 64: return launch_tc<64, CG>(ma, mb, md, p, kNumSMs, st);
    case 96: return launch_tc<96, CG>(ma, mb, md, p, kNumSMs, st);
    case 128: return launch_tc<128, CG>(ma, mb, md, p, kNumSMs, st);
    case 160: return launch_tc<160, CG>(ma, mb, md, p, kNumSMs, st);
    case 192: return launch_tc<192, CG>(ma, mb, md, p, kNumSMs, st);
    case 224: return launch_tc<224, CG>(ma, mb, md, p, kNumSMs, st);
    case 320:
      if constexpr (CG == 2) return launch_tc<320, 2>(ma, mb, md, p, kNumSMs, st);
      [[fallthrough]];
    default: return launch_tc<256, CG>(ma, mb, md, p, kNumSMs, st);
  }
}

static void choose_split(TcParams& p, int requested, bool allowed);

// ---------------------------------------------------------------- split-K for bf16 outputs
// A bf16 STORE launch whose tiles cover only a fraction of the SMs (U-Net 4x4 / 8x8 level
// convs, M = 32 time-embedding linears, ...) is re-run as an fp32 atomic split-K / stream-K
// GEMM into a caller-provided workspace, then finished (bias, residual, bf16) by one
// elementwise pass: the tensor cores of every SM work on the long K instead of a few.
__global__ void __launch_bounds__(256)
    splitk_finish_kernel(const float* __restrict__ ws, __nv_bfloat16* __restrict__ D, int64_t d_ld,
                         int64_t d_bs1, int64_t d_bs2, const float* __restrict__ bias,
                         const __nv_bfloat16* __restrict__ R, int64_t r_ld, int64_t r_bs1,
                         int64_t r_bs2, int M, int N, int batch1, int64_t total) {
  DP_PDL_ENTRY();
  const int nv = N / 8;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int v = static_cast<int>(i % nv);
    const int64_t r = i / nv;
    const int m = static_cast<int>(r % M);
    const int z = static_cast<int>(r / M);
    const int z1 = z % batch1, z2 = z / batch1;
    const float4* w = reinterpret_cast<const float4*>(ws + ((int64_t)z * M + m) * N + v * 8);
    const float4 a = w[0], b = w[1];
    float f[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
    if (bias) {
      if ((reinterpret_cast<uintptr_t>(bias) & 15) == 0) {  // two 16-byte loads
        const float4 b0 = __ldg(reinterpret_cast<const float4*>(bias + v * 8));
        const float4 b1 = __ldg(reinterpret_cast<const float4*>(bias + v * 8 + 4));
        f[0] += b0.x; f[1] += b0.y; f[2] += b0.z; f[3] += b0.w;
        f[4] += b1.x; f[5] += b1.y; f[6] += b1.z; f[7] += b1.w;
      } else {
#pragma unroll
        for (int j = 0; j < 8; ++j) f[j] += __ldg(bias + v * 8 + j);
      }
    }
    if (R) {
      const uint4 u = *reinterpret_cast<const uint4*>(R + z1 * r_bs1 + z2 * r_bs2 + (int64_t)m * r_ld + v * 8);
      const __nv_bfloat16* rb = reinterpret_cast<const __nv_bfloat16*>(&u);
#pragma unroll
      for (int j = 0; j < 8; ++j) f[j] += __bfloat162float(rb[j]);
    }
    uint4 o;
    o.x = pack_bf16x2(f[0], f[1]);
    o.y = pack_bf16x2(f[2], f[3]);
    o.z = pack_bf16x2(f[4], f[5]);
    o.w = pack_bf16x2(f[6], f[7]);
    *reinterpret_cast<uint4*>(D + z1 * d_bs1 + z2 * d_bs2 + (int64_t)m * d_ld + v * 8) = o;
  }
}

// zero the split-K workspace as a programmatic-dependent-launch kernel: a cudaMemsetAsync node between
// two PDL kernels serialises the stream twice (the memset waits for the previous kernel to drain and the
// split GEMM cannot overlap its prologue with the memset), 16-byte stores
__global__ void __launch_bounds__(256) ws_zero_kernel(float4* __restrict__ ws, int64_t n4) {
  DP_PDL_ENTRY();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x)
    ws[i] = make_float4(0.f, 0.f, 0.f, 0.f);
}

static bool splitk_memset() {  // DP_SPLITK_MEMSET=1: the cudaMemsetAsync path (A/B)
  static const bool v = env_int("DP_SPLITK_MEMSET") > 0;
  return v;
}

// wave efficiency (percent) below which a bf16 launch is split (DP_SPLITK_FRAC; experiments)
static int splitk_pct() {
  static const int v = [] {
    const char* e = getenv("DP_SPLITK_FRAC");
    return e ? atoi(e) : 75;
  }();
  return v;
}

// A bf16 STORE launch whose tiles fill their waves poorly (efficiency = tiles / (waves x tile slots),
// e.g. 40 CTA-pair tiles of an 8x8-map conv on 74 pair slots: 54%) and whose K is long enough for the
// fp32 stream-K pass plus the finish pass to pay: the whole-K tiles were leaving up to half the SMs
// idle (previous rule: split only below half of the SMs).
static int64_t splitk_bytes(const TcParams& p, int cg, int M, int N) {
  if (p.d_f32 || p.out_mode != DP_OUT_STORE || !p.vec_ok || (N % 8) || p.num_kb < 8) return 0;
  const long long units = (long long)p.tiles_m * p.tiles_n * p.nbatch;
  const long long slots = kNumSMs / cg;
  const long long waves = (units + slots - 1) / slots;
  const bool under_half = units * cg * 100 < (long long)kNumSMs * 50;
  const bool poor_waves = p.num_kb >= 16 && units * 100 < waves * slots * splitk_pct();
  if (!under_half && !poor_waves) return 0;
  return 4LL * M * N * p.nbatch;
}

static int launch_bn(int bn, int cg, const CUtensorMap& ma, const CUtensorMap& mb, TcParams& p, int M,
                     int N, int b1, int b2, cudaStream_t st, float* ws = nullptr, int64_t ws_bytes = 0) {
  const int64_t need = splitk_bytes(p, cg, M, N);
  if (need > 0 && ws && ws_bytes >= need && (reinterpret_cast<uintptr_t>(ws) % 16) == 0) {
    TcParams q = p;
    q.D = ws;
    q.d_f32 = 1;
    q.out_mode = DP_OUT_ATOMIC_ADD;
    q.bias = nullptr;
    q.R = nullptr;
    q.d_ld = N;
    q.d_bs1 = (int64_t)M * N;
    q.d_bs2 = (int64_t)M * N * b1;
    q.vec_ok = (N % 4) == 0;
    q.d_tma = 0;
    choose_split(q, 0, true);
    CUtensorMap mq = ma;
    make_dmap(&mq, q, M, N, b1, b2);
    cudaError_t e = cudaSuccess;
    if (splitk_memset() || (need % 16) != 0) {
      e = cudaMemsetAsync(ws, 0, need, st);
    } else {
      const int64_t n4 = need / 16;
      const int64_t zb = (n4 + 255) / 256;
      launch_k(ws_zero_kernel, dim3(static_cast<unsigned>(zb < 4 * kNumSMs ? zb : 4 * kNumSMs)), dim3(256), 0, st,
               reinterpret_cast<float4*>(ws), n4);
      e = cudaGetLastError();
    }
    if (e != cudaSuccess) {
      set_error(std::string("split-K workspace memset: ") + cudaGetErrorString(e));
      return e;
    }
    int rc = cg == 2 ? launch_cg<2>(bn, ma, mb, mq, q, st) : launch_cg<1>(bn, ma, mb, mq, q, st);
    if (rc) return rc;
    const int64_t total = (int64_t)p.nbatch * M * (N / 8);
    const int64_t want = (total + 255) / 256;
    const int grid = static_cast<int>(want < 8 * kNumSMs ? want : 8 * kNumSMs);
    launch_k(splitk_finish_kernel, dim3(grid), dim3(256), 0, st, ws, reinterpret_cast<__nv_bfloat16*>(p.D), p.d_ld, p.d_bs1,
                                               p.d_bs2, p.bias, reinterpret_cast<const __nv_bfloat16*>(p.R),
                                               p.r_ld, p.r_bs1, p.r_bs2, M, N, b1, total);
    e = cudaGetLastError();
    if (e != cudaSuccess) {
      set_error(std::string("split-K finish: ") + cudaGetErrorString(e));
      return e;
    }
    return 0;
  }
  CUtensorMap md = ma;
  make_dmap(&md, p, M, N, b1, b2);
  return cg == 2 ? launch_cg<2>(bn, ma, mb, md, p, st) : launch_cg<1>(bn, ma, mb, md, p, st);
}

static void choose_split(TcParams& p, int requested, bool allowed) {
  const int tiles = p.tiles_m * p.tiles_n * p.nbatch;
  int splits = 1;
  p.stream_k = 0;
  static const int sk_target = env_int("DP_SK_TARGET");  // experiments: split-K to ~N CTAs
  if (allowed && requested <= 0 && sk_target > 0) {
    splits = (sk_target + tiles - 1) / tiles;
    const int max_split = p.num_kb / 4 > 0 ? p.num_kb / 4 : 1;
    if (splits > max_split) splits = max_split;
    p.kb_per_split = (p.num_kb + splits - 1) / splits;
    p.splits = (p.num_kb + p.kb_per_split - 1) / p.kb_per_split;
    return;
  }
  if (allowed && requested <= 0 && tiles < 2 * kNumSMs && (long long)tiles * p.num_kb >= 4 * kNumSMs) {
    // fp32 atomic output: balance k-iterations over all SMs (stream-K)
    p.stream_k = 1;
    p.splits = 1;
    p.kb_per_split = p.num_kb;
    return;
  }
  if (allowed) {
    if (requested > 0) {
      splits = requested;
    } else if (tiles < kNumSMs && p.num_kb >= 8) {
      splits = (2 * kNumSMs + tiles - 1) / tiles;
      const int max_split = p.num_kb / 4;
      if (splits > max_split) splits = max_split;
      if (splits < 1) splits = 1;
    }
  }
  p.kb_per_split = (p.num_kb + splits - 1) / splits;
  p.splits = (p.num_kb + p.kb_per_split - 1) / p.kb_per_split;
}

static void fill_epilogue(TcParams& p, void* D, int d_dtype, int64_t d_ld, int64_t d_bs1,
                          int64_t d_bs2, int out_mode, const float* bias, const void* R,
                          int64_t r_ld, int64_t r_bs1, int64_t r_bs2, float alpha) {
  p.D = D;
  p.d_f32 = d_dtype == DP_F32;
  p.d_ld = d_ld;
  p.d_bs1 = d_bs1;
  p.d_bs2 = d_bs2;
  p.out_mode = out_mode;
  p.bias = bias;
  p.R = R;
  p.r_ld = r_ld;
  p.r_bs1 = r_bs1;
  p.r_bs2 = r_bs2;
  p.alpha = alpha;
  const int esz = p.d_f32 ? 4 : 2;
  bool ok = (reinterpret_cast<uintptr_t>(D) % 16 == 0) && ((d_ld * esz) % 16 == 0) &&
            ((d_bs1 * esz) % 16 == 0) && ((d_bs2 * esz) % 16 == 0);
  if (R)
    ok = ok && (reinterpret_cast<uintptr_t>(R) % 16 == 0) && ((r_ld * esz) % 16 == 0) &&
         ((r_bs1 * esz) % 16 == 0) && ((r_bs2 * esz) % 16 == 0);
  p.vec_ok = ok ? 1 : 0;
}

// Linear forward with the GEGLU epilogue (see DpGemmArgs::geglu_out): tile = BN/2 output columns of
// both halves, CTA pairs for M >= 256 with each CTA staging one half of B.
static int tc_gemm_geglu(const DpGemmArgs* a, cudaStream_t st) {
  const int F = a->N / 2;
  if (a->d_dtype != DP_BF16 || a->dtype != DP_BF16 || a->out_mode != DP_OUT_STORE || a->Res || !a->bias ||
      a->a_mn_major || a->b_mn_major || (a->batch1 > 1) || (a->batch2 > 1) || a->N % 128 || F % 64 ||
      a->alpha != 1.f) {
    set_error("gemm geglu epilogue: bf16 K-major linear with bias, N = 2F, F % 64 == 0, no residual/batch");
    return DP_ERR_UNSUPPORTED;
  }
  const int bn = (F % 128 == 0) ? 256 : 128;
  const int cg = a->M >= 256 ? 2 : 1;
  TcParams p{};
  p.M = a->M;
  p.N = a->N;
  p.F = F;
  p.geglu = 1;
  p.num_kb = (a->K + BK - 1) / BK;
  p.tiles_m = (a->M + BM * cg - 1) / (BM * cg);
  p.tiles_n = F / (bn / 2);
  p.batch1 = 1;
  p.nbatch = 1;
  p.a_mode = A_KMAJ;
  p.b_mode = B_KMAJ;
  choose_split(p, 0, false);
  fill_epilogue(p, a->D, DP_BF16, a->d_ld, 0, 0, DP_OUT_STORE, a->bias, nullptr, 0, 0, 0, 1.f);
  if (!p.vec_ok || reinterpret_cast<uintptr_t>(a->geglu_out) % 16 || (a->geglu_ld * 2) % 16 ||
      reinterpret_cast<uintptr_t>(a->bias) % 16) {
    set_error("gemm geglu epilogue: 16-byte aligned outputs, bias and row strides");
    return DP_ERR_ARGS;
  }
  CUtensorMap ma, mb, md, md2;
  const uint32_t ones[4] = {1, 1, 1, 1};
  {
    const uint64_t d[4] = {(uint64_t)a->K, (uint64_t)a->M, 1, 1};
    const int64_t s[3] = {a->a_ld, (int64_t)a->M * a->a_ld, (int64_t)a->M * a->a_ld};
    const uint32_t box[4] = {BK, BM, 1, 1};
    if (int e = make_map(&ma, a->A, d, s, box, ones)) return e;
  }
  {
    const uint64_t d[4] = {(uint64_t)a->K, (uint64_t)a->N, 1, 1};
    const int64_t s[3] = {a->b_ld, (int64_t)a->N * a->b_ld, (int64_t)a->N * a->b_ld};
    const uint32_t box[4] = {BK, (uint32_t)(bn / 2), 1, 1};
    if (int e = make_map(&mb, a->B, d, s, box, ones)) return e;
  }
  make_dmap(&md, p, a->M, a->N, 1, 1);
  if (!p.d_tma) {
    set_error("gemm geglu epilogue: output not TMA-storable");
    return DP_ERR_ARGS;
  }
  {
    const uint64_t d[4] = {(uint64_t)F, (uint64_t)a->M, 1, 1};
    const int64_t s[3] = {a->geglu_ld, (int64_t)a->M * a->geglu_ld, (int64_t)a->M * a->geglu_ld};
    const uint32_t box[4] = {32, 32, 1, 1};
    if (int e = make_map(&md2, a->geglu_out, d, s, box, ones, CU_TENSOR_MAP_SWIZZLE_64B)) return e;
  }
  if (cg == 2)
    return bn == 256 ? launch_tc<256, 2, false, false, 1>(ma, mb, md, p, kNumSMs, st, &md2)
                     : launch_tc<128, 2, false, false, 1>(ma, mb, md, p, kNumSMs, st, &md2);
  return bn == 256 ? launch_tc<256, 1, false, false, 1>(ma, mb, md, p, kNumSMs, st, &md2)
                   : launch_tc<128, 1, false, false, 1>(ma, mb, md, p, kNumSMs, st, &md2);
}

int tc_gemm(const DpGemmArgs* a, cudaStream_t st, int64_t* query = nullptr) {
  if (query) *query = 0;
  if (a->M <= 0 || a->N <= 0 || a->K <= 0) return 0;
  if (a->geglu_mode == 1) return query ? 0 : tc_gemm_geglu(a, st);
  if (a->geglu_mode == 2) {
    if (query) return 0;
    if (a->d_dtype != DP_BF16 || a->out_mode != DP_OUT_STORE || a->Res || a->bias || a->a_mn_major ||
        a->b_mn_major || a->batch1 > 1 || a->batch2 > 1 || a->N % 32 || a->alpha != 1.f ||
        reinterpret_cast<uintptr_t>(a->geglu_out) % 16 || a->geglu_ld % 8) {
      set_error("gemm geglu backward epilogue: bf16 K-major dgrad, N % 32 == 0, aligned h, no bias/residual");
      return DP_ERR_UNSUPPORTED;
    }
  }
  if (a->out_mode == DP_OUT_ATOMIC_ADD && a->d_dtype != DP_F32) {
    set_error("atomic accumulation needs an fp32 output");
    return DP_ERR_ARGS;
  }
  int bn, cg;
  if (a->out_mode == DP_OUT_STORE && a->d_dtype == DP_BF16 && !env_int("DP_OLD_TILES")) {
    bn = 64;
    cg = 1;
    choose_tile(a->M, a->N, a->K, a->b_mn_major != 0, bn, cg);
  } else {
    const int bn0 = pick_bn(a->N, a->b_mn_major != 0);
    cg = decide_cg(a->M, bn0, a->b_mn_major != 0, a->K);
    bn = widen_bn(bn0, cg, a->b_mn_major != 0, a->N, (a->K + BK - 1) / BK);
    // weight gradients (fp32 accumulate, both operands MN-major, long K): 256 x 256 CTA-pair tiles
    // for M >= 1024, N >= 512, padding included (8192x5120x640: 67 -> 52 us, 8192x1920x640: 31 -> 27).
    // These GEMMs are bound by the TMA feed (L2 -> SM bytes per MMA cycle), not the tensor core: 128 x 128 single-CTA tiles move 128 B per SM per MMA
    // cycle, pairs of 256 x 256 62.5 (the swapped conv weight gradient measured 85 -> 59 us at
    // 16x16x640 with the same change; DP_WG_NARROW=1: previous choice, experiments)
    static const bool narrow = env_int("DP_WG_NARROW") != 0;
    if (!narrow && a->out_mode == DP_OUT_ATOMIC_ADD && a->a_mn_major && a->b_mn_major && a->M >= 1024 &&
        a->N >= 512 && a->K >= 1024) {  // (M = 640 measured slower with the padded pairs)
      bn = 256;
      cg = 2;
    }
  }
  if (a->geglu_mode == 2) {  // the GEGLU-backward instantiations: 128 / 256-wide tiles
    bn = (a->N % 256 == 0) ? 256 : 128;
    cg = (a->M >= 256 && a->K > 512) ? 2 : 1;
  }
  if (a->geglu_mode == 3) {  // GELU epilogue instantiations (GEG = 4): 128 / 256-wide tiles, no split-K
    if (a->dtype != DP_BF16 || a->d_dtype != DP_BF16 || a->out_mode != DP_OUT_STORE || a->Res ||
        a->a_mn_major || a->b_mn_major || a->batch1 > 1 || a->batch2 > 1 || a->N % 128 || a->alpha != 1.f) {
      set_error("gemm gelu epilogue: bf16 K-major linear store, N % 128 == 0, no residual / batch / alpha");
      return DP_ERR_UNSUPPORTED;
    }
    bn = (a->N % 256 == 0) ? 256 : 128;
    cg = a->M >= 256 ? 2 : 1;
  }
  TcParams p{};
  p.M = a->M;
  p.N = a->N;
  p.num_kb = (a->K + BK - 1) / BK;
  p.tiles_m = (a->M + BM * cg - 1) / (BM * cg);
  p.tiles_n = (a->N + bn - 1) / bn;
  p.batch1 = a->batch1 > 0 ? a->batch1 : 1;
  const int batch2 = a->batch2 > 0 ? a->batch2 : 1;
  p.nbatch = p.batch1 * batch2;
  p.a_mode = a->a_mn_major ? A_MNMAJ : A_KMAJ;
  p.b_mode = a->b_mn_major ? B_MNMAJ : B_KMAJ;
  choose_split(p, a->split_k, a->out_mode == DP_OUT_ATOMIC_ADD);
  fill_epilogue(p, a->D, a->d_dtype, a->d_ld, a->d_bs1, a->d_bs2, a->out_mode, a->bias, a->Res,
                a->r_ld, a->r_bs1, a->r_bs2, a->alpha);
  if (query) {
    *query = a->geglu_mode == 3 ? 0 : splitk_bytes(p, cg, a->M, a->N);
    return 0;
  }
  CUtensorMap ma, mb;
  const uint32_t ones[4] = {1, 1, 1, 1};
  {
    const int64_t s[3] = {a->a_ld, a->a_bs1, a->a_bs2};
    if (a->a_mn_major) {
      const uint64_t d[4] = {(uint64_t)a->M, (uint64_t)a->K, (uint64_t)p.batch1, (uint64_t)batch2};
      const uint32_t box[4] = {64, BK, 1, 1};
      if (int e = make_map(&ma, a->A, d, s, box, ones)) return e;
    } else {
      const uint64_t d[4] = {(uint64_t)a->K, (uint64_t)a->M, (uint64_t)p.batch1, (uint64_t)batch2};
      const uint32_t box[4] = {BK, BM, 1, 1};
      if (int e = make_map(&ma, a->A, d, s, box, ones)) return e;
    }
  }
  {
    const int64_t s[3] = {a->b_ld, a->b_bs1, a->b_bs2};
    if (a->b_mn_major) {
      const uint64_t d[4] = {(uint64_t)a->N, (uint64_t)a->K, (uint64_t)p.batch1, (uint64_t)batch2};
      const uint32_t box[4] = {64, BK, 1, 1};
      if (int e = make_map(&mb, a->B, d, s, box, ones)) return e;
    } else {
      const uint64_t d[4] = {(uint64_t)a->K, (uint64_t)a->N, (uint64_t)p.batch1, (uint64_t)batch2};
      const uint32_t box[4] = {BK, (uint32_t)(bn / cg / (bn > 256 ? 2 : 1)), 1, 1};
      if (int e = make_map(&mb, a->B, d, s, box, ones)) return e;
    }
  }
  if (a->geglu_mode == 2) {
    p.geglu = 2;
    p.F = a->N;
    p.gh = a->geglu_out;
    p.gh_ld = a->geglu_ld;
    CUtensorMap md = ma;
    make_dmap(&md, p, a->M, 2 * a->N, 1, 1);  // dh = [da | dg]: 2F columns
    if (!p.d_tma) {
      set_error("gemm geglu backward epilogue: output not TMA-storable");
      return DP_ERR_ARGS;
    }
    if (cg == 2)
      return bn == 256 ? launch_tc<256, 2, false, false, 2>(ma, mb, md, p, kNumSMs, st)
                       : launch_tc<128, 2, false, false, 2>(ma, mb, md, p, kNumSMs, st);
    return bn == 256 ? launch_tc<256, 1, false, false, 2>(ma, mb, md, p, kNumSMs, st)
                     : launch_tc<128, 1, false, false, 2>(ma, mb, md, p, kNumSMs, st);
  }
  if (a->geglu_mode == 3) {
    CUtensorMap md = ma;
    make_dmap(&md, p, a->M, a->N, 1, 1);
    if (!p.d_tma) {
      set_error("gemm gelu epilogue: output not TMA-storable");
      return DP_ERR_ARGS;
    }
    if (cg == 2)
      return bn == 256 ? launch_tc<256, 2, false, false, 4>(ma, mb, md, p, kNumSMs, st)
                       : launch_tc<128, 2, false, false, 4>(ma, mb, md, p, kNumSMs, st);
    return bn == 256 ? launch_tc<256, 1, false, false, 4>(ma, mb, md, p, kNumSMs, st)
                     : launch_tc<128, 1, false, false, 4>(ma, mb, md, p, kNumSMs, st);
  }
  return launch_bn(bn, cg, ma, mb, p, a->M, a->N, p.batch1, batch2, st, a->workspace, a->workspace_bytes);
}

// Tile the output pixels (P x Q per image, N images) with boxes of `pixels`
// pixels that are contiguous in NHWC order. Returns false when the geometry
// does not tile (caller must lower through im2col instead).
static bool pixel_box(int P, int Q, int pixels, int& tw, int& th, int& tn) {
  if (Q >= pixels) {
    if (Q % pixels) return false;
    tw = pixels;
    th = 1;
    tn = 1;
    return true;
  }
  if (pixels % Q) return false;
  tw = Q;
  if (P * Q >= pixels) {
    if ((P * Q) % pixels) return false;
    th = pixels / Q;
    tn = 1;
    return true;
  }
  if (pixels % (P * Q)) return false;
  th = P;
  tn = pixels / (P * Q);
  return true;
}

int tc_conv_fwd(const DpConvArgs* a, cudaStream_t st, int64_t* query = nullptr) {
  if (query) *query = 0;
  if (a->C % 64) {
    set_error("implicit conv needs C % 64 == 0");
    return DP_ERR_UNSUPPORTED;
  }
  if (a->stride < 1 || a->stride > 2) {
    set_error("implicit conv supports stride 1 or 2");
    return DP_ERR_UNSUPPORTED;
  }
  TcParams p{};
  if (!pixel_box(a->P, a->Q, BM, p.tw, p.th, p.tn)) {
    set_error("output spatial size does not tile into 128-pixel boxes");
    return DP_ERR_UNSUPPORTED;
  }
  int bn = pick_bn(a->K, false);
  const int cg = decide_cg(a->N * a->P * a->Q, bn, false, a->R * a->S * a->C);
  p.M = a->N * a->P * a->Q;
  p.N = a->K;
  p.cblk = a->C / 64;
  // halo strips: 3x3, stride 1, symmetric 1-pixel padding, tiles inside one image row
  p.halo = (halo_enabled() && a->R == 3 && a->S == 3 && a->stride == 1 && a->pad_w == 1 && p.th == 1 &&
            p.tn == 1 && (bn == 128 || bn == 160 || bn == 192 || bn == 256)) ? 1 : 0;
  if (!p.halo) bn = widen_bn(bn, cg, false, a->K, a->R * a->S * p.cblk);
  p.num_kb = p.halo ? a->R * p.cblk : a->R * a->S * p.cblk;
  p.tiles_m = (p.M + BM * cg - 1) / (BM * cg);
  p.tiles_n = (a->K + bn - 1) / bn;
  p.batch1 = 1;
  p.nbatch = 1;
  p.a_mode = A_CONV;
  p.b_mode = B_KMAJ;
  p.P = a->P;
  p.Q = a->Q;
  p.stride = a->stride;
  p.pad_h = a->pad_h;
  p.pad_w = a->pad_w;
  p.S = a->S;
  p.C = a->C;
  choose_split(p, a->split_k, a->out_mode == DP_OUT_ATOMIC_ADD);
  fill_epilogue(p, a->y, a->dtype == DP_BF16 && a->out_mode != DP_OUT_ATOMIC_ADD ? DP_BF16 : DP_F32,
                a->K, 0, 0, a->out_mode, a->bias, a->Res, a->K, 0, 0, a->alpha);
  if (query) {
    *query = splitk_bytes(p, cg, p.M, p.N);
    return 0;
  }
  CUtensorMap ma, mb;
  {
    const uint64_t d[4] = {(uint64_t)a->C, (uint64_t)a->W, (uint64_t)a->H, (uint64_t)a->N};
    const int64_t s[3] = {a->C, (int64_t)a->W * a->C, (int64_t)a->H * a->W * a->C};
    const uint32_t box[4] = {64, (uint32_t)(p.halo ? HALO_ROWS : p.tw * a->stride),
                             (uint32_t)(p.th * a->stride), (uint32_t)p.tn};
    const uint32_t es[4] = {1, (uint32_t)a->stride, (uint32_t)a->stride, 1};
    if (int e = make_map(&ma, a->x, d, s, box, es)) return e;
  }
  {
    const int64_t Kdim = (int64_t)a->R * a->S * a->C;
    const uint64_t d[4] = {(uint64_t)Kdim, (uint64_t)a->K, 1, 1};
    const int64_t s[3] = {Kdim, 0, 0};
    const uint32_t box[4] = {BK, (uint32_t)(bn / cg / (bn > 256 ? 2 : 1)), 1, 1};
    const uint32_t ones[4] = {1, 1, 1, 1};
    if (int e = make_map(&mb, a->w, d, s, box, ones)) return e;
  }
  if (a->gn_sums) {
    // GroupNorm statistics epilogue (GEG == 3 instantiations: 128 / 256-wide tiles, no split-K)
    const int G = a->gn_groups;
    const int cpg = G > 0 ? a->K / G : 0;
    int lg = 0;
    while ((1 << lg) < cpg) ++lg;
    if (a->dtype != DP_BF16 || a->out_mode != DP_OUT_STORE || G <= 0 || a->K % G || (1 << lg) != cpg || lg < 2 ||
        lg > 5 || (a->P * a->Q) % 32 || (bn != 128 && bn != 256) || reinterpret_cast<uintptr_t>(a->gn_sums) % 16) {
      set_error("conv gn_sums: bf16 store, K / gn_groups a power of two in [4, 32], P*Q % 32 == 0, 128/256 tiles");
      return DP_ERR_UNSUPPORTED;
    }
    p.gn_sums = a->gn_sums;
    p.gn_lg = lg;
    p.gn_hw = a->P * a->Q;
    p.gn_G = G;
    cudaError_t e = cudaMemsetAsync(a->gn_sums, 0, sizeof(float) * 2 * (size_t)DP_GN_SLOTS * a->N * G, st);
    if (e != cudaSuccess) {
      set_error(std::string("gn_sums memset: ") + cudaGetErrorString(e));
      return e;
    }
    CUtensorMap md = ma;
    make_dmap(&md, p, p.M, p.N, 1, 1);
    if (p.d_tma != 1) {
      set_error("conv gn_sums: output not TMA-storable");
      return DP_ERR_UNSUPPORTED;
    }
    if (p.halo) {
      if (cg == 2)
        return bn == 256 ? launch_tc<256, 2, true, false, 3>(ma, mb, md, p, kNumSMs, st)
                         : launch_tc<128, 2, true, false, 3>(ma, mb, md, p, kNumSMs, st);
      return bn == 256 ? launch_tc<256, 1, true, false, 3>(ma, mb, md, p, kNumSMs, st)
                       : launch_tc<128, 1, true, false, 3>(ma, mb, md, p, kNumSMs, st);
    }
    if (cg == 2)
      return bn == 256 ? launch_tc<256, 2, false, false, 3>(ma, mb, md, p, kNumSMs, st)
                       : launch_tc<128, 2, false, false, 3>(ma, mb, md, p, kNumSMs, st);
    return bn == 256 ? launch_tc<256, 1, false, false, 3>(ma, mb, md, p, kNumSMs, st)
                     : launch_tc<128, 1, false, false, 3>(ma, mb, md, p, kNumSMs, st);
  }
  return launch_bn(bn, cg, ma, mb, p, p.M, p.N, 1, 1, st, a->workspace, a->workspace_bytes);
}

// Input gradient of a stride-1 convolution as an implicit GEMM over dy with the weights read
// tap-flipped in place (B_DGRAD): dx[n][h][w][c] = sum_{kk,r,s} dy[n][h+r-(R-1-pad_h)]
// [w+s-(S-1-pad_w)][kk] * w[kk][R-1-r][S-1-s][c]. Args: N,H,W,C describe dx, P,Q dy, x := dy,
// w := weights [K][R][S][C], y := dx. Strided convolutions zero-dilate dy first (dp_dilate).
int tc_conv_dgrad(const DpConvArgs* a, cudaStream_t st, int64_t* query = nullptr) {
  if (query) *query = 0;
  if (a->C % 64 || a->K % 64) {
    set_error("implicit dgrad needs C % 64 == 0 and K % 64 == 0");
    return DP_ERR_UNSUPPORTED;
  }
  if (a->stride != 1) {
    set_error("implicit dgrad is stride 1 (dilate dy for strided convolutions)");
    return DP_ERR_UNSUPPORTED;
  }
  TcParams p{};
  if (!pixel_box(a->H, a->W, BM, p.tw, p.th, p.tn)) {
    set_error("input spatial size does not tile into 128-pixel boxes");
    return DP_ERR_UNSUPPORTED;
  }
  const int bn = pick_bn(a->C, true);
  const int cg = decide_cg(a->N * a->H * a->W, bn, true, a->R * a->S * a->K);
  p.M = a->N * a->H * a->W;
  p.N = a->C;
  p.cblk = a->K / 64;
  p.num_kb = a->R * a->S * p.cblk;
  p.tiles_m = (p.M + BM * cg - 1) / (BM * cg);
  p.tiles_n = (a->C + bn - 1) / bn;
  p.batch1 = 1;
  p.nbatch = 1;
  p.a_mode = A_CONV;
  p.b_mode = B_DGRAD;
  p.P = a->H;
  p.Q = a->W;
  p.stride = 1;
  p.pad_h = a->R - 1 - a->pad_h;
  p.pad_w = a->S - 1 - a->pad_w;
  p.S = a->S;
  p.Rf = a->R;
  p.C = a->C;
  choose_split(p, a->split_k, a->out_mode == DP_OUT_ATOMIC_ADD);
  fill_epilogue(p, a->y, a->dtype == DP_BF16 && a->out_mode != DP_OUT_ATOMIC_ADD ? DP_BF16 : DP_F32,
                a->C, 0, 0, a->out_mode, nullptr, a->Res, a->C, 0, 0, a->alpha);
  if (query) {
    *query = splitk_bytes(p, cg, p.M, p.N);
    return 0;
  }
  CUtensorMap ma, mb;
  {
    const uint64_t d[4] = {(uint64_t)a->K, (uint64_t)a->Q, (uint64_t)a->P, (uint64_t)a->N};
    const int64_t s[3] = {a->K, (int64_t)a->Q * a->K, (int64_t)a->P * a->Q * a->K};
    const uint32_t box[4] = {64, (uint32_t)p.tw, (uint32_t)p.th, (uint32_t)p.tn};
    const uint32_t ones[4] = {1, 1, 1, 1};
    if (int e = make_map(&ma, a->x, d, s, box, ones)) return e;
  }
  {
    const uint64_t d[4] = {(uint64_t)a->C, (uint64_t)a->S, (uint64_t)a->R, (uint64_t)a->K};
    const int64_t s[3] = {a->C, (int64_t)a->S * a->C, (int64_t)a->R * a->S * a->C};
    const uint32_t box[4] = {64, 1, 1, BK};
    const uint32_t ones[4] = {1, 1, 1, 1};
    if (int e = make_map(&mb, a->w, d, s, box, ones)) return e;
  }
  return launch_bn(bn, cg, ma, mb, p, p.M, p.N, 1, 1, st, a->workspace, a->workspace_bytes);
}

// Swapped weight gradient: dW^T[(r,s,c)][k] = sum_pixels x_window[p][(r,s,c)] * dy[p][k], i.e. M = R*S*C
// (shifted input windows, MN-major A) and N = K (dy, MN-major B), so the long dimension takes the
// 256-row CTA-pair tiles and the output-channel count (a multiple of 128) the tile width; the fp32
// result is added into dW[k][(r,s,c)] by transposed TMA reduce boxes. The classic orientation
// (M = K) leaves K = 640 / 1280 layers on single CTAs or 17%-padded pairs.
static int conv_wgrad_swapped(const DpConvArgs* a, TcParams& p, cudaStream_t st) {
  const int Ntot = a->R * a->S * a->C;
  // 256-wide tiles also for K = 640 (three tiles, the last half empty): per-CTA L2->SM bytes per MMA
  // cycle drop by a third against 128-wide tiles, and the swapped weight gradient is bound by the TMA
  // feed, not by the tensor core (DP_WGRAD_BN128=1: 128-wide tiles, experiments)
  static const bool bn128 = getenv("DP_WGRAD_BN128") != nullptr;
  const int bn = (a->K % 256 == 0 || (!bn128 && a->K >= 512)) ? 256 : 128;
  const int cg = 2;
  p.M = Ntot;
  p.N = a->K;
  p.num_kb = (a->N * a->P * a->Q + BK - 1) / BK;
  p.tiles_m = (Ntot + BM * cg - 1) / (BM * cg);
  p.tiles_n = (a->K + bn - 1) / bn;
  p.batch1 = 1;
  p.nbatch = 1;
  p.a_mode = A_WG_X;
  p.b_mode = B_WG_DY;
  p.P = a->P;
  p.Q = a->Q;
  p.stride = a->stride;
  p.pad_h = a->pad_h;
  p.pad_w = a->pad_w;
  p.S = a->S;
  p.C = a->C;
  choose_split(p, a->split_k, true);
  fill_epilogue(p, a->y, DP_F32, Ntot, 0, 0, DP_OUT_ATOMIC_ADD, nullptr, nullptr, 0, 0, 0, a->alpha);
  CUtensorMap ma, mb, md;
  const uint32_t ones[4] = {1, 1, 1, 1};
  {  // x windows as the A operand (the B_WG_X map)
    const uint64_t d[4] = {(uint64_t)a->C, (uint64_t)a->W, (uint64_t)a->H, (uint64_t)a->N};
    const int64_t s[3] = {a->C, (int64_t)a->W * a->C, (int64_t)a->H * a->W * a->C};
    const uint32_t box[4] = {64, (uint32_t)(p.tw * a->stride), (uint32_t)(p.th * a->stride), (uint32_t)p.tn};
    const uint32_t es[4] = {1, (uint32_t)a->stride, (uint32_t)a->stride, 1};
    if (int e = make_map(&ma, a->x, d, s, box, es)) return e;
  }
  {  // dy [pixels][K] as the B operand
    const uint64_t d[4] = {(uint64_t)a->K, (uint64_t)a->Q, (uint64_t)a->P, (uint64_t)a->N};
    const int64_t s[3] = {a->K, (int64_t)a->Q * a->K, (int64_t)a->P * a->Q * a->K};
    const uint32_t box[4] = {64, (uint32_t)p.tw, (uint32_t)p.th, (uint32_t)p.tn};
    if (int e = make_map(&mb, a->w, d, s, box, ones)) return e;
  }
  {  // dW [K][R*S*C] fp32: (m = r,s,c contiguous, n = k) boxes of 32 m x 16 n
    const uint64_t d[4] = {(uint64_t)Ntot, (uint64_t)a->K, 1, 1};
    const int64_t s[3] = {Ntot, (int64_t)Ntot * a->K, (int64_t)Ntot * a->K};
    const uint32_t box[4] = {32, 16, 1, 1};
    if (int e = make_map(&md, a->y, d, s, box, ones, CU_TENSOR_MAP_SWIZZLE_NONE, 4)) return e;
    p.d_tma = 3;
  }
  return bn == 256 ? launch_tc<256, 2>(ma, mb, md, p, kNumSMs, st) : launch_tc<128, 2>(ma, mb, md, p, kNumSMs, st);
}

static bool wgrad_swap_enabled() {
  static const int v = [] {
    const char* e = getenv("DP_WGRAD_SWAP");  // experiments: 0 = classic orientation only
    return e ? atoi(e) : 1;
  }();
  return v != 0;
}

// dW[k][r][s][c] += sum_{n,p,q} dy[n][p][q][k] * x[n][p*stride+r-pad][q*stride+s-pad][c]
int tc_conv_wgrad(const DpConvArgs* a, cudaStream_t st) {
  if (a->C % 64 || a->K % 64) {
    set_error("implicit wgrad needs C % 64 == 0 and K % 64 == 0");
    return DP_ERR_UNSUPPORTED;
  }
  TcParams p{};
  if (!pixel_box(a->P, a->Q, BK, p.tw, p.th, p.tn)) {
    set_error("output spatial size does not tile into 64-pixel boxes");
    return DP_ERR_UNSUPPORTED;
  }
  const int Ntot = a->R * a->S * a->C;
  if (wgrad_swap_enabled() && a->K % 128 == 0 && Ntot >= 256 &&
      reinterpret_cast<uintptr_t>(a->y) % 16 == 0 && (Ntot * 4) % 16 == 0)
    return conv_wgrad_swapped(a, p, st);
  const int bn = pick_bn(Ntot, true);
  const int cg = decide_cg(a->K, bn, true, a->N * a->P * a->Q);
  p.M = a->K;
  p.N = Ntot;
  p.num_kb = (a->N * a->P * a->Q + BK - 1) / BK;
  p.tiles_m = (a->K + BM * cg - 1) / (BM * cg);
  p.tiles_n = (Ntot + bn - 1) / bn;
  p.batch1 = 1;
  p.nbatch = 1;
  p.a_mode = A_WG_DY;
  p.b_mode = B_WG_X;
  p.P = a->P;
  p.Q = a->Q;
  p.stride = a->stride;
  p.pad_h = a->pad_h;
  p.pad_w = a->pad_w;
  p.S = a->S;
  p.C = a->C;
  choose_split(p, a->split_k, true);
  fill_epilogue(p, a->y, DP_F32, Ntot, 0, 0, DP_OUT_ATOMIC_ADD, nullptr, nullptr, 0, 0, 0,
                a->alpha);
  CUtensorMap ma, mb;
  {  // dy as [K][pixels] MN-major, pixel tiles as 3-D boxes
    const uint64_t d[4] = {(uint64_t)a->K, (uint64_t)a->Q, (uint64_t)a->P, (uint64_t)a->N};
    const int64_t s[3] = {a->K, (int64_t)a->Q * a->K, (int64_t)a->P * a->Q * a->K};
    const uint32_t box[4] = {64, (uint32_t)p.tw, (uint32_t)p.th, (uint32_t)p.tn};
    const uint32_t ones[4] = {1, 1, 1, 1};
    if (int e = make_map(&ma, a->w, d, s, box, ones)) return e;
  }
  {
    const uint64_t d[4] = {(uint64_t)a->C, (uint64_t)a->W, (uint64_t)a->H, (uint64_t)a->N};
    const int64_t s[3] = {a->C, (int64_t)a->W * a->C, (int64_t)a->H * a->W * a->C};
    const uint32_t box[4] = {64, (uint32_t)(p.tw * a->stride), (uint32_t)(p.th * a->stride),
                             (uint32_t)p.tn};
    const uint32_t es[4] = {1, (uint32_t)a->stride, (uint32_t)a->stride, 1};
    if (int e = make_map(&mb, a->x, d, s, box, es)) return e;
  }
  return launch_bn(bn, cg, ma, mb, p, p.M, p.N, 1, 1, st);
}

// ====================================================================== fp32 / generic SIMT GEMM
// 64x64 output tile, 256 threads x (4x4) outputs, K staged 16 at a time through smem.
// Arbitrary strides on both operands (any major), batch, epilogue identical to the TC path.
template <typename TI>
__global__ void __launch_bounds__(256) simt_gemm_kernel(DpGemmArgs a) {
  DP_PDL_ENTRY();
  __shared__ float As[16][64 + 4];
  __shared__ float Bs[16][64 + 4];
  const int z = blockIdx.z;
  const int z1 = z % a.batch1, z2 = z / a.batch1;
  const TI* A = reinterpret_cast<const TI*>(a.A) + z1 * a.a_bs1 + z2 * a.a_bs2;
  const TI* B = reinterpret_cast<const TI*>(a.B) + z1 * a.b_bs1 + z2 * a.b_bs2;
  const int m0 = blockIdx.y * 64, n0 = blockIdx.x * 64;
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  float acc[4][4] = {};
  for (int k0 = 0; k0 < a.K; k0 += 16) {
    for (int i = threadIdx.x; i < 16 * 64; i += 256) {
      int kk, mm;
      if (a.a_mn_major) { mm = i % 64; kk = i / 64; } else { kk = i % 16; mm = i / 16; }
      const int m = m0 + mm, k = k0 + kk;
      float v = 0.f;
      if (m < a.M && k < a.K)
        v = to_f<TI>(a.a_mn_major ? A[(int64_t)k * a.a_ld + m] : A[(int64_t)m * a.a_ld + k]);
      As[kk][mm] = v;
    }
    for (int i = threadIdx.x; i < 16 * 64; i += 256) {
      int kk, nn;
      if (a.b_mn_major) { nn = i % 64; kk = i / 64; } else { kk = i % 16; nn = i / 16; }
      const int n = n0 + nn, k = k0 + kk;
      float v = 0.f;
      if (n < a.N && k < a.K)
        v = to_f<TI>(a.b_mn_major ? B[(int64_t)k * a.b_ld + n] : B[(int64_t)n * a.b_ld + k]);
      Bs[kk][nn] = v;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < 16; ++kk) {
      float av[4], bv[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) av[i] = As[kk][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) bv[j] = Bs[kk][tx * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int m = m0 + ty * 4 + i;
    if (m >= a.M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int n = n0 + tx * 4 + j;
      if (n >= a.N) continue;
      float v = acc[i][j] * a.alpha;
      if (a.bias) v += a.bias[n];
      if (a.Res) {
        const int64_t ro = z1 * a.r_bs1 + z2 * a.r_bs2 + (int64_t)m * a.r_ld + n;
        v += a.d_dtype == DP_F32 ? reinterpret_cast<const float*>(a.Res)[ro]
                                 : __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(a.Res)[ro]);
      }
      const int64_t o = z1 * a.d_bs1 + z2 * a.d_bs2 + (int64_t)m * a.d_ld + n;
      if (a.d_dtype == DP_F32) {
        float* d = reinterpret_cast<float*>(a.D) + o;
        if (a.out_mode == DP_OUT_ATOMIC_ADD) atomicAdd(d, v); else *d = v;
      } else {
        reinterpret_cast<__nv_bfloat16*>(a.D)[o] = __float2bfloat16_rn(v);
      }
    }
  }
}

int simt_gemm(const DpGemmArgs* in, cudaStream_t st) {
  DpGemmArgs a = *in;
  if (a.M <= 0 || a.N <= 0) return 0;
  if (a.batch1 <= 0) a.batch1 = 1;
  if (a.batch2 <= 0) a.batch2 = 1;
  dim3 grid((a.N + 63) / 64, (a.M + 63) / 64, a.batch1 * a.batch2);
  if (a.dtype == DP_F32)
    launch_k(simt_gemm_kernel<float>, dim3(grid), dim3(256), 0, st, a);
  else
    launch_k(simt_gemm_kernel<__nv_bfloat16>, dim3(grid), dim3(256), 0, st, a);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) set_error(std::string("simt_gemm: ") + cudaGetErrorString(e));
  return e;
}

}  // namespace dp

extern "C" {

int dp_gemm(const DpGemmArgs* a, dp_stream_t stream) {
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (a->dtype == DP_BF16) {
    // TMA needs 16-byte aligned strides; otherwise use the generic kernel.
    const bool ok = (a->a_ld % 8 == 0) && (a->b_ld % 8 == 0) && (a->a_bs1 % 8 == 0) &&
                    (a->a_bs2 % 8 == 0) && (a->b_bs1 % 8 == 0) && (a->b_bs2 % 8 == 0) &&
                    (reinterpret_cast<uintptr_t>(a->A) % 16 == 0) &&
                    (reinterpret_cast<uintptr_t>(a->B) % 16 == 0) &&
                    ((a->batch1 <= 1 || a->a_bs1 != 0) && (a->batch1 <= 1 || a->b_bs1 != 0)) &&
                    ((a->batch2 <= 1 || a->a_bs2 != 0) && (a->batch2 <= 1 || a->b_bs2 != 0));
    if (ok) return dp::tc_gemm(a, st);
  }
  if (a->geglu_mode) {
    dp::set_error("dp_gemm: the GEGLU epilogue needs the bf16 tensor-core path (16-byte aligned operands)");
    return DP_ERR_UNSUPPORTED;
  }
  return dp::simt_gemm(a, st);
}

int dp_conv_fwd(const DpConvArgs* a, dp_stream_t stream) {
  if (a->dtype != DP_BF16) {
    dp::set_error("dp_conv_fwd is the bf16 tensor-core path; lower fp32 convs via dp_im2col");
    return DP_ERR_UNSUPPORTED;
  }
  return dp::tc_conv_fwd(a, reinterpret_cast<cudaStream_t>(stream));
}

int dp_conv_dgrad(const DpConvArgs* a, dp_stream_t stream) {
  if (a->dtype != DP_BF16) {
    dp::set_error("dp_conv_dgrad is the bf16 tensor-core path");
    return DP_ERR_UNSUPPORTED;
  }
  return dp::tc_conv_dgrad(a, reinterpret_cast<cudaStream_t>(stream));
}

int dp_conv_wgrad(const DpConvArgs* a, dp_stream_t stream) {
  if (a->dtype != DP_BF16) {
    dp::set_error("dp_conv_wgrad is the bf16 tensor-core path");
    return DP_ERR_UNSUPPORTED;
  }
  return dp::tc_conv_wgrad(a, reinterpret_cast<cudaStream_t>(stream));
}

int64_t dp_gemm_workspace(const DpGemmArgs* a) {
  int64_t q = 0;
  if (a->dtype != DP_BF16) return 0;
  dp::tc_gemm(a, nullptr, &q);
  return q;
}

int64_t dp_conv_fwd_workspace(const DpConvArgs* a) {
  int64_t q = 0;
  if (a->dtype == DP_BF16) dp::tc_conv_fwd(a, nullptr, &q);
  return q;
}

int64_t dp_conv_dgrad_workspace(const DpConvArgs* a) {
  int64_t q = 0;
  if (a->dtype == DP_BF16) dp::tc_conv_dgrad(a, nullptr, &q);
  return q;
}

const char* dp_last_error(void) { return dp::g_last_error.c_str(); }
int dp_version(void) { return 2; }

}  // extern "C"
