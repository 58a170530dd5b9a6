// gemm.cu -- persistent warp-specialised tcgen05 GEMM with fused epilogues,
// 2-SM (CTA pair) version.
//
// C[M][N] = A[M][K] * B[N][K]^T (+ LoRA K-extension), bf16 in, fp32 in TMEM.
// A cluster of 2 CTAs (one SM pair) owns a 256 x 256 output tile: CTA r loads
// A rows [m0 + 128 r, +128) and B rows [n0 + 128 r, +128) (half of N) and
// keeps accumulator rows [128 r, +128) in its TMEM; the leader issues
// tcgen05.mma.cta_group::2 (M = 256, N = 256, K = 16), which reads both CTAs'
// shared memory -- each SM streams half the B operand.
// Roles (384 threads per CTA, 1 CTA per SM):
//   warps 0-7   epilogue: warp w reads TMEM lanes 32 (w % 4).. and column half
//               w / 4 of a double-buffered accumulator, then the fused
//               epilogue of the step row: bias, QK-RMSNorm + RoPE + head-major
//               scatter, GELU, gated residual (+ControlNet), Euler, LoRA shrink.
//   warp 8      TMA producer (both CTAs): 6-stage ring of A 128x64 + B 128x64
//               (SWIZZLE_128B); complete_tx lands on the LEADER's full barrier.
//   warp 9      MMA issuer (leader only, one thread) + TMEM allocator; tcgen05.commit multicast
//               releases the stage / publishes the accumulator in both CTAs.
//   (The producer / MMA warps take the HIGHEST warp ids: the SMSP arbiter
//   issues highest-id-first, so the single MMA thread never waits behind the
//   epilogue warps that share its SMSP.)
// Tiles are scheduled statically per cluster over up to two problems (the
// img and txt streams of a double block share one launch), rasterised in
// groups of 16 M-tiles so the A rows stay L2-resident while N is swept.
#include <cstdio>
#include <cstdlib>
#include <algorithm>

#include "common.cuh"
#include "kernels.h"

namespace dit {

constexpr int STAGES = 6;
constexpr int A_BYTES = GEMM_BM * GEMM_BK * 2;           // 128 rows x 64 per CTA
constexpr int B_BYTES = (GEMM_BN / 2) * GEMM_BK * 2;     // 128 rows x 64 per CTA (half of N)
constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
constexpr int TMEM_COLS = 512;
constexpr int NUM_THREADS = 320;
constexpr int W_LOAD = 8, W_MMA = 9;
#ifndef GEMM_RESID_TMA
#define GEMM_RESID_TMA 1
#endif
// gated residual via TMA reduce-add: per epilogue warp a 32 x 32 fp32 staging box (4 KB, 1024-B
// aligned for SWIZZLE_128B) after a 1 KB barrier area
constexpr int EPI_BOX_OFF = STAGES * STAGE_BYTES + 1024;
constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 /*align*/ + (GEMM_RESID_TMA ? 1024 + 8 * 4096 : 256);
size_t gemm_smem_bytes() { return SMEM_BYTES; }

struct TileInfo {
  int p, m, n, slot, nk_base, nk_total;
};

DEVI TileInfo decode_tile(const GemmArgs& A, int t) {
  TileInfo ti;
  ti.p = (A.num_problems > 1 && t >= A.p[1].tile_begin) ? 1 : 0;
  const GemmProblem& P = A.p[ti.p];
  int local = t - P.tile_begin;
  ti.slot = -1;
  if (P.shrink) {
    int2 e = P.shrink_list[local];
    ti.m = e.x;
    ti.slot = e.y;
    ti.n = 0;
  } else {
    int per_group = P.group_m * P.tiles_n;   // tiles_m counts 256-row pair tiles
    int g = local / per_group;
    int first_m = g * P.group_m;
    int gm = min(P.group_m, P.tiles_m - first_m);
    int within = local - g * per_group;
    ti.m = first_m + within % gm;
    ti.n = within / gm;
  }
  ti.nk_base = (P.K + GEMM_BK - 1) / GEMM_BK;
  ti.nk_total = ti.nk_base;
  if (P.ext_kblocks > 0 && !P.shrink) ti.nk_total += P.tile_slot_cnt[ti.m] * P.ext_kblocks;
  return ti;
}

// GELU (tanh form) with the MUFU tanh (rel. error ~2^-11, below the bf16 rounding
// of the stored activation).
DEVI float gelu_tanh_f(float x) {
  const float k0 = 0.7978845608028654f, k1 = 0.044715f;
  const float u = k0 * (x + k1 * x * x * x);
  float t;
  asm("tanh.approx.f32 %0, %1;" : "=f"(t) : "f"(u));
  return 0.5f * x * (1.0f + t);
}

DEVI void load_bias32(const bf16* bias, int col, int N, float (&bv)[32]) {
  if (col + 32 <= N) {
    const uint4* p = reinterpret_cast<const uint4*>(bias + col);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      uint4 u = __ldg(p + q);
      uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        bv[q * 8 + 2 * e] = bf16_lo(w[e]);
        bv[q * 8 + 2 * e + 1] = bf16_hi(w[e]);
      }
    }
  } else {
#pragma unroll
    for (int j = 0; j < 32; ++j) bv[j] = (col + j < N) ? __bfloat162float(bias[col + j]) : 0.f;
  }
}

DEVI void store_bf16_32(bf16* dst, const float (&x)[32], int valid) {
  if (valid >= 32 && (reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
    uint4* p = reinterpret_cast<uint4*>(dst);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      uint4 u;
      u.x = pack_bf16(x[q * 8 + 0], x[q * 8 + 1]);
      u.y = pack_bf16(x[q * 8 + 2], x[q * 8 + 3]);
      u.z = pack_bf16(x[q * 8 + 4], x[q * 8 + 5]);
      u.w = pack_bf16(x[q * 8 + 6], x[q * 8 + 7]);
      p[q] = u;
    }
  } else {
#pragma unroll
    for (int j = 0; j < 32; ++j)
      if (j < valid) dst[j] = __float2bfloat16_rn(x[j]);
  }
}

// Block until a ControlNet producer (another stream or another GPU writing into this GPU's
// memory) has published its residual: *flag >= expect, system-scope acquire.  Bounded spin:
// a producer that never publishes traps instead of hanging the GPU.
DEVI void cn_acquire(const uint32_t* flag, uint32_t expect) {
  if (flag == nullptr) return;
  uint32_t v, spins = 0;
  while (true) {
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(flag) : "memory");
    if (v >= expect) break;
    __nanosleep(256);
    if (++spins > (1u << 24)) __trap();
  }
}

// h4[0..7] (32 fp32) += kap * R[0..31] (bf16).  L2-coherent loads (ld.cg): the residual may
// have been written by a producer after this kernel started.
DEVI void cn_add8(float4 (&h4)[8], const bf16* cn, float kap) {
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const uint2 c2 = __ldcg(reinterpret_cast<const uint2*>(cn) + q);
    h4[q].x = fmaf(kap, bf16_lo(c2.x), h4[q].x);
    h4[q].y = fmaf(kap, bf16_hi(c2.x), h4[q].y);
    h4[q].z = fmaf(kap, bf16_lo(c2.y), h4[q].z);
    h4[q].w = fmaf(kap, bf16_hi(c2.y), h4[q].w);
  }
}

// d = 128 QKV epilogue helpers: 64 accumulator columns + bias -> y (fp32)
DEVI void load_head_half(uint32_t taddr, const bf16* bias, float (&y)[64]) {
  tmem_ld32(taddr, *reinterpret_cast<uint32_t(*)[32]>(&y[0]));
  tmem_ld32(taddr + 32, *reinterpret_cast<uint32_t(*)[32]>(&y[32]));
  tmem_ld_wait();
#pragma unroll
  for (int j = 0; j < 64; j += 8) {
    const uint4 u = __ldg(reinterpret_cast<const uint4*>(bias + j));
    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      y[j + 2 * e] += bf16_lo(w[e]);
      y[j + 2 * e + 1] += bf16_hi(w[e]);
    }
  }
}
// RMSNorm scale (rs * gamma) then RoPE on interleaved pairs; cs = (cos, sin) pairs of these columns
DEVI void norm_rope_half(float (&y)[64], float rs, const bf16* g, const float4* cs) {
#pragma unroll
  for (int j = 0; j < 64; j += 8) {
    const uint4 gu = __ldg(reinterpret_cast<const uint4*>(g + j));
    const uint32_t gw[4] = {gu.x, gu.y, gu.z, gu.w};
    const float4 c01 = __ldg(cs + j / 4), c23 = __ldg(cs + j / 4 + 1);
    const float cr[4][2] = {{c01.x, c01.y}, {c01.z, c01.w}, {c23.x, c23.y}, {c23.z, c23.w}};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float x0 = y[j + 2 * e] * rs * bf16_lo(gw[e]);
      const float x1 = y[j + 2 * e + 1] * rs * bf16_hi(gw[e]);
      y[j + 2 * e] = cr[e][0] * x0 - cr[e][1] * x1;
      y[j + 2 * e + 1] = cr[e][1] * x0 + cr[e][0] * x1;
    }
  }
}

// Epilogue for one accumulator tile.  Thread = one accumulator row; this warp
// covers columns [c_lo, c_lo + 128) of the 256-wide tile.
#ifndef GEMM_EPI_FAKE
#define GEMM_EPI_FAKE 0
#endif
DEVI void epilogue_tile(const GemmProblem& P, const TileInfo& ti, uint32_t tbase, int row_in_tile, int c_lo,
                        float4* box) {
  const EpiParams& E = P.epi;
  const int r = ti.m * GEMM_TM + row_in_tile;
  const bool row_ok = r < P.M;
  const int n0 = ti.n * GEMM_BN;
  const int b = row_ok ? r / E.rows_per_req : 0;
  const int nloc = row_ok ? r - b * E.rows_per_req : 0;
  const int jrow = b * E.joint_n + E.joint_off + nloc;
  const bf16* bias = reinterpret_cast<const bf16*>(E.bias);
  const int c_hi = c_lo + GEMM_BN / 2;
#if GEMM_EPI_FAKE
  {  // timing experiment: accumulator read only, no epilogue math or global traffic
    uint32_t acc = 0;
    for (int c0 = c_lo; c0 < c_hi; c0 += 32) {
      uint32_t rr[32];
      tmem_ld32(tbase + c0, rr);
      tmem_ld_wait();
      acc += rr[0];
    }
    if (acc == 0x7f7f7f7fu && r == -5) P.epi.h[0] = 0.f;
    return;
  }
#endif

  if (E.kind == EPI_QKV) {
    const int d = E.head_dim;
    const int D = E.D;
#pragma unroll 1
    for (int c0 = c_lo; c0 < c_hi; c0 += d) {
      const int col0 = n0 + c0;
      if (col0 >= P.N) break;
      if (col0 < E.qkv_cols) {
        const int sec = col0 / D;
        const int head = (col0 - sec * D) / d;
        const int hl_n = E.heads / E.sp_world;
        const int dest = head / hl_n, hl = head - dest * hl_n;
        bf16* dst =
            E.qkv_peer[0] != nullptr
                ? reinterpret_cast<bf16*>(E.qkv_peer[dest]) +   // fused exchange: the owner's attention buffer
                      (size_t)sp_attn_vec(E.batch, hl_n, E.sp_world * E.seq_len, sec, b, hl,
                                          sp_global_row(E.sp_world, E.sp_nt, E.sp_ni, E.sp_rank, E.joint_off + nloc)) * d
                : reinterpret_cast<bf16*>(E.qkv) +
                      (size_t)sp_qkv_send_vec(E.batch, hl_n, E.seq_len, dest, sec, b, hl, E.joint_off + nloc) * d;
        const bool nrm = sec < 2 && E.q_gamma != nullptr;   // SD3-medium: no QK-norm (RoPE table = identity)
        if (d == 128) {
          // head in two 64-column halves: half 0 read for the RMS statistic, half 1 read and
          // kept, processed, then half 0 re-read and processed (3 TMEM reads instead of 8)
          float ss = 0.f;
          if (nrm) {
            float y[64];
            load_head_half(tbase + c0, bias + col0, y);
#pragma unroll
            for (int e = 0; e < 64; ++e) ss = fmaf(y[e], y[e], ss);
          }
          float y[64];
          load_head_half(tbase + c0 + 64, bias + col0 + 64, y);   // (tcgen05.ld: all lanes)
          float rs = 1.f;
          if (nrm) {
#pragma unroll
            for (int e = 0; e < 64; ++e) ss = fmaf(y[e], y[e], ss);
            rs = rsqrtf(ss / (float)d + 1e-6f);
          }
          const bf16* g = reinterpret_cast<const bf16*>(sec == 0 ? E.q_gamma : E.k_gamma);
          const float4* cs = reinterpret_cast<const float4*>(E.rope + (size_t)b * E.rope_stride +
                                                             (size_t)(E.joint_off + nloc) * (d / 2));
          if (nrm) norm_rope_half(y, rs, g + 64, cs + 16);
          if (row_ok) {
#pragma unroll
            for (int j = 0; j < 64; j += 32) store_bf16_32(dst + 64 + j, *reinterpret_cast<const float(*)[32]>(&y[j]), 32);
          }
          load_head_half(tbase + c0, bias + col0, y);
          if (nrm) norm_rope_half(y, rs, g, cs);
          if (row_ok) {
#pragma unroll
            for (int j = 0; j < 64; j += 32) store_bf16_32(dst + j, *reinterpret_cast<const float(*)[32]>(&y[j]), 32);
          }
          continue;
        }
        if (d == 64) {
          // SD3 / SD3.5 heads: the whole head in one pair of TMEM reads, the RMS statistic and the
          // normalise(+RoPE) pass from registers (2 TMEM reads per head instead of 4)
          float y[64];
          load_head_half(tbase + c0, bias + col0, y);   // (tcgen05.ld: all lanes)
          if (nrm) {
            float ss = 0.f;
#pragma unroll
            for (int e = 0; e < 64; ++e) ss = fmaf(y[e], y[e], ss);
            const bf16* g = reinterpret_cast<const bf16*>(sec == 0 ? E.q_gamma : E.k_gamma);
            const float4* cs = reinterpret_cast<const float4*>(E.rope + (size_t)b * E.rope_stride +
                                                               (size_t)(E.joint_off + nloc) * (d / 2));
            norm_rope_half(y, rsqrtf(ss / 64.f + 1e-6f), g, cs);
          }
          if (row_ok) {
#pragma unroll
            for (int j = 0; j < 64; j += 32) store_bf16_32(dst + j, *reinterpret_cast<const float(*)[32]>(&y[j]), 32);
          }
          continue;
        }
        // generic head size (d = 32 test configurations): two passes of 32 columns
        // pass 1: sum of squares over the head (q, k only)
        float rs = 1.f;
        if (nrm) {
          float ss = 0.f;
#pragma unroll 1
          for (int j = 0; j < d; j += 32) {
            uint32_t rr[32];
            tmem_ld32(tbase + c0 + j, rr);
            tmem_ld_wait();
            float bv[32];
            load_bias32(bias, col0 + j, P.N, bv);
#pragma unroll
            for (int e = 0; e < 32; ++e) {
              const float x = __uint_as_float(rr[e]) + bv[e];
              ss += x * x;
            }
          }
          rs = rsqrtf(ss / (float)d + 1e-6f);
        }
        const bf16* g = reinterpret_cast<const bf16*>(sec == 0 ? E.q_gamma : E.k_gamma);
        const float2* cs = E.rope + (size_t)b * E.rope_stride + (size_t)(E.joint_off + nloc) * (d / 2);
        // pass 2: normalise, rotate interleaved pairs, store
#pragma unroll 1
        for (int j = 0; j < d; j += 32) {
          uint32_t rr[32];
          tmem_ld32(tbase + c0 + j, rr);
          tmem_ld_wait();
          float bv[32], y[32];
          load_bias32(bias, col0 + j, P.N, bv);
#pragma unroll
          for (int e = 0; e < 32; ++e) y[e] = __uint_as_float(rr[e]) + bv[e];
          if (nrm && row_ok) {
#pragma unroll
            for (int e = 0; e < 16; ++e) {
              const float x0 = y[2 * e] * rs * __bfloat162float(g[j + 2 * e]);
              const float x1 = y[2 * e + 1] * rs * __bfloat162float(g[j + 2 * e + 1]);
              const float2 c = __ldg(cs + j / 2 + e);
              y[2 * e] = c.x * x0 - c.y * x1;
              y[2 * e + 1] = c.y * x0 + c.x * x1;
            }
          }
          if (row_ok) store_bf16_32(dst + j, y, 32);
        }
      } else {
        // GELU branch of the single-block linear1 (cols >= 3D)
#pragma unroll 1
        for (int j = 0; j < d; j += 32) {
          const int col = col0 + j;
          uint32_t rr[32];
          tmem_ld32(tbase + c0 + j, rr);
          tmem_ld_wait();
          if (col >= P.N || !row_ok) continue;
          float bv[32], y[32];
          load_bias32(bias, col, P.N, bv);
#pragma unroll
          for (int e = 0; e < 32; ++e) y[e] = gelu_tanh_f(__uint_as_float(rr[e]) + bv[e]);
          bf16* dst = reinterpret_cast<bf16*>(E.out) + (size_t)r * E.ld_out + E.out_col0 + (col - E.qkv_cols);
          store_bf16_32(dst, y, min(32, P.N - col));
        }
      }
    }
    // fused exchange: this thread's peer stores reach system scope before the kernel ends
    // (the barrier kernel's release then covers them on the peer)
    if (E.qkv_peer[0] != nullptr) __threadfence_system();
    return;
  }

  if (E.kind == EPI_SHRINK) {
    const int rs = row_ok ? E.row_slot[r] : -2;
    const float sc = E.slot_scale[ti.slot];
#pragma unroll 1
    for (int c0 = c_lo; c0 < min(c_hi, E.r_alloc); c0 += 32) {
      uint32_t rr[32];
      tmem_ld32(tbase + c0, rr);
      tmem_ld_wait();
      if (!row_ok) continue;
      float y[32];
#pragma unroll
      for (int e = 0; e < 32; ++e) y[e] = (rs == ti.slot) ? sc * __uint_as_float(rr[e]) : 0.f;
      bf16* dst = reinterpret_cast<bf16*>(E.out) + (size_t)r * E.ld_out + ti.slot * E.r_alloc + c0;
      store_bf16_32(dst, y, 32);
    }
    return;
  }

#if GEMM_RESID_TMA
  // the warp's 32 rows: one contiguous block of h rows (same request, all < M) -> TMA reduce-add
  const int lw = row_in_tile & 31;
  const int rw0 = r - lw;
  const bool boxed = E.kind == EPI_RESID && P.tmH_ok && rw0 + 31 < P.M &&
                     rw0 / E.rows_per_req == (rw0 + 31) / E.rows_per_req;
  const int jrow0 = boxed ? (rw0 / E.rows_per_req) * E.joint_n + E.joint_off + rw0 % E.rows_per_req : 0;
#else
  constexpr bool boxed = false;
  constexpr int lw = 0, jrow0 = 0;
#endif
#pragma unroll 1
  for (int c2 = c_lo; c2 < c_hi; c2 += 64) {
    if (n0 + c2 >= P.N) break;
    // two 32-column accumulator reads in flight per wait
    uint32_t rr2[64];
    tmem_ld32(tbase + c2, *reinterpret_cast<uint32_t(*)[32]>(&rr2[0]));
    tmem_ld32(tbase + c2 + 32, *reinterpret_cast<uint32_t(*)[32]>(&rr2[32]));
    tmem_ld_wait();
#pragma unroll
  for (int hh = 0; hh < 2; ++hh) {
    const int c0 = c2 + hh * 32;
    const int col = n0 + c0;
    if (col >= P.N) break;
    const int valid = min(32, P.N - col);
    const bool tma_chunk = boxed && valid == 32;   // warp-uniform
    if (!row_ok && !tma_chunk) continue;
    float bv[32], y[32];
    load_bias32(bias, col, P.N, bv);
#pragma unroll
    for (int e = 0; e < 32; ++e) y[e] = __uint_as_float(rr2[hh * 32 + e]) + bv[e];
    if (E.kind == EPI_GELU || E.kind == EPI_BIAS) {
      if (E.kind == EPI_GELU) {
#pragma unroll
        for (int e = 0; e < 32; ++e) y[e] = gelu_tanh_f(y[e]);
      }
      store_bf16_32(reinterpret_cast<bf16*>(E.out) + (size_t)r * E.ld_out + E.out_col0 + col, y, valid);
    } else if (E.kind == EPI_STORE_H) {
      float* hp = E.h + (size_t)jrow * E.D + col;
      if (valid == 32) {
#pragma unroll
        for (int q = 0; q < 8; ++q)
          reinterpret_cast<float4*>(hp)[q] = make_float4(y[4 * q], y[4 * q + 1], y[4 * q + 2], y[4 * q + 3]);
      } else {
#pragma unroll
        for (int e = 0; e < 32; ++e)
          if (e < valid) hp[e] = y[e];
      }
    } else if (E.kind == EPI_RESID) {
      float* hp = E.h + (size_t)jrow * E.D + col;
      const float* gp = E.mod + (size_t)b * E.mod_stride + E.gate_off + col;
      // ControlNet fan-in: up to CN_FANIN residuals per (request, block), rows from cn_row0
      const bf16* cn0 = nullptr;
      const bf16* cn1 = nullptr;
      float kap0 = 0.f, kap1 = 0.f;
      if (E.cn_ptr != nullptr && nloc >= E.cn_row0 &&
          (E.img_valid == nullptr || nloc - E.cn_row0 < E.img_valid[b])) {   // (ragged: residual has Ni_b rows)
        const size_t roff = (size_t)(nloc - E.cn_row0) * E.D + col;
        cn0 = reinterpret_cast<const bf16*>(E.cn_ptr[b]);
        cn1 = reinterpret_cast<const bf16*>(E.cn_ptr[MAX_SEQ + b]);
        if (cn0 != nullptr) { kap0 = E.cn_scale[b]; cn0 += roff; }
        if (cn1 != nullptr) { kap1 = E.cn_scale[MAX_SEQ + b]; cn1 += roff; }
        if (E.cn_flag != nullptr) {   // deferred fetch with device flags
          cn_acquire(E.cn_flag[b], E.cn_expect[b]);
          cn_acquire(E.cn_flag[MAX_SEQ + b], E.cn_expect[MAX_SEQ + b]);
        }
      }
      // h += v with v = g (acc + bias) (+ kappa R per ControlNet), v rounded once and added to h
      // with a single rounding on EVERY path (TMA reduce-add, vector and scalar fallbacks), so a
      // row's result does not depend on which path its warp takes (batch / shard invariance)
      if (valid == 32) {
        float4 v4[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const float4 g4 = __ldg(reinterpret_cast<const float4*>(gp) + q);
          v4[q] = make_float4(__fmul_rn(g4.x, y[4 * q]), __fmul_rn(g4.y, y[4 * q + 1]), __fmul_rn(g4.z, y[4 * q + 2]),
                              __fmul_rn(g4.w, y[4 * q + 3]));
        }
        if (cn0 != nullptr) cn_add8(v4, cn0, kap0);
        if (cn1 != nullptr) cn_add8(v4, cn1, kap1);
        if (tma_chunk) {
          // the warp's swizzled 32 x 32 box, then ONE TMA reduce-add h[jrow0 .. +32)[col .. +32) += box:
          // the SM never loads h
#if GEMM_RESID_TMA
#pragma unroll
          for (int q = 0; q < 8; ++q) box[lw * 8 + (q ^ (lw & 7))] = v4[q];
          __syncwarp();
          fence_async_shared();
          if (lw == 0) {
            asm volatile("cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                             reinterpret_cast<uint64_t>(&P.tmH)),
                         "r"(smem_u32(box)), "r"(col), "r"(jrow0)
                         : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");   // box reusable
          }
          __syncwarp();
#endif
        } else {
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            float4 h4 = reinterpret_cast<float4*>(hp)[q];
            h4.x = __fadd_rn(h4.x, v4[q].x);
            h4.y = __fadd_rn(h4.y, v4[q].y);
            h4.z = __fadd_rn(h4.z, v4[q].z);
            h4.w = __fadd_rn(h4.w, v4[q].w);
            reinterpret_cast<float4*>(hp)[q] = h4;
          }
        }
      } else {
#pragma unroll
        for (int e = 0; e < 32; ++e) {   // static indices keep y in registers
          if (e < valid) {
            float v = __fmul_rn(gp[e], y[e]);
            if (cn0 != nullptr) v = fmaf(kap0, __bfloat162float(__ldcg(cn0 + e)), v);
            if (cn1 != nullptr) v = fmaf(kap1, __bfloat162float(__ldcg(cn1 + e)), v);
            hp[e] = __fadd_rn(hp[e], v);
          }
        }
      }
    } else if (E.kind == EPI_FINAL) {
      const float ds = E.dsig[b];
#pragma unroll
      for (int e = 0; e < 32; ++e) {
        if (e < valid) {
          const size_t off = (size_t)r * P.N + col + e;
          if (E.lat_out != nullptr) E.lat_out[off] = E.lat_in[off] + ds * y[e];   // (CFG: Euler after the combine)
          if (E.v_out != nullptr) E.v_out[off] = y[e];
          if (E.v_peer != nullptr) E.v_peer[off] = y[e];   // latent parallelism: the fused all-gather
        }
      }
      if (E.v_peer != nullptr) __threadfence_system();   // before the barrier kernel's release
    }
  }
  }
}

// While the MMAs of a tile run, pull the rows the residual epilogue will read-modify-write
// (h fp32, 512 B per thread) and the ControlNet residual into L2, so the epilogue's global
// loads hit L2 instead of HBM.
DEVI void prefetch_epilogue_rows(const GemmProblem& P, const TileInfo& ti, int row_in_tile, int c_lo) {
  const EpiParams& E = P.epi;
  if (E.kind != EPI_RESID) return;
  const int r = ti.m * GEMM_TM + row_in_tile;
  const int col = ti.n * GEMM_BN + c_lo;
  if (r >= P.M || col >= P.N) return;
  const int b = r / E.rows_per_req;
  const int nloc = r - b * E.rows_per_req;
  const int jrow = b * E.joint_n + E.joint_off + nloc;
  const float* hp = E.h + (size_t)jrow * E.D + col;
#pragma unroll
  for (int q = 0; q < 4; ++q) asm volatile("prefetch.global.L2 [%0];" ::"l"(hp + q * 32));
  if (E.cn_ptr != nullptr && nloc >= E.cn_row0 && (E.img_valid == nullptr || nloc - E.cn_row0 < E.img_valid[b])) {
#pragma unroll
    for (int k = 0; k < CN_FANIN; ++k) {
      const bf16* cn = reinterpret_cast<const bf16*>(E.cn_ptr[MAX_SEQ * k + b]);
      if (cn != nullptr) {
        cn += (size_t)(nloc - E.cn_row0) * E.D + col;
        asm volatile("prefetch.global.L2 [%0];" ::"l"(cn));
        asm volatile("prefetch.global.L2 [%0];" ::"l"(cn + 64));
      }
    }
  }
}

#ifndef GEMM_TRACE
#define GEMM_TRACE 0
#endif
#if GEMM_TRACE
// timing experiment (variant builds only, tools/gemm_trace.py): clock64 stamps of CTA 0 per
// tile -- 0 epilogue start, 1 / 2 epilogue end (warp 0 / 7), 3 / 4 MMA warp before / after the
// accumulator-free wait, 5 last MMA of the tile issued
__device__ long long* g_gemm_trace = nullptr;
extern "C" int dit_debug_gemm_trace(long long* buf) {
  return cudaMemcpyToSymbol(g_gemm_trace, &buf, sizeof(buf)) == cudaSuccess ? 0 : 1;
}
#define GTRACE(ev, it)                                                                            \
  do {                                                                                            \
    if (blockIdx.x == 0 && g_gemm_trace != nullptr && (it) < 64) g_gemm_trace[(ev) * 64 + (it)] = clock64(); \
  } while (0)
#else
#define GTRACE(ev, it) do {} while (0)
#endif

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(NUM_THREADS, 1)
    gemm_kernel(const __grid_constant__ GemmArgs args) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * A_BYTES;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  uint64_t* full = bars;
  uint64_t* empty = bars + STAGES;
  uint64_t* tfull = bars + 2 * STAGES;
  uint64_t* tempty = bars + 2 * STAGES + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * STAGES + 4);

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const uint32_t cta = cluster_rank();
  const bool leader = cta == 0;
  const int cid = blockIdx.x >> 1, ncl = gridDim.x >> 1;

  if (warp == W_LOAD && lane == 0) {
    for (int p = 0; p < args.num_problems; ++p) {
      tma_prefetch_desc(&args.p[p].tmA);
      tma_prefetch_desc(&args.p[p].tmB);
      if (args.p[p].ext_kblocks > 0) {
        tma_prefetch_desc(&args.p[p].tmAx);
        tma_prefetch_desc(&args.p[p].tmBx);
      }
    }
  }
  if (warp == W_MMA && lane == 0) {
    for (int i = 0; i < STAGES; ++i) {
      mbar_init(&full[i], 2);      // leader: own expect_tx arrival + the peer producer's remote arrival
      mbar_init(&empty[i], 1);     // one multicast commit per phase
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 16);   // 8 epilogue warps x 2 CTAs (leader's copy)
    }
    fence_barrier_init();
  }
  if (warp == W_MMA) tmem_alloc_2sm<TMEM_COLS>(tmem_slot);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == W_LOAD) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int t = cid; t < args.total_tiles; t += ncl) {
        const TileInfo ti = decode_tile(args, t);
        const GemmProblem& P = args.p[ti.p];
        const int a_row = ti.m * GEMM_TM + (int)cta * GEMM_BM;
        for (int kb = 0; kb < ti.nk_total; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          if (leader)
            mbar_expect_tx(&full[stage], 2 * STAGE_BYTES);
          else
            mbar_arrive_cta(&full[stage], 0);
          uint8_t* a_dst = sA + stage * A_BYTES;
          uint8_t* b_dst = sB + stage * B_BYTES;
          if (kb < ti.nk_base) {
            tma_load_2d_2sm(&P.tmA, &full[stage], a_dst, kb * GEMM_BK, a_row);
            if (P.shrink)
              tma_load_2d_2sm(&P.tmB, &full[stage], b_dst, kb * GEMM_BK,
                              ti.slot * P.epi.r_alloc + (int)cta * (P.epi.r_alloc / 2));
            else
              tma_load_2d_2sm(&P.tmB, &full[stage], b_dst, kb * GEMM_BK, ti.n * GEMM_BN + (int)cta * 128);
          } else {
            const int e = kb - ti.nk_base;
            const int si = e / P.ext_kblocks;
            const int ek = e - si * P.ext_kblocks;
            const int slot = P.tile_slots[ti.m * P.slot_cap + si];
            tma_load_2d_2sm(&P.tmAx, &full[stage], a_dst, slot * P.epi.r_alloc + ek * GEMM_BK, a_row);
            tma_load_2d_2sm(&P.tmBx, &full[stage], b_dst, ek * GEMM_BK, slot * P.N + ti.n * GEMM_BN + (int)cta * 128);
          }
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == W_MMA) {
    // whole warp walks the tile loop; one elected lane issues inside the asm blocks, so the
    // descriptors stay warp-uniform (a lane-0 branch costs R2UR/elect loops per MMA)
    if (leader) {
      constexpr uint32_t idesc_full = idesc_bf16_f32(2 * GEMM_BM, GEMM_BN);

      int stage = 0;
      uint32_t phase = 0;
      int iter = 0;
      for (int t = cid; t < args.total_tiles; t += ncl, ++iter) {
        const TileInfo ti = decode_tile(args, t);
        // LoRA-shrink tiles only need N = r_alloc (64 or 128) columns
        const uint32_t idesc = __shfl_sync(0xffffffffu,
            args.p[ti.p].shrink ? idesc_bf16_f32(2 * GEMM_BM, args.p[ti.p].epi.r_alloc) : idesc_full, 0);
        const int nk_total = __shfl_sync(0xffffffffu, ti.nk_total, 0);
        const int acc = iter & 1;
        const uint32_t acc_phase = (iter >> 1) & 1;
        if (lane == 0) GTRACE(3, iter);
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        if (lane == 0) GTRACE(4, iter);
        tc_fence_after();
        const uint32_t d_tmem = __shfl_sync(0xffffffffu, tmem_base, 0) + acc * GEMM_BN;
        for (int kb = 0; kb < nk_total; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t a_addr = smem_u32(sA + stage * A_BYTES);
          const uint32_t b_addr = smem_u32(sB + stage * B_BYTES);
          mma_2sm_k64_warp(d_tmem, smem_desc_k_sw128(a_addr), smem_desc_k_sw128(b_addr), idesc, kb != 0);
          commit_2sm_mc_warp(&empty[stage]);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        if (lane == 0) GTRACE(5, iter);
        commit_2sm_mc_warp(&tfull[acc]);
      }
    }
  } else {
    const int wq = warp & 3;              // TMEM lane quarter this warp may access
    const int half = warp >> 2;           // column half of the tile
    const int row_in_tile = (int)cta * GEMM_BM + wq * 32 + lane;
    float4* epi_box = reinterpret_cast<float4*>(smem + EPI_BOX_OFF + warp * 4096);
    int iter = 0;
    for (int t = cid; t < args.total_tiles; t += ncl, ++iter) {
      const TileInfo ti = decode_tile(args, t);
      const int acc = iter & 1;
      const uint32_t acc_phase = (iter >> 1) & 1;
      prefetch_epilogue_rows(args.p[ti.p], ti, row_in_tile, half * (GEMM_BN / 2));
      mbar_wait(&tfull[acc], acc_phase);
      if (warp == 0 && lane == 0) GTRACE(0, iter);
      tc_fence_after();
      const uint32_t tbase = tmem_base + ((uint32_t)(wq * 32) << 16) + acc * GEMM_BN;
      epilogue_tile(args.p[ti.p], ti, tbase, row_in_tile, half * (GEMM_BN / 2), epi_box);
      if (lane == 0 && (warp == 0 || warp == 7)) GTRACE(warp == 0 ? 1 : 2, iter);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (leader)
          mbar_arrive(&tempty[acc]);
        else
          mbar_arrive_cta(&tempty[acc], 0);
      }
    }
#if GEMM_RESID_TMA
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");   // reduce-adds complete
#endif
  }
  tc_fence_before();
  cluster_sync();
  if (warp == W_MMA) {
    tc_fence_after();
    tmem_dealloc_2sm<TMEM_COLS>(tmem_base);
  }
}

// ------------------------------------------------------------------ host
typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                      const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                      CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static PFN_encodeTiled get_encode() {
  static PFN_encodeTiled fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_encodeTiled>(p);
  }
  return fn;
}

bool make_tmap_2d(CUtensorMap* m, const void* ptr, uint64_t inner, uint64_t outer, uint64_t row_stride_bytes,
                  uint32_t box_inner, uint32_t box_outer) {
  PFN_encodeTiled enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {row_stride_bytes};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    fprintf(stderr, "[libdit] cuTensorMapEncodeTiled failed (%d): inner=%llu outer=%llu stride=%llu ptr=%p\n",
            (int)r, (unsigned long long)inner, (unsigned long long)outer, (unsigned long long)row_stride_bytes, ptr);
    return false;
  }
  return true;
}

bool make_tmap_2d_f32(CUtensorMap* m, const void* ptr, uint64_t inner, uint64_t outer, uint64_t row_stride_bytes,
                      uint32_t box_inner, uint32_t box_outer) {
  PFN_encodeTiled enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {row_stride_bytes};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t estr[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(ptr), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

bool make_tmap_3d(CUtensorMap* m, const void* ptr, uint64_t d0, uint64_t d1, uint64_t d2, uint64_t stride1_bytes,
                  uint64_t stride2_bytes, uint32_t box0, uint32_t box1) {
  PFN_encodeTiled enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[3] = {d0, d1, d2};
  cuuint64_t strides[2] = {stride1_bytes, stride2_bytes};
  cuuint32_t box[3] = {box0, box1, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(ptr), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

cudaError_t gemm_launch(const GemmArgs& args_in, int num_sms, cudaStream_t s) {
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  if (args_in.total_tiles <= 0) return cudaSuccess;
  // rasterisation group per problem: K <= 4096 groups of GEMM_GROUP_M (16) M-tiles (the weight is
  // re-read once per group), K-heavy (fc2 / linear2) groups of 8 (a group's 6-8 MB A panels must
  // stay in L2 while N is swept): cfg3 +0.2-0.35% over 16 on two boxes;
  // DIT_GEMM_GROUP_LIGHT / DIT_GEMM_GROUP_HEAVY override
  static int g_light = -1, g_heavy = -1;
  if (g_light < 0) {
    const char* a = getenv("DIT_GEMM_GROUP_LIGHT");
    const char* b = getenv("DIT_GEMM_GROUP_HEAVY");
    g_light = a ? std::max(1, atoi(a)) : GEMM_GROUP_M;
    g_heavy = b ? std::max(1, atoi(b)) : 8;
  }
  GemmArgs args = args_in;
  for (int i = 0; i < args.num_problems; ++i) args.p[i].group_m = args.p[i].K <= 4096 ? g_light : g_heavy;
  const int pairs = num_sms / 2;
  const int clusters = args.total_tiles < pairs ? args.total_tiles : pairs;
  gemm_kernel<<<2 * clusters, NUM_THREADS, SMEM_BYTES, s>>>(args);
  return cudaGetLastError();
}

cudaError_t gemm_preload() { return preload_module_of(reinterpret_cast<const void*>(&gemm_kernel)); }

}  // namespace dit
