// attention_tc.cu -- joint (txt+img) attention on the 5th-gen tensor cores (d = 128).
//
// One CTA = one 128-row query tile of one (request, head); KV tiles of 128 keys.
// TMEM (512 columns): S0 [0,128) S1 [128,256) O [256,384) P0 [384,448) P1 [448,512).
//   warp 0      TMA producer: Q once, K ring (2 stages) and V ring (2 stages), 3D
//               tensor maps [B*H][N][128] so rows past N are zero-filled.
//   warp 1      MMA issuer (one thread): S_j = Q K_j^T (SS, both K-major), then
//               O += P_j V_j with P_j read from TMEM (TS form) and V_j MN-major
//               in smem.  QK_{j+2} is issued right after PV_j so the tensor
//               pipe works on the next scores while softmax runs.
//   warps 4-7   softmax (thread = query row = TMEM lane): tcgen05.ld of S_j,
//               online softmax in fp32 with exp2, lazy O rescale (only when the
//               running max grows by > 8 in log2 units, warp-uniform), P_j
//               packed to bf16 and written with tcgen05.st; final O / l epilogue.
// Synchronisation is all mbarriers (TMA complete_tx, tcgen05.commit, thread
// arrivals); see DESIGN.md §5.3 for the phase argument.
#include "common.cuh"
#include "kernels.h"

namespace dit {

namespace attn_tc {

constexpr int BQ = 128, BKV = 128, HD = 128;
constexpr int TILE_BYTES = 128 * HD * 2;         // 32 KB: 128 rows x 128 bf16 (two 64-col swizzle panels)
constexpr int PANEL = 128 * 64 * 2;              // 16 KB
constexpr int KST = 2, VST = 2;
constexpr int SMEM = TILE_BYTES * (1 + KST + VST) + 1024 + 256;
constexpr int THREADS = 256;
constexpr uint32_t COL_S0 = 0, COL_O = 256, COL_P0 = 384;
constexpr float RESCALE_THRESH = 8.0f;

DEVI void tmem_st32(uint32_t taddr, const uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
      "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]),
      "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]),
      "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
      : "memory");
}
DEVI void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// D[tmem] (+)= A[tmem] * B[smem]  (A operand from tensor memory)
DEVI void mma_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc, uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accum)
      : "memory");
}

// MN-major SWIZZLE_128B descriptor: 64-element (128 B) rows along MN, 8-row
// core groups along K 1024 B apart (SBO), next 64-wide MN panel at LBO.
DEVI uint64_t desc_mn_sw128(uint32_t saddr, uint32_t lbo_bytes) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo_bytes >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

DEVI float fast_exp2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

struct Maps {
  CUtensorMap q, k, v;   // 3D {128 (d), N, B*H}, box {64, 128, 1}
};

__global__ void __launch_bounds__(THREADS, 1) attn_tc_kernel(const __grid_constant__ Maps maps, const AttnParams p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;
  uint8_t* sK = smem + TILE_BYTES;
  uint8_t* sV = sK + KST * TILE_BYTES;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sV + VST * TILE_BYTES);
  uint64_t* q_full = bars;
  uint64_t* k_full = bars + 1;        // [KST]
  uint64_t* k_empty = bars + 3;       // [KST]
  uint64_t* v_full = bars + 5;        // [VST]
  uint64_t* v_empty = bars + 7;       // [VST]
  uint64_t* s_full = bars + 9;        // [2]
  uint64_t* p_full = bars + 11;       // [2]
  uint64_t* o_done = bars + 13;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 14);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int qt = blockIdx.x, h = blockIdx.y, b = blockIdx.z;
  const int N = p.N;
  const int bh = b * p.H + h;
  const int q0 = qt * BQ;
  const int nkv = (N + BKV - 1) / BKV;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&maps.q);
    tma_prefetch_desc(&maps.k);
    tma_prefetch_desc(&maps.v);
  }
  if (warp == 1 && lane == 0) {
    mbar_init(q_full, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&k_full[i], 1);
      mbar_init(&k_empty[i], 1);
      mbar_init(&v_full[i], 1);
      mbar_init(&v_empty[i], 1);
      mbar_init(&s_full[i], 1);
      mbar_init(&p_full[i], 128);
    }
    mbar_init(o_done, 1);
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      mbar_expect_tx(q_full, TILE_BYTES);
      tma_load_3d(&maps.q, q_full, sQ, 0, q0, bh);
      tma_load_3d(&maps.q, q_full, sQ + PANEL, 64, q0, bh);
      for (int j = 0; j < nkv; ++j) {
        const int st = j & 1;
        const uint32_t ph = (j >> 1) & 1;
        mbar_wait(&k_empty[st], ph ^ 1);
        mbar_expect_tx(&k_full[st], TILE_BYTES);
        tma_load_3d(&maps.k, &k_full[st], sK + st * TILE_BYTES, 0, j * BKV, bh);
        tma_load_3d(&maps.k, &k_full[st], sK + st * TILE_BYTES + PANEL, 64, j * BKV, bh);
        mbar_wait(&v_empty[st], ph ^ 1);
        mbar_expect_tx(&v_full[st], TILE_BYTES);
        tma_load_3d(&maps.v, &v_full[st], sV + st * TILE_BYTES, 0, j * BKV, bh);
        tma_load_3d(&maps.v, &v_full[st], sV + st * TILE_BYTES + PANEL, 64, j * BKV, bh);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc_qk = idesc_bf16_f32(BQ, BKV);
      constexpr uint32_t idesc_pv = idesc_bf16_f32(BQ, HD) | (1u << 16);   // B (V) MN-major
      const uint32_t q_addr = smem_u32(sQ);
      auto issue_qk = [&](int j) {
        const int st = j & 1;
        mbar_wait(&k_full[st], (j >> 1) & 1);
        tc_fence_after();
        const uint32_t k_addr = smem_u32(sK + st * TILE_BYTES);
        const uint32_t d = tmem + COL_S0 + st * 128;
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk) {
          const uint32_t off = (kk >> 2) * PANEL + (kk & 3) * 32;
          tc_mma_f16(d, smem_desc_k_sw128(q_addr + off), smem_desc_k_sw128(k_addr + off), idesc_qk, kk != 0);
        }
        tc_commit(&k_empty[st]);
        tc_commit(&s_full[st]);
      };
      mbar_wait(q_full, 0);
      issue_qk(0);
      if (nkv > 1) issue_qk(1);
      for (int j = 0; j < nkv; ++j) {
        const int st = j & 1;
        const uint32_t ph = (j >> 1) & 1;
        mbar_wait(&p_full[st], ph);
        mbar_wait(&v_full[st], ph);
        tc_fence_after();
        const uint32_t v_addr = smem_u32(sV + st * TILE_BYTES);
#pragma unroll
        for (int kk = 0; kk < BKV / 16; ++kk) {
          mma_ts(tmem + COL_O, tmem + COL_P0 + st * 64 + kk * 8, desc_mn_sw128(v_addr + kk * 2048, PANEL), idesc_pv,
                 (j | kk) != 0);
        }
        tc_commit(&v_empty[st]);
        tc_commit(o_done);
        if (j + 2 < nkv) issue_qk(j + 2);
      }
    }
  } else if (warp >= 4) {
    const int wq = warp & 3;
    const int row = wq * 32 + lane;
    const uint32_t lane_base = (uint32_t)(wq * 32) << 16;
    const float sl2 = p.scale_log2;
    float m_used = -INFINITY, l = 0.f;
    for (int j = 0; j < nkv; ++j) {
      const int st = j & 1;
      mbar_wait(&s_full[st], (j >> 1) & 1);
      tc_fence_after();
      float s[128];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        uint32_t r[32];
        tmem_ld32(tmem + lane_base + COL_S0 + st * 128 + c * 32, r);
        tmem_ld_wait();
#pragma unroll
        for (int e = 0; e < 32; ++e) s[c * 32 + e] = __uint_as_float(r[e]) * sl2;
      }
      const int kv_valid = N - j * BKV;
      if (kv_valid < BKV) {
#pragma unroll
        for (int e = 0; e < 128; ++e)
          if (e >= kv_valid) s[e] = -INFINITY;
      }
      float mx = s[0];
#pragma unroll
      for (int e = 1; e < 128; ++e) mx = fmaxf(mx, s[e]);
      const bool need = mx > m_used + RESCALE_THRESH;
      const float m_new = need ? mx : m_used;
      if (j > 0 && __any_sync(0xffffffff, need)) {
        const float alpha = need ? fast_exp2(m_used - m_new) : 1.0f;
        mbar_wait(o_done, (j - 1) & 1);
        tc_fence_after();
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          uint32_t r[32];
          tmem_ld32(tmem + lane_base + COL_O + c * 32, r);
          tmem_ld_wait();
#pragma unroll
          for (int e = 0; e < 32; ++e) r[e] = __float_as_uint(__uint_as_float(r[e]) * alpha);
          tmem_st32(tmem + lane_base + COL_O + c * 32, r);
        }
        tmem_st_wait();
        l *= alpha;
      }
      m_used = m_new;
      float sum = 0.f;
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        uint32_t r[32];
#pragma unroll
        for (int e = 0; e < 32; ++e) {
          const float p0 = fast_exp2(s[c * 64 + 2 * e] - m_used);
          const float p1 = fast_exp2(s[c * 64 + 2 * e + 1] - m_used);
          sum += p0 + p1;
          r[e] = pack_bf16(p0, p1);
        }
        tmem_st32(tmem + lane_base + COL_P0 + st * 64 + c * 32, r);
      }
      l += sum;
      tmem_st_wait();
      tc_fence_before();
      mbar_arrive(&p_full[st]);
    }
    // epilogue: O / l -> bf16 rows
    mbar_wait(o_done, (nkv - 1) & 1);
    tc_fence_after();
    const int n = q0 + row;
    const float inv = 1.0f / l;
    bf16* out = reinterpret_cast<bf16*>(p.out);
    const size_t orow = n < N ? (size_t)attn_out_row(p, b, n) : 0;
    uint4* dst = reinterpret_cast<uint4*>(out + orow * p.ld_out + (size_t)h * HD);
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      uint32_t r[32];
      tmem_ld32(tmem + lane_base + COL_O + c * 32, r);
      tmem_ld_wait();
      if (n < N) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          uint4 u;
          u.x = pack_bf16(__uint_as_float(r[8 * q + 0]) * inv, __uint_as_float(r[8 * q + 1]) * inv);
          u.y = pack_bf16(__uint_as_float(r[8 * q + 2]) * inv, __uint_as_float(r[8 * q + 3]) * inv);
          u.z = pack_bf16(__uint_as_float(r[8 * q + 4]) * inv, __uint_as_float(r[8 * q + 5]) * inv);
          u.w = pack_bf16(__uint_as_float(r[8 * q + 6]) * inv, __uint_as_float(r[8 * q + 7]) * inv);
          dst[c * 4 + q] = u;
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

}  // namespace attn_tc

cudaError_t attention_tc_launch(const AttnParams& p, cudaStream_t s) {
  using namespace attn_tc;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(attn_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  Maps m;
  const uint64_t rows = (uint64_t)p.N, heads = (uint64_t)p.B * p.H;
  const uint64_t s1 = (uint64_t)HD * 2, s2 = rows * HD * 2;
  if (!make_tmap_3d(&m.q, p.q, HD, rows, heads, s1, s2, 64, 128) ||
      !make_tmap_3d(&m.k, p.k, HD, rows, heads, s1, s2, 64, 128) ||
      !make_tmap_3d(&m.v, p.v, HD, rows, heads, s1, s2, 64, 128))
    return cudaErrorInvalidValue;
  dim3 grid((p.N + BQ - 1) / BQ, p.H, p.B);
  attn_tc_kernel<<<grid, THREADS, SMEM, s>>>(m, p);
  return cudaGetLastError();
}

}  // namespace dit
