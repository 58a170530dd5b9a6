// attention.cu -- joint (txt+img) non-causal attention, O = softmax(Q K^T / sqrt(d)) V.
//
// Version 1: flash-attention-2 style on mma.sync m16n8k16 (bf16 in, fp32 out),
// 128 query rows per CTA (8 warps x 16 rows), 64-key K/V tiles double-buffered
// with cp.async, online softmax in fp32 with exp2.  The tcgen05/TMEM version
// is the planned replacement.
// q/k/v: bf16 [B][H][N][d] (head-major, joint order txt first).
// O rows go to `out` either joint (row b*N+n) or stream-split (txt rows first,
// then img rows) so the projection GEMM can read them as one A operand.
#include "common.cuh"
#include <cstdlib>

#include "kernels.h"

namespace dit {

template <int HD>
struct AttnCfg {
  static constexpr int BQ = 128;
  static constexpr int BKV = 64;
  static constexpr int WARPS = 8;
  static constexpr int CHUNKS = HD / 8;                      // 16-byte chunks per row
  static constexpr int SWZ = (CHUNKS >= 8 ? 8 : CHUNKS) - 1;
  static constexpr int Q_BYTES = BQ * HD * 2;
  static constexpr int KV_BYTES = BKV * HD * 2;
  static constexpr int SMEM = Q_BYTES + 4 * KV_BYTES;          // Q + 2x(K, V)
};

template <int HD>
DEVI uint32_t swz_off(int row, int chunk) {
  return (uint32_t)(row * HD * 2 + ((chunk ^ (row & AttnCfg<HD>::SWZ)) << 4));
}

template <int HD>
DEVI void load_tile_async(uint32_t s_base, const bf16* g, int row0, int rows_total, int nrows, int tid, int nthreads) {
  constexpr int CH = AttnCfg<HD>::CHUNKS;
  for (int i = tid; i < nrows * CH; i += nthreads) {
    const int r = i / CH, c = i % CH;
    const int gr = row0 + r;
    const bool ok = gr < rows_total;
    const bf16* src = g + (size_t)(ok ? gr : 0) * HD + c * 8;
    cp_async16(s_base + swz_off<HD>(r, c), src, ok);
  }
}

template <int HD>
__global__ void __launch_bounds__(256, 1) attn_fwd_kernel(const __grid_constant__ AttnParams p) {
  using C = AttnCfg<HD>;
  extern __shared__ __align__(128) uint8_t smem[];
  const uint32_t sQ = smem_u32(smem);
  const uint32_t sK0 = sQ + C::Q_BYTES;
  const uint32_t sV0 = sK0 + 2 * C::KV_BYTES;

  const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
  const int qt = blockIdx.x, h = blockIdx.y, b = blockIdx.z;
  const int N = p.N;
  const size_t head_off = ((size_t)b * p.H + h) * (size_t)N * HD;
  const bf16* Q = reinterpret_cast<const bf16*>(p.q) + head_off;
  const bf16* K = reinterpret_cast<const bf16*>(p.k) + head_off;
  const bf16* V = reinterpret_cast<const bf16*>(p.v) + head_off;
  const int q0 = qt * C::BQ;
  const int Nv = p.seq_valid ? p.seq_valid[b] : N;   // ragged batch: keys [Nv, N) are padding
  const int nkv = (Nv + C::BKV - 1) / C::BKV;

  load_tile_async<HD>(sQ, Q, q0, N, C::BQ, tid, 256);
  load_tile_async<HD>(sK0, K, 0, Nv, C::BKV, tid, 256);
  load_tile_async<HD>(sV0, V, 0, Nv, C::BKV, tid, 256);
  cp_async_commit();

  // Q fragments (16 rows of this warp, all HD)
  uint32_t qf[HD / 16][4];
  float o[HD / 8][4];
#pragma unroll
  for (int i = 0; i < HD / 8; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
  float m_r[2] = {-INFINITY, -INFINITY}, l_r[2] = {0.f, 0.f};
  const int gid = lane / 4, tig = lane % 4;

  for (int j = 0; j < nkv; ++j) {
    const int buf = j & 1;
    if (j + 1 < nkv) {
      const int nb = buf ^ 1;
      load_tile_async<HD>(sK0 + nb * C::KV_BYTES, K, (j + 1) * C::BKV, Nv, C::BKV, tid, 256);
      load_tile_async<HD>(sV0 + nb * C::KV_BYTES, V, (j + 1) * C::BKV, Nv, C::BKV, tid, 256);
    }
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
    if (j == 0) {
#pragma unroll
      for (int ks = 0; ks < HD / 16; ++ks) {
        const int mat = lane / 8;
        const int row = warp * 16 + (mat & 1) * 8 + lane % 8;
        const int ch = ks * 2 + (mat >> 1);
        ldmatrix_x4(qf[ks], sQ + swz_off<HD>(row, ch));
      }
    }
    const uint32_t sK = sK0 + buf * C::KV_BYTES;
    const uint32_t sV = sV0 + buf * C::KV_BYTES;

    // S = Q K^T : 16 x 64 per warp
    float s[8][4];
#pragma unroll
    for (int i = 0; i < 8; ++i) s[i][0] = s[i][1] = s[i][2] = s[i][3] = 0.f;
#pragma unroll
    for (int np = 0; np < 4; ++np) {          // pairs of 8-key n-tiles
#pragma unroll
      for (int ks = 0; ks < HD / 16; ++ks) {
        uint32_t kb[4];
        const int mat = lane / 8;
        const int key = np * 16 + (mat >> 1) * 8 + lane % 8;
        const int ch = ks * 2 + (mat & 1);
        ldmatrix_x4(kb, sK + swz_off<HD>(key, ch));
        uint32_t b0[2] = {kb[0], kb[1]}, b1[2] = {kb[2], kb[3]};
        mma_bf16_16816(s[2 * np], qf[ks], b0);
        mma_bf16_16816(s[2 * np + 1], qf[ks], b1);
      }
    }
    // mask keys beyond Nv
    const int kbase = j * C::BKV;
    if (kbase + C::BKV > Nv) {
#pragma unroll
      for (int nt = 0; nt < 8; ++nt) {
        const int key = kbase + nt * 8 + 2 * tig;
        if (key >= Nv) { s[nt][0] = -INFINITY; s[nt][2] = -INFINITY; }
        if (key + 1 >= Nv) { s[nt][1] = -INFINITY; s[nt][3] = -INFINITY; }
      }
    }
    // online softmax (rows gid and gid+8)
    float mx[2] = {-INFINITY, -INFINITY};
#pragma unroll
    for (int nt = 0; nt < 8; ++nt) {
      mx[0] = fmaxf(mx[0], fmaxf(s[nt][0], s[nt][1]));
      mx[1] = fmaxf(mx[1], fmaxf(s[nt][2], s[nt][3]));
    }
    float corr[2];
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffff, mx[r], 1));
      mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffff, mx[r], 2));
      const float mnew = fmaxf(m_r[r], mx[r] * p.scale_log2);
      corr[r] = exp2f(m_r[r] - mnew);
      m_r[r] = mnew;
    }
    float ls[2] = {0.f, 0.f};
    uint32_t pf[4][4];   // P as A fragments, 4 k-steps of 16 keys
#pragma unroll
    for (int nt = 0; nt < 8; ++nt) {
      const float p0 = exp2f(s[nt][0] * p.scale_log2 - m_r[0]);
      const float p1 = exp2f(s[nt][1] * p.scale_log2 - m_r[0]);
      const float p2 = exp2f(s[nt][2] * p.scale_log2 - m_r[1]);
      const float p3 = exp2f(s[nt][3] * p.scale_log2 - m_r[1]);
      ls[0] += p0 + p1;
      ls[1] += p2 + p3;
      const int ks = nt / 2, hi = nt & 1;
      pf[ks][hi * 2 + 0] = pack_bf16(p0, p1);
      pf[ks][hi * 2 + 1] = pack_bf16(p2, p3);
    }
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      ls[r] += __shfl_xor_sync(0xffffffff, ls[r], 1);
      ls[r] += __shfl_xor_sync(0xffffffff, ls[r], 2);
      l_r[r] = l_r[r] * corr[r] + ls[r];
    }
#pragma unroll
    for (int i = 0; i < HD / 8; ++i) {
      o[i][0] *= corr[0]; o[i][1] *= corr[0];
      o[i][2] *= corr[1]; o[i][3] *= corr[1];
    }
    // O += P V
#pragma unroll
    for (int ks = 0; ks < 4; ++ks) {
#pragma unroll
      for (int dp = 0; dp < HD / 16; ++dp) {   // pairs of 8-wide d n-tiles
        uint32_t vb[4];
        const int mat = lane / 8;
        const int key = ks * 16 + (mat & 1) * 8 + lane % 8;
        const int ch = dp * 2 + (mat >> 1);
        ldmatrix_x4_trans(vb, sV + swz_off<HD>(key, ch));
        uint32_t b0[2] = {vb[0], vb[1]}, b1[2] = {vb[2], vb[3]};
        uint32_t a[4] = {pf[ks][0], pf[ks][1], pf[ks][2], pf[ks][3]};
        mma_bf16_16816(o[2 * dp], a, b0);
        mma_bf16_16816(o[2 * dp + 1], a, b1);
      }
    }
    __syncthreads();
  }

  // normalise, stage through the (now free) Q smem, write 16-byte chunks
  const float inv0 = 1.f / l_r[0], inv1 = 1.f / l_r[1];
  uint8_t* sq = smem;
#pragma unroll
  for (int i = 0; i < HD / 8; ++i) {
    const int col = i * 8 + 2 * tig;
    const int r0 = warp * 16 + gid, r1 = r0 + 8;
    *reinterpret_cast<uint32_t*>(sq + swz_off<HD>(r0, col / 8) + (col % 8) * 2) = pack_bf16(o[i][0] * inv0, o[i][1] * inv0);
    *reinterpret_cast<uint32_t*>(sq + swz_off<HD>(r1, col / 8) + (col % 8) * 2) = pack_bf16(o[i][2] * inv1, o[i][3] * inv1);
  }
  __syncthreads();
  for (int i = tid; i < C::BQ * C::CHUNKS; i += 256) {
    const int r = i / C::CHUNKS, c = i % C::CHUNKS;
    const int n = q0 + r;
    if (n >= N) continue;
    const uint4 val = *reinterpret_cast<const uint4*>(sq + swz_off<HD>(r, c));
    *reinterpret_cast<uint4*>(attn_out_addr(p, b, n, h, HD) + c * 8) = val;
  }
  if (p.split == 3) __threadfence_system();   // fused exchange: peer stores, system scope
}

template <int HD>
static cudaError_t launch_hd(const AttnParams& p, cudaStream_t s) {
  using C = AttnCfg<HD>;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(attn_fwd_kernel<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  dim3 grid((p.N + C::BQ - 1) / C::BQ, p.H, p.B);
  attn_fwd_kernel<HD><<<grid, 256, C::SMEM, s>>>(p);
  return cudaGetLastError();
}

cudaError_t attention_tc_launch(const AttnParams& p, cudaStream_t s);

// d = 128 (Flux) and d = 64 (SD3 / SD3.5) run on the tcgen05 kernel (attention_tc.cu);
// the mma.sync kernel serves d = 32 (tiny parity configs) and, with DIT_ATTN_MMA_SYNC=1,
// d = 64 (the pre-tcgen05 baseline, for comparison only).
cudaError_t attention_launch(const AttnParams& p, cudaStream_t s) {
  static const bool legacy64 = [] {
    const char* e = getenv("DIT_ATTN_MMA_SYNC");
    return e && e[0] == '1';
  }();
  switch (p.d) {
    case 32: return launch_hd<32>(p, s);
    case 64: return legacy64 ? launch_hd<64>(p, s) : attention_tc_launch(p, s);
    case 128: return attention_tc_launch(p, s);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t attention_mma_preload() { return preload_module_of(reinterpret_cast<const void*>(&attn_fwd_kernel<32>)); }

}  // namespace dit
