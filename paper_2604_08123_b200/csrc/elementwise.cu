// elementwise.cu -- HBM-bound kernels of the step:
//   * LN-modulate: u = (1 + scale_b) * LN(h) + shift_b, fp32 in, bf16 out,
//     one warp per row, float4 loads, two-pass mean/variance in registers;
//   * skinny GEMM for the conditioning MLPs and ALL adaLN modulations in one
//     launch: out[b][n] = x[b] . W[n] + bias[n] for b < B <= 16 on mma.sync with the
//     weight rows streamed straight from HBM (16-byte loads, K permuted
//     consistently between the A (weights) and B (x) fragments);
//   * small helpers: sinusoid embedding, RoPE table, casts, synthetic fill.
#include "common.cuh"
#include "kernels.h"

namespace dit {

// ------------------------------------------------------------------ LN-modulate
// One 128-thread block per row: thread t holds float4 columns t + 128 i
// (i < 6 for D <= 3072) in registers, two block reductions (mean, then the
// centred variance), modulated bf16 out.  ~40 registers -> full occupancy, so
// enough 16-byte loads are in flight to run near the HBM roofline.
constexpr int LN_THREADS = 128;
constexpr int LN_MAXV = 6;   // float4 per thread: D <= 3072

DEVI float block_sum_128(float v, float* red) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffff, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) red[w] = v;
  __syncthreads();
  v = (red[0] + red[1]) + (red[2] + red[3]);
  __syncthreads();
  return v;
}

__global__ void __launch_bounds__(LN_THREADS) lnmod_kernel(const LnModParams p, int total_rows) {
  __shared__ float red[4];
  int r = blockIdx.x;
  if (r >= total_rows) return;
  int seg = 0;
  if (p.nseg > 1 && r >= p.seg_rows[0]) {
    seg = 1;
    r -= p.seg_rows[0];
  }
  const int rpr = p.seg_rows_per_req[seg];
  const int b = r / rpr;
  const int n = r - b * rpr;
  const int jrow = b * p.joint_n + p.seg_joint_off[seg] + n;
  const int D = p.D;
  const int nv = D / 4;
  const int t = threadIdx.x;
  const float4* hrow = reinterpret_cast<const float4*>(p.h + (size_t)jrow * D);
  float4 x[LN_MAXV];
  float sum = 0.f;
#pragma unroll
  for (int i = 0; i < LN_MAXV; ++i) {
    const int c = t + LN_THREADS * i;
    if (c < nv) {
      x[i] = __ldcs(hrow + c);
      sum += (x[i].x + x[i].y) + (x[i].z + x[i].w);
    }
  }
  const float mean = block_sum_128(sum, red) / (float)D;
  float var = 0.f;
#pragma unroll
  for (int i = 0; i < LN_MAXV; ++i) {
    const int c = t + LN_THREADS * i;
    if (c < nv) {
      const float a = x[i].x - mean, bb = x[i].y - mean, cc = x[i].z - mean, dd = x[i].w - mean;
      var += (a * a + bb * bb) + (cc * cc + dd * dd);
    }
  }
  const float rstd = rsqrtf(block_sum_128(var, red) / (float)D + 1e-6f);
  const float* modb = p.seg_mod[seg] + (size_t)b * p.mod_stride;
  const float4* sh = reinterpret_cast<const float4*>(modb + p.seg_shift_off[seg]);
  const float4* sc = reinterpret_cast<const float4*>(modb + p.seg_scale_off[seg]);
  const int out_row = (seg == 1 ? p.seg_rows[0] : 0) + r;
  uint2* urow = reinterpret_cast<uint2*>(reinterpret_cast<bf16*>(p.u) + (size_t)out_row * D);
#pragma unroll
  for (int i = 0; i < LN_MAXV; ++i) {
    const int c = t + LN_THREADS * i;
    if (c < nv) {
      const float4 s4 = __ldg(sh + c), c4 = __ldg(sc + c);
      uint2 o;
      o.x = pack_bf16((1.f + c4.x) * ((x[i].x - mean) * rstd) + s4.x, (1.f + c4.y) * ((x[i].y - mean) * rstd) + s4.y);
      o.y = pack_bf16((1.f + c4.z) * ((x[i].z - mean) * rstd) + s4.z, (1.f + c4.w) * ((x[i].w - mean) * rstd) + s4.w);
      urow[c] = o;
    }
  }
}

// Persistent variant for large row counts: each 128-thread block walks rows
// r = blockIdx.x, +gridDim.x, ...; one thread streams the NEXT row of fp32 h into
// a shared-memory stage with a bulk copy (cp.async.bulk, mbarrier complete_tx)
// while the block normalises the current one from the other stage, so the HBM
// reads stay in flight independently of the reductions (the one-block-per-row
// kernel is limited by register occupancy to ~120 KB in flight per SM).
constexpr int LNP_STAGES = 2;
#ifndef LNP_CTAS_PER_SM
#define LNP_CTAS_PER_SM 8
#endif
constexpr int LNP_MAXD = 3072;

DEVI int ln_row_of(const LnModParams& p, int r, int& seg, int& b, int& n, int& out_row) {
  seg = 0;
  out_row = r;
  if (p.nseg > 1 && r >= p.seg_rows[0]) {
    seg = 1;
    r -= p.seg_rows[0];
  }
  const int rpr = p.seg_rows_per_req[seg];
  b = r / rpr;
  n = r - b * rpr;
  return b * p.joint_n + p.seg_joint_off[seg] + n;   // row of h
}

__global__ void __launch_bounds__(LN_THREADS) lnmod_persistent_kernel(const __grid_constant__ LnModParams p, int total_rows) {
  __shared__ __align__(128) float4 stage[LNP_STAGES][LNP_MAXD / 4];
  __shared__ __align__(8) uint64_t full[LNP_STAGES];
  __shared__ float red[4];
  const int D = p.D, nv = D / 4, t = threadIdx.x;
  const uint32_t bytes = (uint32_t)D * 4;
  if (t == 0) {
    for (int i = 0; i < LNP_STAGES; ++i) mbar_init(&full[i], 1);
    fence_barrier_init();
  }
  __syncthreads();
  auto issue = [&](int r, int st) {
    int seg, b, n, orow;
    const int jrow = ln_row_of(p, r, seg, b, n, orow);
    mbar_expect_tx(&full[st], bytes);
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
                     "r"(smem_u32(&stage[st][0])), "l"(p.h + (size_t)jrow * D), "r"(bytes), "r"(smem_u32(&full[st]))
                 : "memory");
  };
  int it = 0;
  if (t == 0 && (int)blockIdx.x < total_rows) issue(blockIdx.x, 0);
  for (int r = blockIdx.x; r < total_rows; r += gridDim.x, ++it) {
    const int st = it % LNP_STAGES;
    // the stage being refilled was released by the __syncthreads at the end of the last row
    if (t == 0 && r + (int)gridDim.x < total_rows) issue(r + gridDim.x, (it + 1) % LNP_STAGES);
    mbar_wait(&full[st], (it / LNP_STAGES) & 1);
    int seg, b, n, out_row;
    ln_row_of(p, r, seg, b, n, out_row);
    float4 x[LN_MAXV];
    float sum = 0.f;
#pragma unroll
    for (int i = 0; i < LN_MAXV; ++i) {
      const int c = t + LN_THREADS * i;
      if (c < nv) {
        x[i] = stage[st][c];
        sum += (x[i].x + x[i].y) + (x[i].z + x[i].w);
      }
    }
    const float mean = block_sum_128(sum, red) / (float)D;
    float var = 0.f;
#pragma unroll
    for (int i = 0; i < LN_MAXV; ++i) {
      const int c = t + LN_THREADS * i;
      if (c < nv) {
        const float a = x[i].x - mean, bb = x[i].y - mean, cc = x[i].z - mean, dd = x[i].w - mean;
        var += (a * a + bb * bb) + (cc * cc + dd * dd);
      }
    }
    const float rstd = rsqrtf(block_sum_128(var, red) / (float)D + 1e-6f);
    const float* modb = p.seg_mod[seg] + (size_t)b * p.mod_stride;
    const float4* sh = reinterpret_cast<const float4*>(modb + p.seg_shift_off[seg]);
    const float4* sc = reinterpret_cast<const float4*>(modb + p.seg_scale_off[seg]);
    uint2* urow = reinterpret_cast<uint2*>(reinterpret_cast<bf16*>(p.u) + (size_t)out_row * D);
#pragma unroll
    for (int i = 0; i < LN_MAXV; ++i) {
      const int c = t + LN_THREADS * i;
      if (c < nv) {
        const float4 s4 = __ldg(sh + c), c4 = __ldg(sc + c);
        uint2 o;
        o.x = pack_bf16((1.f + c4.x) * ((x[i].x - mean) * rstd) + s4.x, (1.f + c4.y) * ((x[i].y - mean) * rstd) + s4.y);
        o.y = pack_bf16((1.f + c4.z) * ((x[i].z - mean) * rstd) + s4.z, (1.f + c4.w) * ((x[i].w - mean) * rstd) + s4.w);
        urow[c] = o;
      }
    }
    // (block_sum_128's trailing __syncthreads already ordered every read of this stage
    // before the next iteration's refill of it)
  }
}

cudaError_t lnmod_launch(const LnModParams& p, cudaStream_t s) {
  if (p.D % 4 != 0 || p.D / 4 > LN_MAXV * LN_THREADS) return cudaErrorInvalidValue;
  const int total = p.seg_rows[0] + (p.nseg > 1 ? p.seg_rows[1] : 0);
  if (total <= 0) return cudaSuccess;
  static int sms = 0;
  if (sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  const bool aligned = (reinterpret_cast<uintptr_t>(p.h) & 15) == 0 && (p.D * 4) % 16 == 0;
  if (p.D <= LNP_MAXD && aligned && total >= LNP_CTAS_PER_SM * sms) {
    lnmod_persistent_kernel<<<LNP_CTAS_PER_SM * sms, LN_THREADS, 0, s>>>(p, total);
  } else {
    lnmod_kernel<<<total, LN_THREADS, 0, s>>>(p, total);
  }
  return cudaGetLastError();
}

// ------------------------------------------------------------------ deferred-fetch test producer
__global__ void delayed_publish_kernel(uint4* __restrict__ dst, const uint4* __restrict__ src, size_t n16,
                                       uint32_t* flag, uint32_t value, uint64_t delay_ns) {
  if (threadIdx.x == 0) {
    uint64_t t0, t1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    do {
      __nanosleep(1000);
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    } while (t1 - t0 < delay_ns);
  }
  __syncthreads();
  for (size_t i = threadIdx.x; i < n16; i += blockDim.x) dst[i] = src[i];
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(flag), "r"(value) : "memory");
  }
}

cudaError_t delayed_publish_launch(void* dst, const void* src, size_t bytes, uint32_t* flag, uint32_t value,
                                   uint64_t delay_ns, cudaStream_t s) {
  if (bytes % 16 || (reinterpret_cast<uintptr_t>(dst) & 15) || (reinterpret_cast<uintptr_t>(src) & 15))
    return cudaErrorInvalidValue;
  delayed_publish_kernel<<<1, 1024, 0, s>>>(static_cast<uint4*>(dst), static_cast<const uint4*>(src), bytes / 16,
                                            flag, value, delay_ns);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ fused Ulysses exchange barrier
__global__ void sp_signal_kernel(PeerFlags peers, int me, int P, uint32_t epoch) {
  const int t = threadIdx.x;
  if (t < P && t != me) {
    __threadfence_system();   // the producing kernel's peer stores (earlier on this stream) first
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(peers.f[t] + me), "r"(epoch) : "memory");
  }
}
__global__ void sp_wait_kernel(const uint32_t* flags, int me, int P, uint32_t epoch) {
  const int t = threadIdx.x;
  if (t < P && t != me) {
    uint32_t v, spins = 0;
    while (true) {
      asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(flags + t) : "memory");
      if ((int32_t)(v - epoch) >= 0) break;
      __nanosleep(128);
      if (++spins > (1u << 28)) __trap();   // a peer that never arrives (~30 s): fail loudly, do not hang
    }
  }
  // the next kernels read the peers' stores, also through TMA (async proxy)
  asm volatile("fence.proxy.async.global;" ::: "memory");
}
cudaError_t sp_signal_launch(const PeerFlags& peers, int me, int P, uint32_t epoch, cudaStream_t s) {
  sp_signal_kernel<<<1, 32, 0, s>>>(peers, me, P, epoch);
  return cudaGetLastError();
}
cudaError_t sp_wait_launch(const uint32_t* flags, int me, int P, uint32_t epoch, cudaStream_t s) {
  sp_wait_kernel<<<1, 32, 0, s>>>(flags, me, P, epoch);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ ControlNet push (f2)
__global__ void __launch_bounds__(256) push_copy_kernel(uint4* __restrict__ dst, const uint4* __restrict__ src,
                                                        size_t n16) {
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  // 4 independent 16-byte loads in flight per thread before the (possibly remote) stores
  for (; i + 3 * stride < n16; i += 4 * stride) {
    const uint4 a = __ldg(src + i), b = __ldg(src + i + stride), c = __ldg(src + i + 2 * stride),
                d = __ldg(src + i + 3 * stride);
    dst[i] = a;
    dst[i + stride] = b;
    dst[i + 2 * stride] = c;
    dst[i + 3 * stride] = d;
  }
  for (; i < n16; i += stride) dst[i] = __ldg(src + i);
}
__global__ void push_release_kernel(uint32_t* flag, uint32_t value) {
  // every store of the copy kernel happens-before this kernel (same stream); the system-scope
  // fence + release make them visible to a consumer that acquires the flag (any GPU / process)
  __threadfence_system();
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(flag), "r"(value) : "memory");
}
cudaError_t controlnet_push_launch(void* dst, const void* src, size_t bytes, uint32_t* flag, uint32_t value,
                                   int num_sms, cudaStream_t s) {
  if (bytes % 16 || (reinterpret_cast<uintptr_t>(dst) & 15) || (reinterpret_cast<uintptr_t>(src) & 15))
    return cudaErrorInvalidValue;
  const size_t n16 = bytes / 16;
  if (n16 > 0) {
    const size_t want = (n16 + 1023) / 1024;
    const unsigned grid = (unsigned)std::min<size_t>(want, (size_t)num_sms * 4);
    push_copy_kernel<<<grid, 256, 0, s>>>(static_cast<uint4*>(dst), static_cast<const uint4*>(src), n16);
  }
  push_release_kernel<<<1, 1, 0, s>>>(flag, value);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ merged LoRA
// Weight patching: W' = bf16(W + s * B A) for one adapted linear.
// A 128 x 128 output tile per CTA, 8 warps x 16 rows; the rank-r product runs on
// mma.sync m16n8k16 (r <= 128: 8 K-steps at most) with the B rows (A operand) and the
// A columns (B operand, ldmatrix .trans from its [k][n] storage) staged in shared memory.
// Bandwidth-bound: 2 bytes read + 2 written per weight (+ the tiny factors).
#ifndef LORA_MERGE_ROWS
#define LORA_MERGE_ROWS 128
#endif
constexpr int LM_TILE = 128, LM_ROWS = LORA_MERGE_ROWS, LM_PAD = 8, LM_MAXR = 128;   // tile: LM_ROWS x LM_TILE

DEVI void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(addr));
}
DEVI void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(addr));
}

__global__ void __launch_bounds__(LM_ROWS * 2, LM_ROWS == 64 ? 6 : 3) lora_merge_kernel(const bf16* __restrict__ W, const bf16* __restrict__ A,
                                                         const bf16* __restrict__ Bm, bf16* __restrict__ out, int rows,
                                                         int cols, int ra, float scale) {
  // smem: W tile [LM_ROWS][128 + PAD] (staged in and out with 16-byte coalesced copies), B rows of
  // the tile [128][ra + PAD], A columns of the tile [ra][128 + PAD]
  extern __shared__ __align__(16) uint8_t lm_smem[];
  constexpr int LDW = LM_TILE + LM_PAD;
  bf16* sW = reinterpret_cast<bf16*>(lm_smem);
  bf16* sB = sW + LM_ROWS * LDW;
  bf16* sA = sB + LM_ROWS * (ra + LM_PAD);
  const int row0 = blockIdx.y * LM_ROWS, col0 = blockIdx.x * LM_TILE;
  const int t = threadIdx.x, warp = t / 32, lane = t % 32;
  const int ldb = ra + LM_PAD, lda = LM_TILE + LM_PAD;
  const bool full = row0 + LM_ROWS <= rows && col0 + LM_TILE <= cols && (cols % 8) == 0;
  // 1. everything in flight at once: W tile, B rows, A columns (cp.async, 16 B per request)
  if (full) {
    for (int i = t; i < LM_ROWS * (LM_TILE / 8); i += blockDim.x) {
      const int r = i / (LM_TILE / 8), c8 = (i % (LM_TILE / 8)) * 8;
      cp_async16(smem_u32(sW + r * LDW + c8), W + (size_t)(row0 + r) * cols + col0 + c8, true);
    }
  } else {
    for (int i = t; i < LM_ROWS * LM_TILE; i += blockDim.x) {
      const int r = i / LM_TILE, c = i % LM_TILE;
      sW[r * LDW + c] = (row0 + r < rows && col0 + c < cols) ? W[(size_t)(row0 + r) * cols + col0 + c]
                                                             : __float2bfloat16_rn(0.f);
    }
  }
  for (int i = t; i < LM_ROWS * (ra / 8); i += blockDim.x) {
    const int r = i / (ra / 8), k8 = (i - r * (ra / 8)) * 8;
    const bool ok = row0 + r < rows;
    cp_async16(smem_u32(sB + r * ldb + k8), Bm + (size_t)(ok ? row0 + r : 0) * ra + k8, ok);
  }
  for (int i = t; i < ra * (LM_TILE / 8); i += blockDim.x) {
    const int k = i / (LM_TILE / 8), c8 = (i - k * (LM_TILE / 8)) * 8;
    if (col0 + c8 + 8 <= cols && (cols % 8) == 0) {
      cp_async16(smem_u32(sA + k * lda + c8), A + (size_t)k * cols + col0 + c8, true);
    } else {
      for (int q = 0; q < 8; ++q)
        sA[k * lda + c8 + q] = col0 + c8 + q < cols ? A[(size_t)k * cols + col0 + c8 + q] : __float2bfloat16_rn(0.f);
    }
  }
  cp_async_commit();
  cp_async_wait<0>();
  __syncthreads();
  // 2. the rank-r product on mma.sync (LM_ROWS / 16 warps x 16 rows x 128 columns)
  float acc[16][4];
#pragma unroll
  for (int j = 0; j < 16; ++j) acc[j][0] = acc[j][1] = acc[j][2] = acc[j][3] = 0.f;
  const uint32_t sB_base = smem_u32(sB), sA_base = smem_u32(sA);
  for (int k0 = 0; k0 < ra; k0 += 16) {
    uint32_t a[4];
    ldsm_x4(sB_base + (uint32_t)(((warp * 16 + (lane & 15)) * ldb + k0 + (lane >> 4) * 8) * 2), a[0], a[1], a[2], a[3]);
#pragma unroll
    for (int j = 0; j < 16; j += 2) {
      uint32_t b[4];
      // lanes 0-15: k rows k0..k0+15 of n-block j; lanes 16-31: the same rows of n-block j+1
      ldsm_x4_t(sA_base + (uint32_t)(((k0 + (lane & 15)) * lda + j * 8 + (lane >> 4) * 8) * 2), b[0], b[1], b[2], b[3]);
      const uint32_t b0[2] = {b[0], b[1]}, b1[2] = {b[2], b[3]};
      mma_bf16_16816(acc[j], a, b0);
      mma_bf16_16816(acc[j + 1], a, b1);
    }
  }
  // 3. W' = bf16(W + s * acc) in place in smem (fragment: rows gid / gid + 8, cols 2 tig, 2 tig + 1)
  const int gid = lane >> 2, tig = lane & 3;
#pragma unroll
  for (int j = 0; j < 16; ++j)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      uint32_t* p = reinterpret_cast<uint32_t*>(sW + (warp * 16 + gid + h * 8) * LDW + j * 8 + 2 * tig);
      const uint32_t w2 = *p;
      *p = pack_bf16(bf16_lo(w2) + scale * acc[j][2 * h], bf16_hi(w2) + scale * acc[j][2 * h + 1]);
    }
  __syncthreads();
  // 4. coalesced write-out
  if (full) {
    for (int i = t; i < LM_ROWS * (LM_TILE / 8); i += blockDim.x) {
      const int r = i / (LM_TILE / 8), c8 = (i % (LM_TILE / 8)) * 8;
      __stcs(reinterpret_cast<uint4*>(out + (size_t)(row0 + r) * cols + col0 + c8),
             *reinterpret_cast<const uint4*>(sW + r * LDW + c8));
    }
  } else {
    for (int i = t; i < LM_ROWS * LM_TILE; i += blockDim.x) {
      const int r = i / LM_TILE, c = i % LM_TILE;
      if (row0 + r < rows && col0 + c < cols) out[(size_t)(row0 + r) * cols + col0 + c] = sW[r * LDW + c];
    }
  }
}

cudaError_t lora_merge_launch(const void* W, const void* A, const void* Bm, void* out, int rows, int cols, int ra,
                              float scale, cudaStream_t s) {
  if (rows <= 0 || cols <= 0 || ra <= 0 || ra % 16 || ra > LM_MAXR || cols % 2) return cudaErrorInvalidValue;
  const int smem = (LM_ROWS * (LM_TILE + LM_PAD) + LM_ROWS * (ra + LM_PAD) + ra * (LM_TILE + LM_PAD)) * 2;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(lora_merge_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (LM_ROWS * (LM_TILE + LM_PAD) + LM_ROWS * (LM_MAXR + LM_PAD) +
                                          LM_MAXR * (LM_TILE + LM_PAD)) * 2);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  dim3 grid((cols + LM_TILE - 1) / LM_TILE, (rows + LM_ROWS - 1) / LM_ROWS);
  lora_merge_kernel<<<grid, LM_ROWS * 2, smem, s>>>(static_cast<const bf16*>(W), static_cast<const bf16*>(A),
                                            static_cast<const bf16*>(Bm), static_cast<bf16*>(out), rows, cols, ra, scale);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ skinny GEMM
// One warp computes 16 output rows n (all batch columns: one n8 group, two when B > 8) over the full K.
// Per 32-wide K chunk, thread (gid, tig) loads 16 B of W row gid and row gid+8
// at k = base + 8*tig and 16 B of x row gid at the same k; two m16n8k16 MMAs
// consume them with logical k slots {2tig,2tig+1,2tig+8,2tig+9} mapped to
// physical k = base + 8 tig + {0,1,2,3} (first MMA) / {4,5,6,7} (second).
__global__ void __launch_bounds__(256) skinny_kernel(const bf16* __restrict__ x, int K, const SkinnySeg* __restrict__ segs,
                                                     int nseg, int total_rows, float* __restrict__ out, int out_stride,
                                                     int B, int accumulate) {
  const int warp_global = (blockIdx.x * blockDim.x + threadIdx.x) / 32;
  const int lane = threadIdx.x % 32;
  const int row0 = warp_global * 16;
  if (row0 >= total_rows) return;
  // find segment (rows of a segment are a multiple of 16 except possibly the last tile)
  int sidx = 0, srow = row0;
  while (sidx < nseg - 1 && srow >= segs[sidx].rows) {
    srow -= segs[sidx].rows;
    ++sidx;
  }
  const SkinnySeg sg = segs[sidx];
  const int gid = lane / 4, tig = lane % 4;
  const bf16* w0 = reinterpret_cast<const bf16*>(sg.w) + (size_t)min(srow + gid, sg.rows - 1) * K;
  const bf16* w1 = reinterpret_cast<const bf16*>(sg.w) + (size_t)min(srow + gid + 8, sg.rows - 1) * K;
  const bf16* xr = x + (size_t)gid * K;
  const bf16* xr2 = x + (size_t)(gid + 8) * K;   // batch columns 8..15 (B > 8)
  float acc0[4] = {0.f, 0.f, 0.f, 0.f}, acc1[4] = {0.f, 0.f, 0.f, 0.f};
  float acc2[4] = {0.f, 0.f, 0.f, 0.f}, acc3[4] = {0.f, 0.f, 0.f, 0.f};
  const int Kpad = (K + 31) & ~31;
  const bool two = B > 8;   // (uniform) second n8 group of batch columns; the weights are read once
#pragma unroll 4
  for (int k = 8 * tig; k < Kpad; k += 32) {
    const bool ok = k < K;
    const uint4 z = make_uint4(0, 0, 0, 0);
    const uint4 a0 = ok ? __ldg(reinterpret_cast<const uint4*>(w0 + k)) : z;
    const uint4 a1 = ok ? __ldg(reinterpret_cast<const uint4*>(w1 + k)) : z;
    const uint4 xv = ok ? __ldg(reinterpret_cast<const uint4*>(xr + k)) : z;
    uint32_t fa[4] = {a0.x, a1.x, a0.y, a1.y};
    uint32_t fb[2] = {xv.x, xv.y};
    mma_bf16_16816(acc0, fa, fb);
    uint32_t fa2[4] = {a0.z, a1.z, a0.w, a1.w};
    uint32_t fb2[2] = {xv.z, xv.w};
    mma_bf16_16816(acc1, fa2, fb2);
    if (two) {
      const uint4 xw = ok ? __ldg(reinterpret_cast<const uint4*>(xr2 + k)) : z;
      uint32_t fb3[2] = {xw.x, xw.y};
      mma_bf16_16816(acc2, fa, fb3);
      uint32_t fb4[2] = {xw.z, xw.w};
      mma_bf16_16816(acc3, fa2, fb4);
    }
  }
  // C fragment: c0,c1 = (row gid, batch 2tig, 2tig+1), c2,c3 = (row gid+8, ...)
  const bf16* bias = reinterpret_cast<const bf16*>(sg.bias);
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    const int rr = srow + gid + ((e & 3) >= 2 ? 8 : 0);
    const int bb = 2 * tig + (e & 1) + (e >= 4 ? 8 : 0);
    if (rr < sg.rows && bb < B) {
      float v = (e < 4 ? acc0[e & 3] + acc1[e & 3] : acc2[e & 3] + acc3[e & 3]) + __bfloat162float(bias[rr]);
      float* o = out + (size_t)bb * out_stride + sg.out_off + rr;
      if (accumulate) v += *o;
      *o = v;
    }
  }
}

cudaError_t skinny_launch(const void* x, int K, const SkinnySeg* segs_dev, int nseg, int total_rows, float* out,
                          int out_stride, int B, int accumulate, cudaStream_t s) {
  if (K % 8 != 0) return cudaErrorInvalidValue;
  int warps = (total_rows + 15) / 16;
  int blocks = (warps * 32 + 255) / 256;
  skinny_kernel<<<blocks, 256, 0, s>>>(reinterpret_cast<const bf16*>(x), K, segs_dev, nseg, total_rows, out,
                                       out_stride, B, accumulate);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ small helpers
__global__ void prep_x_kernel(const float* x, int B, int K, int silu, bf16* out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= MAX_SEQ * K) return;
  const int b = i / K;
  float v = 0.f;
  if (b < B) {
    v = x[i];
    if (silu) v = v / (1.f + expf(-v));
  }
  out[i] = __float2bfloat16_rn(v);
}
cudaError_t prep_x_launch(const float* x, int B, int K, int silu, void* out, cudaStream_t s) {
  prep_x_kernel<<<(MAX_SEQ * K + 255) / 256, 256, 0, s>>>(x, B, K, silu, reinterpret_cast<bf16*>(out));
  return cudaGetLastError();
}

// e(t) = [cos(1000 t w_k), sin(1000 t w_k)], w_k = 10000^(-k/128), k < 128 (fp64 args).
__global__ void temb_kernel(const float* vals, int B, bf16* out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= MAX_SEQ * 256) return;
  const int b = i / 256, j = i % 256;
  double v = 0.0;
  if (b < B) {
    const int k = j % 128;
    const double w = exp(-log(10000.0) * (double)k / 128.0);
    const double a = 1000.0 * (double)vals[b] * w;
    v = (j < 128) ? cos(a) : sin(a);
  }
  out[i] = __float2bfloat16_rn((float)v);
}
cudaError_t temb_launch(const float* vals, int B, void* out, cudaStream_t s) {
  temb_kernel<<<MAX_SEQ, 256, 0, s>>>(vals, B, reinterpret_cast<bf16*>(out));
  return cudaGetLastError();
}

// RoPE (cos, sin) for local joint rows: rows [0, nt_loc) are txt (position 0),
// rows [nt_loc, nt_loc + ni_loc) are img tokens ni_off + i -> (0, n / W, n % W).
__global__ void rope_table_kernel(float2* tab, int nt_loc, int ni_loc, int ni_off, int img_w, int a0, int a1, int a2,
                                  float theta) {
  const int half = (a0 + a1 + a2) / 2;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (nt_loc + ni_loc) * half) return;
  const int row = i / half, j = i % half;
  double pos[3] = {0.0, 0.0, 0.0};
  if (row >= nt_loc) {
    const int n = ni_off + (row - nt_loc);
    pos[1] = (double)(n / img_w);
    pos[2] = (double)(n % img_w);
  }
  int axis, jj, da;
  if (j < a0 / 2) { axis = 0; jj = j; da = a0; }
  else if (j < (a0 + a1) / 2) { axis = 1; jj = j - a0 / 2; da = a1; }
  else { axis = 2; jj = j - (a0 + a1) / 2; da = a2; }
  const double ang = pos[axis] * pow((double)theta, -2.0 * jj / (double)da);
  tab[i] = make_float2((float)cos(ang), (float)sin(ang));
}
cudaError_t rope_table_launch(float2* tab, int nt_loc, int ni_loc, int nt_off, int ni_off, int img_w, int a0, int a1,
                              int a2, float theta, cudaStream_t s) {
  (void)nt_off;
  const int half = (a0 + a1 + a2) / 2;
  const int n = (nt_loc + ni_loc) * half;
  rope_table_kernel<<<(n + 255) / 256, 256, 0, s>>>(tab, nt_loc, ni_loc, ni_off, img_w, a0, a1, a2, theta);
  return cudaGetLastError();
}

__global__ void cast_bf16_kernel(const float* x, bf16* out, int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = __float2bfloat16_rn(x[i]);
}
__global__ void cast_latents_ragged_kernel(const float* x, bf16* out, int ni_pad, int C, const int* valid,
                                           int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t row = i / C;
  const int b = (int)(row / ni_pad), r = (int)(row - (int64_t)b * ni_pad);
  out[i] = __float2bfloat16_rn(r < valid[b] ? x[i] : 0.f);
}
cudaError_t cast_latents_ragged_launch(const float* x, void* out, int B, int ni_pad, int C, const int* valid,
                                       cudaStream_t s) {
  const int64_t n = (int64_t)B * ni_pad * C;
  if (n <= 0) return cudaSuccess;
  cast_latents_ragged_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(x, reinterpret_cast<bf16*>(out), ni_pad, C,
                                                                          valid, n);
  return cudaGetLastError();
}
cudaError_t cast_bf16_launch(const float* x, void* out, int64_t n, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  cast_bf16_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(x, reinterpret_cast<bf16*>(out), n);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ Ulysses SP layout
// 16-byte granules; rank r_s's local row i is global joint row
//   i <  nt : r_s*nt + i            (txt)
//   i >= nt : P*nt + r_s*ni + i-nt   (img)
__global__ void sp_gather_qkv_kernel(const uint4* __restrict__ recv, uint4* __restrict__ out, int P, int B, int Hl,
                                     int nt, int ni, int g_per_row, long long total) {
  const long long gidx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (gidx >= total) return;
  const int nloc = nt + ni, N = P * nloc;
  long long t = gidx;
  const int g = (int)(t % g_per_row); t /= g_per_row;
  const int i = (int)(t % nloc); t /= nloc;
  const int hl = (int)(t % Hl); t /= Hl;
  const int b = (int)(t % B); t /= B;
  const int sec = (int)(t % 3); t /= 3;
  const int rs = (int)t;
  const int n = sp_global_row(P, nt, ni, rs, i);
  out[sp_attn_vec(B, Hl, N, sec, b, hl, n) * g_per_row + g] = recv[gidx];
}
cudaError_t sp_gather_qkv_launch(const void* recv, void* out, int P, int B, int Hl, int nt_loc, int ni_loc, int d,
                                 cudaStream_t s) {
  const int gpr = d / 8;
  const long long total = (long long)P * 3 * B * Hl * (nt_loc + ni_loc) * gpr;
  if (total == 0) return cudaSuccess;
  sp_gather_qkv_kernel<<<(unsigned)((total + 255) / 256), 256, 0, s>>>(reinterpret_cast<const uint4*>(recv),
                                                                      reinterpret_cast<uint4*>(out), P, B, Hl,
                                                                      nt_loc, ni_loc, gpr, total);
  return cudaGetLastError();
}

__global__ void sp_scatter_o_kernel(const uint4* __restrict__ recv, bf16* __restrict__ out, int ld_out, int split,
                                    int P, int B, int Hl, int nt, int ni, int d, long long total) {
  const long long gidx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (gidx >= total) return;
  const int nloc = nt + ni, gpr = Hl * d / 8;
  long long t = gidx;
  const int g = (int)(t % gpr); t /= gpr;
  const int i = (int)(t % nloc); t /= nloc;
  const int b = (int)(t % B); t /= B;
  const int rs = (int)t;
  const long long row = sp_local_row(split, B, nt, ni, b, i);
  *reinterpret_cast<uint4*>(out + row * ld_out + (long long)rs * Hl * d + g * 8) = recv[gidx];
}
cudaError_t sp_scatter_o_launch(const void* recv, void* out, int ld_out, int split, int P, int B, int Hl, int nt_loc,
                                int ni_loc, int d, cudaStream_t s) {
  const long long total = (long long)P * B * (nt_loc + ni_loc) * (Hl * d / 8);
  if (total == 0) return cudaSuccess;
  sp_scatter_o_kernel<<<(unsigned)((total + 255) / 256), 256, 0, s>>>(reinterpret_cast<const uint4*>(recv),
                                                                     reinterpret_cast<bf16*>(out), ld_out, split, P,
                                                                     B, Hl, nt_loc, ni_loc, d, total);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ synthetic fill (synth/__init__.py)
DEVI uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  uint64_t z = x;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
__global__ void fill_synth_kernel(bf16* dst, int64_t n, uint64_t seed, uint64_t tid, float scale, float offset) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t key = seed ^ (tid << 40) ^ (uint64_t)i;
    const float u = (float)(splitmix64(key) >> 40) * 5.9604644775390625e-08f;   // 2^-24, exact
    const float t = __fsub_rn(__fmul_rn(2.0f, u), 1.0f);
    float w = __fmul_rn(t, scale);
    if (offset != 0.0f) w = __fadd_rn(offset, w);
    dst[i] = __float2bfloat16_rn(w);
  }
}
cudaError_t fill_synthetic_launch(void* dst, int64_t n, uint64_t seed, uint64_t tid, float scale, float offset,
                                  cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  int64_t blocks = (n + 255) / 256;
  if (blocks > 148 * 64) blocks = 148 * 64;
  fill_synth_kernel<<<(unsigned)blocks, 256, 0, s>>>(reinterpret_cast<bf16*>(dst), n, seed, tid, scale, offset);
  return cudaGetLastError();
}


// ------------------------------------------------------------------ SD3 position table (reading C21)
// h[q][nt + i][c] += table[n][c] for every sequence q < S, n = ni_off + i the global image token.
// One thread per (token, frequency k < D/4, axis): sincos in fp64 (the argument reaches 64 rad),
// added to the S sequences' rows (the table is sequence-independent).  Channels [0, D/2) take the
// column coordinate, [D/2, D) the row; within a half [sin(p w_k) | cos(p w_k)], w_k = 1e4^(-k/(D/4)).
__global__ void pos_embed_add_kernel(float* __restrict__ h, int S, int N, int nt, int ni, int ni_off, int img_h,
                                     int img_w, int D, int pe_max, int base) {
  const int q4 = D / 4;
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (long long)ni * 2 * q4) return;
  const int k = (int)(t % q4);
  const int axis = (int)((t / q4) % 2);
  const int i = (int)(t / (2 * q4));
  const int n = ni_off + i;
  const int top = (pe_max - img_h) / 2, left = (pe_max - img_w) / 2;
  const double p = (double)(axis == 0 ? left + n % img_w : top + n / img_w) * (double)base / (double)pe_max;
  const double ang = p * pow(10000.0, -(double)k / (double)q4);
  double sv, cv;
  sincos(ang, &sv, &cv);
  const float sf = (float)sv, cf = (float)cv;
  for (int q = 0; q < S; ++q) {
    float* row = h + ((size_t)q * N + nt + i) * D + axis * (D / 2);
    row[k] += sf;
    row[q4 + k] += cf;
  }
}
cudaError_t pos_embed_add_launch(float* h, int S, int N, int nt, int ni, int ni_off, int img_h, int img_w, int D,
                                 int pe_max, int base, cudaStream_t s) {
  const long long n = (long long)ni * (D / 2);
  if (n <= 0) return cudaSuccess;
  pos_embed_add_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(h, S, N, nt, ni, ni_off, img_h, img_w, D, pe_max,
                                                                    base);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ CFG combine + Euler (reading C22)
// v = vu + g_b (vc - vu); lat_out = lat_in + dsig_b v; v_out = v (optional).  Per request b:
// count = Ni_loc * C contiguous fp32 (count % 4 == 0), float4 granules.
__global__ void cfg_euler_kernel(const float4* __restrict__ vc, const float4* __restrict__ vu,
                                 const float* __restrict__ g, const float* __restrict__ dsig,
                                 const float4* __restrict__ lat_in, float4* __restrict__ lat_out,
                                 float4* __restrict__ v_out, int B, int count4) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (long long)B * count4) return;
  const int b = (int)(t / count4);
  const float gb = g[b], ds = dsig[b];
  const float4 c = vc[t], u = vu[t], x = lat_in[t];
  float4 v, o;
  v.x = u.x + gb * (c.x - u.x);
  v.y = u.y + gb * (c.y - u.y);
  v.z = u.z + gb * (c.z - u.z);
  v.w = u.w + gb * (c.w - u.w);
  o.x = x.x + ds * v.x;
  o.y = x.y + ds * v.y;
  o.z = x.z + ds * v.z;
  o.w = x.w + ds * v.w;
  lat_out[t] = o;
  if (v_out != nullptr) v_out[t] = v;
}
cudaError_t cfg_euler_launch(const float* vc, const float* vu, const float* g, const float* dsig, const float* lat_in,
                             float* lat_out, float* v_out, int B, int count, cudaStream_t s) {
  const long long n = (long long)B * (count / 4);
  if (n <= 0) return cudaSuccess;
  cfg_euler_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(
      reinterpret_cast<const float4*>(vc), reinterpret_cast<const float4*>(vu), g, dsig,
      reinterpret_cast<const float4*>(lat_in), reinterpret_cast<float4*>(lat_out), reinterpret_cast<float4*>(v_out), B,
      count / 4);
  return cudaGetLastError();
}
cudaError_t elementwise_preload() { return preload_module_of(reinterpret_cast<const void*>(&cast_bf16_kernel)); }

}  // namespace dit
