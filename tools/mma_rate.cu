// mma_rate.cu -- standalone microbenchmark: cycles per tcgen05.mma (kind::f16, bf16 -> fp32)
// for the shapes the attention / GEMM kernels use.  Operand data is garbage (smem / TMEM
// contents are irrelevant to throughput).  One CTA (or CTA pair) per SM, all SMs busy.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_2604_08123_b200/csrc mma_rate.cu
#include <cstdio>

#include "common.cuh"

#ifndef ITERS_DEF
#define ITERS_DEF 4096
#endif
constexpr int ITERS = ITERS_DEF;

DEVI uint64_t desc_mn(uint32_t saddr, uint32_t lbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

// attention-like mix: groups of 8 SS (K-major B) into S, then 8 TS (MN-major B) into O
template <int MODE, bool RANDOM>
__global__ void __launch_bounds__(128, 1) mma_mix(long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  {  // fill the operand smem with random bf16 values (|x| ~ 1): data-dependent power
    uint32_t* sp = reinterpret_cast<uint32_t*>(smem);
    for (int i = threadIdx.x; i < 100 * 1024 / 4; i += blockDim.x) {
      uint32_t hsh = (uint32_t)(i * 2654435761u) ^ (blockIdx.x * 97u);
      hsh ^= hsh >> 13; hsh *= 0x5bd1e995u; hsh ^= hsh >> 15;
      sp[i] = (RANDOM ? ((hsh & 0x807F807Fu) | 0x3F003F00u) : 0u);
    }
    __syncthreads();
  }

  __shared__ uint32_t tslot;
  __shared__ uint64_t bar;
  const int warp = threadIdx.x / 32;
  if (warp == 0) tmem_alloc<512>(&tslot);
  if (threadIdx.x == 32) { mbar_init(&bar, 1); fence_barrier_init(); }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  if (threadIdx.x == 32) {
    const uint32_t q = smem_u32(smem), kb = smem_u32(smem + 32768), vb = smem_u32(smem + 65536);
    constexpr uint32_t id_qk = idesc_bf16_f32(128, 128);
    constexpr uint32_t id_pv = idesc_bf16_f32(128, 128) | (MODE == 2 ? 0u : (1u << 16));
    long long t0 = clock64();
    for (int i = 0; i < ITERS / 16; ++i) {
      for (int kk = 0; kk < 8; ++kk) {
        const uint32_t off = (kk >> 2) * 16384 + (kk & 3) * 32;
        tc_mma_f16(tmem + (i & 1) * 128, smem_desc_k_sw128(q + off), smem_desc_k_sw128(kb + off), id_qk, kk != 0);
      }
      if (MODE >= 1) tc_commit(&bar);
      for (int kk = 0; kk < 8; ++kk) {
        const uint64_t bdesc = MODE == 2 ? smem_desc_k_sw128(vb + (kk >> 2) * 16384 + (kk & 3) * 32)
                                         : desc_mn(vb + kk * 2048, 16384);
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem + 256),
            "r"(tmem + 384 + (i & 1) * 64 + kk * 8), "l"(bdesc), "r"(id_pv), "r"(1));
      }
      if (MODE >= 1) tc_commit(&bar);
    }
    tc_commit(&bar);
    long long t1 = clock64();
    if (blockIdx.x == 0) out[0] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc<512>(tmem); }
}

// exact attention order: for t in {0,1}: PV(t) [A = P_t from TMEM, D = O_t], QK(t) [D = S_t]
// ALIAS: P_t lives in the first 64 columns of S_t (WAR hazard PV -> QK); else a separate region.
__device__ uint8_t* g_src = nullptr;
template <bool ALIAS, int TMA_STREAM = 0>
__global__ void __launch_bounds__(128, 1) mma_attn_order(long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t tslot;
  __shared__ uint64_t bar;
  const int warp = threadIdx.x / 32;
  __shared__ uint64_t cbar;
  __shared__ volatile int stop;
  if (warp == 0) tmem_alloc<512>(&tslot);
  if (threadIdx.x == 32) { mbar_init(&bar, 1); mbar_init(&cbar, 1); stop = 0; fence_barrier_init(); }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  if (TMA_STREAM && threadIdx.x == 64) {
    // bulk copies of 16 KB from global into smem [98 KB ... ) (a region the MMAs do not read)
    uint32_t ph = 0;
    const uint8_t* src = g_src + (size_t)blockIdx.x * (1 << 20);
    int n = 0;
    while (!stop && n < 100000) {
      mbar_expect_tx(&cbar, TMA_STREAM * 16384);
      for (int c = 0; c < TMA_STREAM; ++c)
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 16384, [%2];" ::
                     "r"(smem_u32(smem + 65536 + 32768 + (c & 1) * 16384)), "l"(src + ((n * TMA_STREAM + c) % 48) * 16384),
                     "r"(smem_u32(&cbar)) : "memory");
      mbar_wait(&cbar, ph);
      ph ^= 1;
      ++n;
    }
  }
  if (threadIdx.x == 32) {
    const uint32_t q = smem_u32(smem), kb = smem_u32(smem + 32768), vb = smem_u32(smem + 65536);
    constexpr uint32_t id_qk = idesc_bf16_f32(128, 128);
    constexpr uint32_t id_pv = idesc_bf16_f32(128, 128) | (1u << 16);
    // ALIAS: S0 0, S1 128, O0 256, O1 384, P_t = S_t.  Separate: S0 0, S1 128, O0 256, P0 384, P1 448 (O1 = O0)
    long long t0 = clock64();
    for (int i = 0; i < ITERS / 32; ++i) {
      for (int t = 0; t < 2; ++t) {
        const uint32_t pcol = ALIAS ? (uint32_t)(t * 128) : (uint32_t)(384 + t * 64);
        const uint32_t ocol = ALIAS ? (uint32_t)(256 + t * 128) : 256u;
        for (int kk = 0; kk < 8; ++kk)
          asm volatile(
              "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
              "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem + ocol),
              "r"(tmem + pcol + kk * 8), "l"(desc_mn(vb + kk * 2048, 16384)), "r"(id_pv), "r"(1));
        tc_commit(&bar);
        for (int kk = 0; kk < 8; ++kk) {
          const uint32_t off = (kk >> 2) * 16384 + (kk & 3) * 32;
          tc_mma_f16(tmem + t * 128, smem_desc_k_sw128(q + off), smem_desc_k_sw128(kb + off), id_qk, kk != 0);
        }
        tc_commit(&bar);
      }
    }
    tc_commit(&bar);
    long long t1 = clock64();
    if (blockIdx.x == 0) out[0] = t1 - t0;
    stop = 1;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc<512>(tmem); }
}


// attention MMA order with LDW extra warps streaming tcgen05.ld (32x32b.x32) from the S
// columns (and, if ST, tcgen05.st of 16 bf16x2 columns into the P region) concurrently:
// does softmax-side TMEM traffic slow the tensor pipe?
template <int LDW, bool ST, bool MMA_ON = true, int NLD = 1>
__global__ void __launch_bounds__(640, 1) mma_with_ld(long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t tslot;
  __shared__ uint64_t bar;
  __shared__ volatile int stop;
  __shared__ unsigned long long nld;
  const int warp = threadIdx.x / 32;
  if (warp == 0) tmem_alloc<512>(&tslot);
  if (threadIdx.x == 32) { mbar_init(&bar, 1); stop = 0; nld = 0; fence_barrier_init(); }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  if (warp >= 4 && warp < 4 + LDW) {
    const uint32_t lq = (uint32_t)(warp & 3) * 32;
    uint32_t r[32], r2[32], r3[32], r4[32];
    unsigned long long n = 0;
    uint32_t acc = 0;
    while (!stop && n < 2000000) {
      const uint32_t col = (uint32_t)((n & 3) * 32);
      tmem_ld32(tmem + (lq << 16) + col, r);
      if (NLD >= 2) tmem_ld32(tmem + (lq << 16) + ((col + 32) & 127), r2);
      if (NLD >= 4) { tmem_ld32(tmem + (lq << 16) + ((col + 64) & 127), r3); tmem_ld32(tmem + (lq << 16) + ((col + 96) & 127), r4); }
      tmem_ld_wait();
      #pragma unroll
      for (int i = 0; i < 32; ++i) acc += r[i] + (NLD >= 2 ? r2[i] : 0u) + (NLD >= 4 ? r3[i] ^ r4[i] : 0u);
      if (ST) {
        asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
                     ::"r"(tmem + (lq << 16) + 128 + (uint32_t)((n & 3) * 16)), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]),
                     "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]),
                     "r"(r[13]), "r"(r[14]), "r"(r[15]) : "memory");
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      }
      ++n;
    }
    if (acc == 0x12345) out[1] = acc;
    if ((threadIdx.x & 31) == 0) atomicAdd(&nld, n);
  }
  if (threadIdx.x == 32) {
    const uint32_t q = smem_u32(smem), kb = smem_u32(smem + 32768), vb = smem_u32(smem + 65536);
    constexpr uint32_t id_qk = idesc_bf16_f32(128, 128);
    constexpr uint32_t id_pv = idesc_bf16_f32(128, 128) | (1u << 16);
    long long t0 = clock64();
    if (!MMA_ON) { while (clock64() - t0 < 64 * ITERS) {} }
    for (int i = 0; i < (MMA_ON ? ITERS / 32 : 0); ++i) {
      for (int t = 0; t < 2; ++t) {
        for (int kk = 0; kk < 8; ++kk)
          asm volatile(
              "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
              "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem + 256 + t * 128),
              "r"(tmem + 192 + kk * 8), "l"(desc_mn(vb + kk * 2048, 16384)), "r"(id_pv), "r"(1));
        tc_commit(&bar);
        for (int kk = 0; kk < 8; ++kk) {
          const uint32_t off = (kk >> 2) * 16384 + (kk & 3) * 32;
          tc_mma_f16(tmem + t * 64, smem_desc_k_sw128(q + off), smem_desc_k_sw128(kb + off), id_qk, kk != 0);
        }
        tc_commit(&bar);
      }
    }
    tc_commit(&bar);
    mbar_wait(&bar, 0);
    long long t1 = clock64();
    if (blockIdx.x == 0) { out[0] = t1 - t0; }
    stop = 1;
  }
  tc_fence_before();
  __syncthreads();
  if (blockIdx.x == 0 && threadIdx.x == 0) out[2] = (long long)nld;
  if (warp == 0) { tc_fence_after(); tmem_dealloc<512>(tmem); }
}

// attention MMA order with ALUW extra warps hammering the FMA pipe (FFMA2) and MUFU (ex2):
// does heavy CUDA-core work on the same SM slow the tensor pipe?
template <int ALUW, int KIND>
__global__ void __launch_bounds__(640, 1) mma_with_alu(long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t tslot;
  __shared__ uint64_t bar;
  __shared__ volatile int stop;
  const int warp = threadIdx.x / 32;
  if (warp == 0) tmem_alloc<512>(&tslot);
  if (threadIdx.x == 32) { mbar_init(&bar, 1); stop = 0; fence_barrier_init(); }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  if (warp >= 4 && warp < 4 + ALUW) {
    float2 a[8];
    for (int i = 0; i < 8; ++i) a[i] = make_float2(threadIdx.x * 1e-3f + i, i * 0.5f);
    float e[8];
    for (int i = 0; i < 8; ++i) e[i] = -(float)i * 0.01f * threadIdx.x;
    int n = 0;
    while (!stop && n < 1000000) {
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        if (KIND & 1) {
#pragma unroll
          for (int i = 0; i < 8; ++i) a[i] = __ffma2_rn(a[i], make_float2(0.999f, 0.999f), make_float2(1e-3f, 2e-3f));
        }
        if (KIND & 2) {
#pragma unroll
          for (int i = 0; i < 8; ++i) { float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(e[i])); e[i] = y * -0.5f; }
        }
      }
      ++n;
    }
    float sacc = 0;
    for (int i = 0; i < 8; ++i) sacc += a[i].x + a[i].y + e[i];
    if (sacc == 1234.5f) out[1] = 1;
  }
  if (threadIdx.x == 32) {
    const uint32_t q = smem_u32(smem), kb = smem_u32(smem + 32768), vb = smem_u32(smem + 65536);
    constexpr uint32_t id_qk = idesc_bf16_f32(128, 128);
    constexpr uint32_t id_pv = idesc_bf16_f32(128, 128) | (1u << 16);
    for (int w = 0; w < 20000; ++w) __nanosleep(100);   // let the ALU warps ramp up
    long long t0 = clock64();
    for (int i = 0; i < ITERS / 32; ++i) {
      for (int t = 0; t < 2; ++t) {
        for (int kk = 0; kk < 8; ++kk)
          asm volatile(
              "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
              "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem + 256 + t * 128),
              "r"(tmem + 192 + kk * 8), "l"(desc_mn(vb + kk * 2048, 16384)), "r"(id_pv), "r"(1));
        tc_commit(&bar);
        for (int kk = 0; kk < 8; ++kk) {
          const uint32_t off = (kk >> 2) * 16384 + (kk & 3) * 32;
          tc_mma_f16(tmem + t * 64, smem_desc_k_sw128(q + off), smem_desc_k_sw128(kb + off), id_qk, kk != 0);
        }
        tc_commit(&bar);
      }
    }
    tc_commit(&bar);
    mbar_wait(&bar, 0);
    long long t1 = clock64();
    if (blockIdx.x == 0) { out[0] = t1 - t0; }
    stop = 1;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc<512>(tmem); }
}

// serialized groups: issue G MMAs (PV-form then QK-form halves) + commit, wait for the
// commit, repeat -- the per-group latency an empty tensor pipe adds.
template <int G>
__global__ void __launch_bounds__(128, 1) mma_group_latency(long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t tslot;
  __shared__ uint64_t bar;
  const int warp = threadIdx.x / 32;
  if (warp == 0) tmem_alloc<512>(&tslot);
  if (threadIdx.x == 32) { mbar_init(&bar, 1); fence_barrier_init(); }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  if (threadIdx.x == 32) {
    const uint32_t q = smem_u32(smem), kb = smem_u32(smem + 32768), vb = smem_u32(smem + 65536);
    constexpr uint32_t id_qk = idesc_bf16_f32(128, 128);
    constexpr uint32_t id_pv = idesc_bf16_f32(128, 128) | (1u << 16);
    const int groups = ITERS / G;
    long long t0 = clock64();
    for (int i = 0; i < groups; ++i) {
      for (int kk = 0; kk < G; ++kk) {
        if (kk < G / 2 || G == 8) {
          asm volatile(
              "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
              "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem + 256),
              "r"(tmem + 192 + (kk & 7) * 8), "l"(desc_mn(vb + (kk & 7) * 2048, 16384)), "r"(id_pv), "r"(1));
        } else {
          const int k2 = kk & 7;
          const uint32_t off = (k2 >> 2) * 16384 + (k2 & 3) * 32;
          tc_mma_f16(tmem, smem_desc_k_sw128(q + off), smem_desc_k_sw128(kb + off), id_qk, k2 != 0);
        }
      }
      tc_commit(&bar);
      mbar_wait(&bar, i & 1);
    }
    long long t1 = clock64();
    if (blockIdx.x == 0) { out[0] = t1 - t0; }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc<512>(tmem); }
}

// attention MMA order (2 tiles x [8 PV + 8 QK]) with the synchronisation the kernel does
// around each group: MODE 1 = tcgen05.fence::after_thread_sync before each group,
// MODE 2 = + mbarrier wait on an already-completed phase, MODE 3 = + the MMA thread waits
// for the commit of the group two groups back (what the data dependencies allow at best).
template <int MODE>
__global__ void __launch_bounds__(128, 1) mma_sync_cost(long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t tslot;
  __shared__ uint64_t bar[4];
  __shared__ uint64_t done;
  const int warp = threadIdx.x / 32;
  if (warp == 0) tmem_alloc<512>(&tslot);
  if (threadIdx.x == 32) {
    for (int i = 0; i < 4; ++i) mbar_init(&bar[i], 1);
    mbar_init(&done, 1);
    fence_barrier_init();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  if (threadIdx.x == 32) {
    mbar_arrive(&done);   // phase 0 complete
    const uint32_t q = smem_u32(smem), kb = smem_u32(smem + 32768), vb = smem_u32(smem + 65536);
    constexpr uint32_t id_qk = idesc_bf16_f32(128, 128);
    constexpr uint32_t id_pv = idesc_bf16_f32(128, 128) | (1u << 16);
    long long t0 = clock64();
    int g = 0;
    for (int i = 0; i < ITERS / 32; ++i) {
      for (int t = 0; t < 2; ++t, ++g) {
        if (MODE >= 2) mbar_wait(&done, 0);
        if (MODE == 3 && g >= 2) mbar_wait(&bar[t], ((g - 2) >> 1) & 1);
        if (MODE >= 1) tc_fence_after();
        for (int kk = 0; kk < 8; ++kk)
          asm volatile(
              "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
              "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem + 256 + t * 128),
              "r"(tmem + t * 128 + kk * 8), "l"(desc_mn(vb + kk * 2048, 16384)), "r"(id_pv), "r"(1));
        tc_commit(&bar[2 + t]);
        for (int kk = 0; kk < 8; ++kk) {
          const uint32_t off = (kk >> 2) * 16384 + (kk & 3) * 32;
          tc_mma_f16(tmem + t * 128, smem_desc_k_sw128(q + off), smem_desc_k_sw128(kb + off), id_qk, kk != 0);
        }
        tc_commit(&bar[t]);
      }
    }
    mbar_wait(&bar[1], ((g - 1) >> 1) & 1);
    long long t1 = clock64();
    if (blockIdx.x == 0) { out[0] = t1 - t0; }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc<512>(tmem); }
}

// attention MMA order while one thread keeps DEPTH 16-KB bulk copies global->smem in flight
// (ring over a 64-KB smem region the MMAs do not read): smem write bandwidth vs. SS operand reads.
template <int DEPTH>
__global__ void __launch_bounds__(128, 1) mma_with_tma_ring(long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t tslot;
  __shared__ uint64_t bar;
  __shared__ uint64_t cb[8];
  __shared__ volatile int stop;
  __shared__ unsigned long long nbytes;
  const int warp = threadIdx.x / 32;
  if (warp == 0) tmem_alloc<512>(&tslot);
  if (threadIdx.x == 32) {
    mbar_init(&bar, 1);
    for (int i = 0; i < 8; ++i) mbar_init(&cb[i], 1);
    stop = 0;
    nbytes = 0;
    fence_barrier_init();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  if (DEPTH > 0 && threadIdx.x == 64) {
    const uint8_t* src = g_src + (size_t)(blockIdx.x % 8) * (1 << 20);   // L2-resident source
    long long n = 0;
    while (!stop && n < 4000000) {
      const int slot = (int)(n % (DEPTH > 0 ? DEPTH : 1));
      if (n >= DEPTH) mbar_wait(&cb[slot], (uint32_t)(((n / (DEPTH > 0 ? DEPTH : 1)) - 1) & 1));
      mbar_expect_tx(&cb[slot], 16384);
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 16384, [%2];" ::
                   "r"(smem_u32(smem + 98304 + slot * 16384)), "l"(src + (n % 64) * 16384), "r"(smem_u32(&cb[slot])) : "memory");
      ++n;
    }
    nbytes = (unsigned long long)n * 16384;
  }
  if (threadIdx.x == 32) {
    const uint32_t q = smem_u32(smem), kb = smem_u32(smem + 32768), vb = smem_u32(smem + 65536);
    constexpr uint32_t id_qk = idesc_bf16_f32(128, 128);
    constexpr uint32_t id_pv = idesc_bf16_f32(128, 128) | (1u << 16);
    for (int w = 0; w < 2000; ++w) __nanosleep(100);
    long long t0 = clock64();
    for (int i = 0; i < ITERS / 32; ++i) {
      for (int t = 0; t < 2; ++t) {
        for (int kk = 0; kk < 8; ++kk)
          asm volatile(
              "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
              "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem + 256 + t * 128),
              "r"(tmem + t * 128 + kk * 8), "l"(desc_mn(vb + kk * 2048, 16384)), "r"(id_pv), "r"(1));
        tc_commit(&bar);
        for (int kk = 0; kk < 8; ++kk) {
          const uint32_t off = (kk >> 2) * 16384 + (kk & 3) * 32;
          tc_mma_f16(tmem + t * 128, smem_desc_k_sw128(q + off), smem_desc_k_sw128(kb + off), id_qk, kk != 0);
        }
        tc_commit(&bar);
      }
    }
    tc_commit(&bar);
    mbar_wait(&bar, 0);
    long long t1 = clock64();
    if (blockIdx.x == 0) { out[0] = t1 - t0; }
    stop = 1;
  }
  tc_fence_before();
  __syncthreads();
  if (blockIdx.x == 0 && threadIdx.x == 0) out[2] = (long long)(nbytes / 64);
  if (warp == 0) { tc_fence_after(); tmem_dealloc<512>(tmem); }
}

template <int N, bool TS, bool RANDOM = false>
__global__ void __launch_bounds__(128, 1) mma_1cta(long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  {  // fill the operand smem with random bf16 values (|x| ~ 1): data-dependent power
    uint32_t* sp = reinterpret_cast<uint32_t*>(smem);
    for (int i = threadIdx.x; i < 100 * 1024 / 4; i += blockDim.x) {
      uint32_t hsh = (uint32_t)(i * 2654435761u) ^ (blockIdx.x * 97u);
      hsh ^= hsh >> 13; hsh *= 0x5bd1e995u; hsh ^= hsh >> 15;
      sp[i] = (RANDOM ? ((hsh & 0x807F807Fu) | 0x3F003F00u) : 0u);
    }
    __syncthreads();
  }

  __shared__ uint32_t tslot;
  __shared__ uint64_t bar;
  const int warp = threadIdx.x / 32;
  if (warp == 0) tmem_alloc<512>(&tslot);
  if (threadIdx.x == 32) { mbar_init(&bar, 1); fence_barrier_init(); }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  if (threadIdx.x == 32) {
    const uint32_t a = smem_u32(smem), b = smem_u32(smem + 32768);
    constexpr uint32_t idesc = idesc_bf16_f32(128, N);
    long long t0 = clock64();
    for (int i = 0; i < ITERS; ++i) {
      if (TS) {
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem),
            "r"(tmem + 384), "l"(smem_desc_k_sw128(b)), "r"(idesc), "r"(1));
      } else {
        tc_mma_f16(tmem, smem_desc_k_sw128(a), smem_desc_k_sw128(b), idesc, 1);
      }
    }
    tc_commit(&bar);
    mbar_wait(&bar, 0);
    long long t1 = clock64();
    if (blockIdx.x == 0) out[0] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc<512>(tmem); }
}

DEVI uint32_t cl_rank() { uint32_t r; asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r)); return r; }
DEVI void cl_sync() { asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory"); }

template <int N>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1) mma_2cta(long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t tslot;
  __shared__ uint64_t bar;
  const int warp = threadIdx.x / 32;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  if (threadIdx.x == 32) { mbar_init(&bar, 1); fence_barrier_init(); }
  tc_fence_before();
  cl_sync();
  tc_fence_after();
  const uint32_t tmem = tslot;
  if (threadIdx.x == 32 && cl_rank() == 0) {
    const uint32_t a = smem_u32(smem), b = smem_u32(smem + 32768);
    constexpr uint32_t idesc = idesc_bf16_f32(256, N);
    long long t0 = clock64();
    for (int i = 0; i < ITERS; ++i)
      asm volatile(
          "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
          "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
          "l"(smem_desc_k_sw128(a)), "l"(smem_desc_k_sw128(b)), "r"(idesc), "r"(1));
    asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
                 ::"r"(smem_u32(&bar)), "h"((uint16_t)1));
    mbar_wait(&bar, 0);
    long long t1 = clock64();
    if (blockIdx.x == 0) out[0] = t1 - t0;
  }
  tc_fence_before();
  cl_sync();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

template <typename K>
void run(K kern, const char* name, double macs_per_instr, int grid) {
  long long* d;
  cudaMalloc(&d, 8);
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 140 * 1024);
  kern<<<grid, 128, 140 * 1024>>>(d);
  kern<<<grid, 128, 140 * 1024>>>(d);
  cudaError_t e = cudaDeviceSynchronize();
  long long cyc = 0;
  cudaMemcpy(&cyc, d, 8, cudaMemcpyDeviceToHost);
  cudaFree(d);
  if (e != cudaSuccess) { printf("%-34s error %s\n", name, cudaGetErrorString(e)); return; }
  const double cpi = (double)cyc / ITERS;
  printf("%-34s %7.1f clk/instr  %7.0f MAC/clk per SM\n", name, cpi, macs_per_instr / cpi / (grid > 148 ? 1 : 1));
}

template <typename K>
void run_ld(K kern, const char* name, int grid, int ldw, int threads = 640, int smem_kb = 140) {
  long long* d;
  cudaMalloc(&d, 24);
  cudaMemset(d, 0, 24);
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_kb * 1024);
  kern<<<grid, threads, smem_kb * 1024>>>(d);
  kern<<<grid, threads, smem_kb * 1024>>>(d);
  if (cudaGetLastError() != cudaSuccess) { printf("%-34s launch error\n", name); return; }
  cudaError_t e = cudaDeviceSynchronize();
  long long h[3] = {0, 0, 0};
  cudaMemcpy(h, d, 24, cudaMemcpyDeviceToHost);
  cudaFree(d);
  if (e != cudaSuccess) { printf("%-34s error %s\n", name, cudaGetErrorString(e)); return; }
  const double cpi = (double)h[0] / ITERS;
  printf("%-34s %7.1f clk/instr  %7.0f MAC/clk per SM  ld batches per clk (all warps) %.3f  clk per batch per warp %.0f\n",
         name, cpi, 128.0 * 128 * 16 / cpi, (double)h[2] / (double)h[0], (double)h[0] * ldw / (double)(h[2] + 1));
}

int main() {
  int sms = 148;
  uint8_t* src;
  cudaMalloc(&src, (size_t)160 << 20);
  cudaMemset(src, 0x3f, (size_t)160 << 20);
  cudaMemcpyToSymbol(g_src, &src, sizeof(src));
  run(mma_1cta<64, false>, "1cta SS M128 N64 K16", 128.0 * 64 * 16, sms);
  run(mma_1cta<128, false>, "1cta SS M128 N128 K16", 128.0 * 128 * 16, sms);
  run(mma_1cta<256, false>, "1cta SS M128 N256 K16", 128.0 * 256 * 16, sms);
  run(mma_1cta<128, true>, "1cta TS M128 N128 K16", 128.0 * 128 * 16, sms);
  run(mma_1cta<256, true>, "1cta TS M128 N256 K16", 128.0 * 256 * 16, sms);
  // per SM of the pair: half the MACs of one 2-CTA instruction
  run_ld(mma_with_tma_ring<0>, "attn order, no TMA", sms, 1, 128, 180);
  run_ld(mma_with_tma_ring<1>, "attn order + TMA ring depth 1", sms, 1, 128, 180);
  run_ld(mma_with_tma_ring<2>, "attn order + TMA ring depth 2", sms, 1, 128, 180);
  run_ld(mma_with_tma_ring<4>, "attn order + TMA ring depth 4", sms, 1, 128, 180);
  run(mma_sync_cost<0>, "attn order, no sync", 128.0 * 128 * 16, sms);
  run(mma_sync_cost<1>, "attn order + fence::after", 128.0 * 128 * 16, sms);
  run(mma_sync_cost<2>, "attn order + done-wait + fence", 128.0 * 128 * 16, sms);
  run(mma_sync_cost<3>, "attn order + wait group g-2", 128.0 * 128 * 16, sms);
  run(mma_group_latency<1>, "serial groups of 1 MMA", 128.0 * 128 * 16, sms);
  run(mma_group_latency<2>, "serial groups of 2 MMA", 128.0 * 128 * 16, sms);
  run(mma_group_latency<8>, "serial groups of 8 MMA (PV)", 128.0 * 128 * 16, sms);
  run(mma_group_latency<16>, "serial groups of 16 MMA (PV+QK)", 128.0 * 128 * 16, sms);
  run(mma_group_latency<64>, "serial groups of 64 MMA", 128.0 * 128 * 16, sms);
  run_ld(mma_with_ld<4, false>, "attn order + 4 ld warps", sms, 4);
  run_ld(mma_with_ld<16, false>, "attn order + 16 ld warps", sms, 16);
  run_ld(mma_with_ld<16, true>, "attn order + 16 ld+st warps", sms, 16);
  run_ld(mma_with_ld<4, false, false>, "NO MMA, 4 ld warps x1", sms, 4);
  run_ld(mma_with_ld<4, false, false, 2>, "NO MMA, 4 ld warps x2", sms, 4);
  run_ld(mma_with_ld<4, false, false, 4>, "NO MMA, 4 ld warps x4", sms, 4);
  run_ld(mma_with_ld<16, false, false>, "NO MMA, 16 ld warps x1", sms, 16);
  run_ld(mma_with_ld<16, false, false, 4>, "NO MMA, 16 ld warps x4", sms, 16);
  run_ld(mma_with_ld<4, false, true, 2>, "MMA, 4 ld warps x2", sms, 4);
  run_ld(mma_with_ld<4, false, true, 4>, "MMA, 4 ld warps x4", sms, 4);
  run_ld(mma_with_ld<16, false, true, 4>, "MMA, 16 ld warps x4", sms, 16);
  run(mma_attn_order<true>, "attn order, P aliased over S", 128.0 * 128 * 16, sms);
  run(mma_attn_order<false>, "attn order, P separate", 128.0 * 128 * 16, sms);
  run(mma_attn_order<true, 1>, "attn order + TMA stream 16KB", 128.0 * 128 * 16, sms);
  run(mma_attn_order<true, 2>, "attn order + TMA stream 2x16KB", 128.0 * 128 * 16, sms);
  run(mma_mix<1, false>, "mix SS-QK + TS-PV +commits zeros", 128.0 * 128 * 16, sms);
  run(mma_mix<1, true>, "mix SS-QK + TS-PV +commits RANDOM", 128.0 * 128 * 16, sms);
  run(mma_1cta<256, false, true>, "1cta SS M128 N256 RANDOM", 128.0 * 256 * 16, sms);
  run(mma_1cta<128, false, true>, "1cta SS M128 N128 RANDOM", 128.0 * 128 * 16, sms);
  run(mma_2cta<128>, "2cta SS M256 N128 K16 (per SM)", 128.0 * 128 * 16, sms);
  run(mma_2cta<256>, "2cta SS M256 N256 K16 (per SM)", 128.0 * 256 * 16, sms);
  return 0;
}
