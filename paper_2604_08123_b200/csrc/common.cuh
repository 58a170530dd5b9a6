// common.cuh -- sm_100a PTX helpers shared by the libdit kernels.
// mbarrier, TMA (cp.async.bulk.tensor), tcgen05 (alloc / mma / commit / ld),
// bf16 packing.  Encodings follow the PTX ISA for sm_100a; the smem / instr
// descriptor bit layouts are the tcgen05 ones.
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <vector>

#define DEVI __device__ __forceinline__

typedef __nv_bfloat16 bf16;

// ------------------------------------------------------------------ misc
DEVI uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

DEVI uint32_t lane_id() { uint32_t l; asm volatile("mov.u32 %0, %%laneid;" : "=r"(l)); return l; }

DEVI bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n\t.reg .pred P;\n\t"
      "elect.sync _|P, 0xffffffff;\n\t"
      "selp.b32 %0, 1, 0, P;\n\t}"
      : "=r"(pred));
  return pred != 0;
}

DEVI uint32_t pack_bf16(float a, float b) {
  __nv_bfloat162 v = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&v);
}

DEVI float bf16_lo(uint32_t v) { return __uint_as_float(v << 16); }
DEVI float bf16_hi(uint32_t v) { return __uint_as_float(v & 0xffff0000u); }

// ------------------------------------------------------------------ mbarrier
DEVI void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
DEVI void fence_barrier_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
DEVI void fence_async_shared() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

DEVI void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
DEVI void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
#ifndef MBAR_SUSPEND_HINT
#define MBAR_SUSPEND_HINT 1
#endif
DEVI void mbar_wait(uint64_t* bar, uint32_t parity) {
#if MBAR_SUSPEND_HINT
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n\t"
      "@!P1 bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity), "r"(0x989680)
      : "memory");
#else
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
#endif
}

// ------------------------------------------------------------------ TMA
DEVI void tma_prefetch_desc(const void* desc) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(desc)) : "memory");
}
DEVI void tma_load_2d(const void* desc, uint64_t* bar, void* smem, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(smem)),
      "l"(reinterpret_cast<uint64_t>(desc)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}
DEVI void tma_load_3d(const void* desc, uint64_t* bar, void* smem, int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(smem_u32(smem)),
      "l"(reinterpret_cast<uint64_t>(desc)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}

// ------------------------------------------------------------------ tcgen05
DEVI void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
DEVI void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

template <int kCols>
DEVI void tmem_alloc(uint32_t* smem_dst) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(smem_dst)),
               "n"(kCols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
template <int kCols>
DEVI void tmem_dealloc(uint32_t taddr) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "n"(kCols) : "memory");
}

// D[tmem] (+)= A[smem] * B[smem]^T, kind::f16 (bf16 in, fp32 accumulate).
DEVI void tc_mma_f16(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc, uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accum)
      : "memory");
}
// Warp-converged issue (call with all 32 lanes; one lane elected inside the asm): eight
// K=16 SS MMAs covering K = 128 of two K-major SWIZZLE_128B operands laid out as two
// 64-column panels `panel` bytes apart.  Descriptor offsets are added in PTX so every
// operand stays warp-uniform (no per-MMA register->uniform moves or elect loops).
template <uint32_t PANEL_BYTES>
DEVI void tc_mma_ss_k128_warp(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc, uint32_t accum) {
  constexpr uint32_t P4 = PANEL_BYTES >> 4;
  asm volatile(
      "{\n\t.reg .pred L, p;\n\t.reg .b32 alo, ahi, blo, bhi, x, y;\n\t.reg .b64 a, b;\n\t"
      "elect.sync _|L, -1;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "mov.b64 {alo, ahi}, %1;\n\tmov.b64 {blo, bhi}, %2;\n\t"
      "@L tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t"
      "add.s32 x, alo, 2;\n\tadd.s32 y, blo, 2;\n\tmov.b64 a, {x, ahi};\n\tmov.b64 b, {y, bhi};\n\t"
      "@L tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %3, 1;\n\t"
      "add.s32 x, alo, 4;\n\tadd.s32 y, blo, 4;\n\tmov.b64 a, {x, ahi};\n\tmov.b64 b, {y, bhi};\n\t"
      "@L tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %3, 1;\n\t"
      "add.s32 x, alo, 6;\n\tadd.s32 y, blo, 6;\n\tmov.b64 a, {x, ahi};\n\tmov.b64 b, {y, bhi};\n\t"
      "@L tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %3, 1;\n\t"
      "add.s32 x, alo, %5;\n\tadd.s32 y, blo, %5;\n\tmov.b64 a, {x, ahi};\n\tmov.b64 b, {y, bhi};\n\t"
      "@L tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %3, 1;\n\t"
      "add.s32 x, alo, %6;\n\tadd.s32 y, blo, %6;\n\tmov.b64 a, {x, ahi};\n\tmov.b64 b, {y, bhi};\n\t"
      "@L tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %3, 1;\n\t"
      "add.s32 x, alo, %7;\n\tadd.s32 y, blo, %7;\n\tmov.b64 a, {x, ahi};\n\tmov.b64 b, {y, bhi};\n\t"
      "@L tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %3, 1;\n\t"
      "add.s32 x, alo, %8;\n\tadd.s32 y, blo, %8;\n\tmov.b64 a, {x, ahi};\n\tmov.b64 b, {y, bhi};\n\t"
      "@L tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %3, 1;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accum), "n"(P4), "n"(P4 + 2), "n"(P4 + 4), "n"(P4 + 6)
      : "memory");
}
// Warp-converged: eight K=16 TS MMAs (A = bf16 pairs in TMEM, 8 columns per step; B
// MN-major SWIZZLE_128B, 8 K-rows = 1024 B per step) covering K = 128.
DEVI void tc_mma_ts_k128_warp(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc, uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred L, p;\n\t.reg .b32 blo, bhi, y, ta;\n\t.reg .b64 b;\n\t"
      "elect.sync _|L, -1;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "mov.b64 {blo, bhi}, %2;\n\t"
      "@L tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t"
      "add.s32 ta, %1, 8;\n\tadd.s32 y, blo, 128;\n\tmov.b64 b, {y, bhi};\n\t"
      "@L tcgen05.mma.cta_group::1.kind::f16 [%0], [ta], b, %3, 1;\n\t"
      "add.s32 ta, %1, 16;\n\tadd.s32 y, blo, 256;\n\tmov.b64 b, {y, bhi};\n\t"
      "@L tcgen05.mma.cta_group::1.kind::f16 [%0], [ta], b, %3, 1;\n\t"
      "add.s32 ta, %1, 24;\n\tadd.s32 y, blo, 384;\n\tmov.b64 b, {y, bhi};\n\t"
      "@L tcgen05.mma.cta_group::1.kind::f16 [%0], [ta], b, %3, 1;\n\t"
      "add.s32 ta, %1, 32;\n\tadd.s32 y, blo, 512;\n\tmov.b64 b, {y, bhi};\n\t"
      "@L tcgen05.mma.cta_group::1.kind::f16 [%0], [ta], b, %3, 1;\n\t"
      "add.s32 ta, %1, 40;\n\tadd.s32 y, blo, 640;\n\tmov.b64 b, {y, bhi};\n\t"
      "@L tcgen05.mma.cta_group::1.kind::f16 [%0], [ta], b, %3, 1;\n\t"
      "add.s32 ta, %1, 48;\n\tadd.s32 y, blo, 768;\n\tmov.b64 b, {y, bhi};\n\t"
      "@L tcgen05.mma.cta_group::1.kind::f16 [%0], [ta], b, %3, 1;\n\t"
      "add.s32 ta, %1, 56;\n\tadd.s32 y, blo, 896;\n\tmov.b64 b, {y, bhi};\n\t"
      "@L tcgen05.mma.cta_group::1.kind::f16 [%0], [ta], b, %3, 1;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accum)
      : "memory");
}
// Warp-converged single TS MMA (one elected lane issues).
DEVI void tc_mma_ts_warp(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc, uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred L, p;\n\t"
      "elect.sync _|L, -1;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@L tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accum)
      : "memory");
}
// Warp-converged commit (one elected lane).
DEVI void tc_commit_warp(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .pred L;\n\telect.sync _|L, -1;\n\t"
      "@L tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(smem_u32(bar))
      : "memory");
}

// Arrive on an mbarrier when all previously issued tcgen05.mma of this thread complete.
DEVI void tc_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}

// 32 lanes x 32 columns of 32-bit: thread t gets columns [col, col+32) of lane (base + t).
DEVI void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
        "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),
        "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),
        "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
DEVI void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// Shared-memory matrix descriptor, K-major, SWIZZLE_128B (tile rows of 128 B,
// 8-row core groups 1024 B apart): start>>4 [0,14), LBO>>4 [16,30) (unused for
// swizzled K-major, set 1), SBO>>4 [32,46) = 1024>>4, version 1 at [46,48),
// layout type 2 (SWIZZLE_128B) at [61,64).
DEVI uint64_t smem_desc_k_sw128(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

// Instruction descriptor kind::f16: D fp32 (bits 4-5 = 1), A bf16 (7-9 = 1),
// B bf16 (10-12 = 1), both K-major, N>>3 at [17,23), M>>4 at [24,29).
__host__ __device__ constexpr uint32_t idesc_bf16_f32(int M, int N) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

// ------------------------------------------------------------------ mma.sync (legacy HMMA)
DEVI void mma_bf16_16816(float (&d)[4], const uint32_t (&a)[4], const uint32_t (&b)[2]) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}

DEVI void ldmatrix_x4(uint32_t (&r)[4], uint32_t saddr) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(saddr));
}
DEVI void ldmatrix_x4_trans(uint32_t (&r)[4], uint32_t saddr) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(saddr));
}

DEVI void cp_async16(uint32_t saddr, const void* g, bool valid) {
  int sz = valid ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(saddr), "l"(g), "r"(sz) : "memory");
}
DEVI void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
DEVI void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// ------------------------------------------------------------------ 2-SM (CTA pair) helpers
constexpr uint32_t PEER_MASK = 0xFEFFFFFFu;   // shared::cluster address of the leader CTA's copy

DEVI uint32_t cluster_rank() { uint32_t r; asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r)); return r; }
DEVI void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// arrive on the mbarrier at the same smem offset in CTA `cta` of the cluster
DEVI void mbar_arrive_cta(uint64_t* bar, uint32_t cta) {
  asm volatile(
      "{\n\t.reg .b32 ra;\n\t"
      "mapa.shared::cluster.u32 ra, %0, %1;\n\t"
      "mbarrier.arrive.shared::cluster.b64 _, [ra];\n\t}" ::"r"(smem_u32(bar)),
      "r"(cta)
      : "memory");
}
// TMA load into this CTA's smem, completing bytes on the LEADER's mbarrier
DEVI void tma_load_2d_2sm(const void* desc, uint64_t* bar, void* smem, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(smem)),
      "l"(reinterpret_cast<uint64_t>(desc)), "r"(smem_u32(bar) & PEER_MASK), "r"(c0), "r"(c1)
      : "memory");
}
DEVI void tma_load_3d_2sm(const void* desc, uint64_t* bar, void* smem, int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(smem_u32(smem)),
      "l"(reinterpret_cast<uint64_t>(desc)), "r"(smem_u32(bar) & PEER_MASK), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
// D (+)= A * B with A, B in smem, M = 256 across the CTA pair (leader issues)
DEVI void mma_2sm(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc, uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accum)
      : "memory");
}
// D (+)= A * B with A in TMEM (each CTA its 128 rows), B in smem, M = 256
DEVI void mma_ts_2sm(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc, uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accum)
      : "memory");
}
// arrive on the mbarrier at this smem offset in BOTH CTAs once prior MMAs complete
// Warp-converged (call with all 32 lanes of the leader CTA's MMA warp): the four K=16 MMAs of
// one 64-wide K-block of two K-major SWIZZLE_128B operands (+32 B per step), one elected lane.
DEVI void mma_2sm_k64_warp(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc, uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred L, p;\n\t.reg .b32 alo, ahi, blo, bhi, x, y;\n\t.reg .b64 a, b;\n\t"
      "elect.sync _|L, -1;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "mov.b64 {alo, ahi}, %1;\n\tmov.b64 {blo, bhi}, %2;\n\t"
      "@L tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t"
      "add.s32 x, alo, 2;\n\tadd.s32 y, blo, 2;\n\tmov.b64 a, {x, ahi};\n\tmov.b64 b, {y, bhi};\n\t"
      "@L tcgen05.mma.cta_group::2.kind::f16 [%0], a, b, %3, 1;\n\t"
      "add.s32 x, alo, 4;\n\tadd.s32 y, blo, 4;\n\tmov.b64 a, {x, ahi};\n\tmov.b64 b, {y, bhi};\n\t"
      "@L tcgen05.mma.cta_group::2.kind::f16 [%0], a, b, %3, 1;\n\t"
      "add.s32 x, alo, 6;\n\tadd.s32 y, blo, 6;\n\tmov.b64 a, {x, ahi};\n\tmov.b64 b, {y, bhi};\n\t"
      "@L tcgen05.mma.cta_group::2.kind::f16 [%0], a, b, %3, 1;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accum)
      : "memory");
}
DEVI void commit_2sm_mc_warp(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .pred L;\n\telect.sync _|L, -1;\n\t"
      "@L tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n\t}" ::"r"(
          smem_u32(bar)),
      "h"((uint16_t)3)
      : "memory");
}
DEVI void commit_2sm_mc(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"((uint16_t)3)
      : "memory");
}
template <int kCols>
DEVI void tmem_alloc_2sm(uint32_t* smem_dst) {
  asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(smem_dst)),
               "n"(kCols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
}
template <int kCols>
DEVI void tmem_dealloc_2sm(uint32_t taddr) {
  asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "n"(kCols) : "memory");
}

// ------------------------------------------------------------------ eager module loading
// Load every kernel of the module (translation unit) holding `kernel` now.  Under CUDA's lazy
// loading (torch turns it on) a kernel's first launch loads its module, and a load that happens
// while another kernel of the process spins waiting for it -- the fused SP exchange barrier, a
// ControlNet flag, in-process ranks -- can stall until that spin gives up.  dit_create preloads
// every libdit module once.
inline cudaError_t preload_module_of(const void* kernel) {
  typedef CUresult (*PFN_getmod)(CUmodule*, CUfunction);
  typedef CUresult (*PFN_count)(unsigned int*, CUmodule);
  typedef CUresult (*PFN_enum)(CUfunction*, unsigned int, CUmodule);
  typedef CUresult (*PFN_load)(CUfunction);
  static PFN_getmod getmod = nullptr;
  static PFN_count count = nullptr;
  static PFN_enum enumerate = nullptr;
  static PFN_load load = nullptr;
  if (!getmod) {
    void* p[4] = {};
    cudaDriverEntryPointQueryResult q;
    const char* names[4] = {"cuFuncGetModule", "cuModuleGetFunctionCount", "cuModuleEnumerateFunctions", "cuFuncLoad"};
    for (int i = 0; i < 4; ++i)
      if (cudaGetDriverEntryPoint(names[i], &p[i], cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess)
        return cudaErrorNotSupported;
    count = reinterpret_cast<PFN_count>(p[1]);
    enumerate = reinterpret_cast<PFN_enum>(p[2]);
    load = reinterpret_cast<PFN_load>(p[3]);
    getmod = reinterpret_cast<PFN_getmod>(p[0]);
  }
  cudaFunction_t f;
  if (cudaGetFuncBySymbol(&f, kernel) != cudaSuccess) return cudaErrorInvalidDeviceFunction;
  CUmodule m;
  unsigned int n = 0;
  if (getmod(&m, reinterpret_cast<CUfunction>(f)) != CUDA_SUCCESS || count(&n, m) != CUDA_SUCCESS)
    return cudaErrorNotSupported;
  std::vector<CUfunction> fs(n);
  if (n && enumerate(fs.data(), n, m) != CUDA_SUCCESS) return cudaErrorNotSupported;
  for (CUfunction fn : fs)
    if (load(fn) != CUDA_SUCCESS) return cudaErrorNotSupported;
  return cudaSuccess;
}

