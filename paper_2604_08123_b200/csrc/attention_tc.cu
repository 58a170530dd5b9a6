// attention_tc.cu -- joint (txt+img) attention on the 5th-gen tensor cores (head dim
// HD = 128: Flux; HD = 64: SD3 / SD3.5, one 64-column swizzle panel per tile and O
// in 64 TMEM columns per query tile -- the schedule below is the same).
//
// One CTA = TWO 128-row query tiles (256 queries) of one (request, head); KV
// tiles of 128 keys shared by both query tiles.  TMEM (512 columns):
//   S0 [0,128)  S1 [128,256)  O0 [256,384)  O1 [384,512);  P_t (bf16) is written
//   over the first 64 columns of S_t once the scores have been read.
// Roles (384 threads = 3 warpgroups; the producer and MMA warps take the HIGHEST
// ids because the SMSP arbiter issues highest-id-first):
//   warp 10     TMA producer: Q0/Q1 once, K ring (2 stages), V ring (2 stages);
//               3D tensor maps [B*H][N][128] so rows past N are zero-filled.
//   warp 11     TMEM allocator + MMA issuer.  The whole warp walks the schedule
//               and one elected lane issues inside each asm block, so every
//               descriptor lives in uniform registers (issuing from a divergent
//               lane-0 branch cost ~80 clk per MMA in R2UR/elect loops and made
//               the MMA issue itself the bottleneck).  Ping-pong schedule:
//                 QK(0,0) QK(1,0) | PV(0,j) QK(0,j+1) PV(1,j) QK(1,j+1) | ...
//               so the tensor pipe computes one query tile's PV + next scores
//               while the other tile's softmax runs.  QK is SS (both K-major),
//               PV is TS (P from TMEM, V MN-major in smem); the PV of a tile
//               starts on kv [0,96) of P and waits for the last quarter
//               (split P arrive).
//   warps 8-9   idle (complete warpgroup 2 for setmaxnreg).
//   warps 0-3   softmax of query tile 0, warps 4-7 of tile 1: one query row per
//               thread (TMEM lane = row), all 128 scores in registers
//               (setmaxnreg: 208 registers for the softmax warpgroups, 80 for
//               warpgroup 2).  Row max, lazy O rescale (only when the running
//               max grows by > 8 in log2 units), packed f32x2 FFMA, exp2 with
//               1/ATTN_POLY_MOD (1/8) of the pairs on a degree-3 polynomial (FMA pipe)
//               and the rest on MUFU, P packed to bf16 and stored with
//               tcgen05.st in 16-column chunks; the row sum is accumulated after
//               P is released (off the MMA's critical path); final O / l
//               epilogue writes one 256-byte output row per thread.
// Synchronisation: mbarriers only (TMA complete_tx, tcgen05.commit, thread
// arrivals); every waiter can be at most one phase behind.
#include "common.cuh"
#include "kernels.h"

namespace dit {

namespace attn_tc {

constexpr int BQ = 128, NQ = 2, BKV = 128;
constexpr int PANEL = 128 * 64 * 2;              // 16 KB: 128 rows x 64 bf16 (one 128-byte swizzle span)
#ifndef ATTN_KST
#define ATTN_KST 2
#endif
#ifndef ATTN_VST
#define ATTN_VST 2
#endif
#ifndef ATTN_KST64
#define ATTN_KST64 3
#endif
#ifndef ATTN_VST128
#define ATTN_VST128 3
#endif
// K / V ring stages (the kv-tile counter g indexes both), with the {64, 96} P releases below:
// d = 64 a 3-stage K ring (+2.5%), d = 128 a 3-stage V ring (+1.1-1.2%)
template <int HD> __host__ __device__ constexpr int kst_of() { return HD == 64 ? ATTN_KST64 : ATTN_KST; }
template <int HD> __host__ __device__ constexpr int vst_of() { return HD == 128 ? ATTN_VST128 : ATTN_VST; }
// per head dim: 128 rows x HD bf16 per tile (HD / 64 swizzle panels)
template <int HD> __host__ __device__ constexpr int tile_bytes() { return 128 * HD * 2; }
template <int HD> __host__ __device__ constexpr int smem_bytes() {
  return tile_bytes<HD>() * (NQ + kst_of<HD>() + vst_of<HD>()) + 1024 + 256;
}
constexpr int SM_WARPS_PER_TILE = 4;
// 12 warps = 3 warpgroups: softmax WG0/WG1, WG2 = 2 idle + producer + MMA (highest ids).
// setmaxnreg moves registers from WG2 to the softmax warpgroups (S row in registers).
constexpr int THREADS = (NQ * SM_WARPS_PER_TILE + 4) * 32;   // 384
#ifndef ATTN_REG_SOFTMAX
#define ATTN_REG_SOFTMAX 208
#endif
#ifndef ATTN_REG_OTHER
#define ATTN_REG_OTHER 80
#endif
// setmaxnreg.inc blocks until the CTA's pool (launch allocation: THREADS x 168) has the
// registers, so the split must fit in it or the softmax warps wait forever.
static_assert(2 * 128 * ATTN_REG_SOFTMAX + 128 * ATTN_REG_OTHER <= THREADS * 168, "register split exceeds the pool");
#ifndef ATTN_FAKE
#define ATTN_FAKE 0
#endif
#ifndef ATTN_POLY_MOD
#define ATTN_POLY_MOD 8
#endif
#ifndef ATTN_POLY_RES
#define ATTN_POLY_RES 1
#endif
constexpr int POLY_MOD = ATTN_POLY_MOD, POLY_RES = ATTN_POLY_RES;   // every POLY_MOD-th exp2 pair on the FMA-pipe polynomial
// d = 64 (half the MMA work per score): 3/8 of the pairs on the polynomial measured best
// (1/2: 723, 1/4: 744, 3/8: 758, 5/8: 664 TFLOP/s at B=8 H=24 N=4429 alone)
#ifndef ATTN_POLY_MOD64
#define ATTN_POLY_MOD64 8
#endif
#ifndef ATTN_POLY_RES64
#define ATTN_POLY_RES64 3
#endif
constexpr uint32_t COL_S = 0, COL_O = 256;
// split P arrive: bit c set = the softmax warps release P columns of kv [0, 32 (c + 1)) after
// chunk c (the MMA warp starts the PV on them); the last chunk is always released at the end
#ifndef ATTN_PMASK
#define ATTN_PMASK 6
#endif
#ifndef ATTN_PMASK64
#define ATTN_PMASK64 6
#endif
template <int HD> __host__ __device__ constexpr int pmask_of() { return (HD == 64 ? ATTN_PMASK64 : ATTN_PMASK) & 7; }
constexpr float RESCALE_THRESH = 8.0f;

DEVI void tmem_st16(uint32_t taddr, const uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
      "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
}
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
DEVI void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr)
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

DEVI float mufu_exp2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// 2^x on the FMA/ALU pipes: x = n + f, n = rint(x), f in [-0.5, 0.5];
// 2^f by a degree-3 minimax polynomial (max rel. error 2.1e-4 < bf16 half-ulp),
// 2^n by adding n to the exponent field.  x is clamped at -125 so the exponent
// of 2^f (126 or 127) minus n never underflows into the sign bit (2^-125 ~ 0).
DEVI float poly_exp2(float x) {
  x = fmaxf(x, -125.0f);
  const float t = x + 12582912.0f;             // 1.5 * 2^23: low mantissa bits = rint(x)
  const float f = x - (t - 12582912.0f);
  float p = fmaf(0.05485438f, f, 0.24182249f);
  p = fmaf(p, f, 0.69324851f);
  p = fmaf(p, f, 0.99998755f);
  return __int_as_float(__float_as_int(p) + (__float_as_int(t) << 23));
}

// Packed version for two arguments (f32x2 FADD/FFMA).
DEVI float2 poly_exp2x2(float2 x) {
  x.x = fmaxf(x.x, -125.0f);
  x.y = fmaxf(x.y, -125.0f);
  const float2 magic = make_float2(12582912.0f, 12582912.0f);
  const float2 t = __fadd2_rn(x, magic);
  const float2 f = __fadd2_rn(x, __fadd2_rn(magic, make_float2(-t.x, -t.y)));
  float2 p = __ffma2_rn(make_float2(0.05485438f, 0.05485438f), f, make_float2(0.24182249f, 0.24182249f));
  p = __ffma2_rn(p, f, make_float2(0.69324851f, 0.69324851f));
  p = __ffma2_rn(p, f, make_float2(0.99998755f, 0.99998755f));
  return make_float2(__int_as_float(__float_as_int(p.x) + (__float_as_int(t.x) << 23)),
                     __int_as_float(__float_as_int(p.y) + (__float_as_int(t.y) << 23)));
}

DEVI void named_bar_sync(int id, int nthreads) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory"); }

// Debug timeline (clock64 stamps of one CTA): compiled in only with -DATTN_TRACE=1 (a variant build,
// `python tools/variant.py trace attention_tc.cu -DATTN_TRACE=1`; enabled at run time by
// dit_debug_attention_trace).  Even predicated off, the stamps cost ~35 issue slots per softmax warp
// and kv tile on the critical path, so the product build has none.
__device__ long long* g_attn_trace = nullptr;
#ifndef ATTN_TRACE
#define ATTN_TRACE 0
#endif
#if ATTN_TRACE
#define TRACE_PTR (blockIdx.x == 0 ? g_attn_trace : nullptr)
#define TRACE(ev, j)                                                                       \
  do {                                                                                     \
    if (trace) trace[(ev) * 64 + ((j) & 63)] = clock64();                                  \
  } while (0)
#else
#define TRACE_PTR (static_cast<long long*>(nullptr))
#define TRACE(ev, j) \
  do {               \
  } while (0)
#endif

struct Maps {
  CUtensorMap q, k, v;   // 3D {HD, N, B*H}, box {64, 128, 1}
};

// S = Q K^T over a K = 64 head (4 MMAs of K = 16 inside one swizzle panel), warp-converged.
DEVI void tc_mma_ss_k64_warp(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc, uint32_t accum) {
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
      "@L tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %3, 1;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accum)
      : "memory");
}

// kv tiles of request b's (possibly ragged) joint sequence
// (RAGGED = false: the uniform-batch instantiation carries no per-request length at all)
template <bool RAGGED>
DEVI int seq_len_of(const AttnParams& p, int b) { return RAGGED ? p.seq_valid[b] : p.N; }
template <bool RAGGED>
DEVI int kv_tiles(const AttnParams& p, int b) { return (seq_len_of<RAGGED>(p, b) + BKV - 1) / BKV; }

// Persistent schedule of one CTA.  Work items (query block of 256, head, request) are dealt
// round-robin; with p.split_tail (opt-in) the items of the last, partial round are each split into
// S key ranges (S = min(4, CTAs / tail items) >= 2) so the tail round runs S times shorter: every
// CTA first walks its full-round items, then at most one (tail item, key part) unit.  A part
// leaves O / m / l of its range in p.tail_ws; the last part to finish (per query tile) merges the
// S partials in part order (deterministic) and writes the output.  The split changes the
// floating-point order of the tail items only -- results are reproducible run to run but no
// longer bitwise independent of the batch composition, hence opt-in (SURVEY.md §8 caveat on
// P3 / P9 / P10).
template <bool SPLIT>
struct TailSched {
  int total, G, full, rem, S;
  // (everything from the kernel parameters and gridDim -- uniform sources -- so the producer / MMA
  // warps keep the schedule in uniform registers after setmaxnreg)
  DEVI explicit TailSched(const AttnParams& p) : G((int)gridDim.x) {
    total = (p.N + NQ * BQ - 1) / (NQ * BQ) * p.H * p.B;
    rem = SPLIT ? total % G : 0;
    S = SPLIT ? min(min(4, G / max(rem, 1)), (p.N + BKV - 1) / BKV) : 1;   // the host launches SPLIT only when S >= 2
    full = SPLIT ? total - rem : total;
  }
  // k-th unit of this CTA (k = 0, 1, ... in order, w carried between calls): item w, key part (0
  // when not split); false when there is none
  DEVI bool unit(int k, int& w, int& part) const {
    if (!SPLIT) {   // (the plain walk, incremental: the same code as before the split existed)
      w = k == 0 ? (int)blockIdx.x : w + G;
      return w < total;
    }
    const int wf = (int)blockIdx.x + k * G;
    part = 0;
    if (wf < full) { w = wf; return true; }
    if (k != full / G || (int)blockIdx.x >= rem * S) return false;
    w = full + (int)blockIdx.x / S;
    part = (int)blockIdx.x % S;
    return true;
  }
  DEVI bool split(int w) const { return SPLIT && w >= full; }
  DEVI int kv0(int part, int nkv) const { return SPLIT ? part * nkv / S : 0; }
  DEVI int kv1(int part, int nkv) const { return SPLIT ? (part + 1) * nkv / S : nkv; }
};

template <int HD, bool RAGGED, bool SPLIT>
__global__ void __launch_bounds__(THREADS, 1) attn_tc_kernel(const __grid_constant__ Maps maps, const __grid_constant__ AttnParams p) {
  constexpr int TILE_BYTES = tile_bytes<HD>();
  constexpr int NPANEL = HD / 64;
  constexpr int KST = kst_of<HD>(), VST = vst_of<HD>(), PMASK = pmask_of<HD>();
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;                              // [NQ] tiles
  uint8_t* sK = smem + NQ * TILE_BYTES;
  uint8_t* sV = sK + KST * TILE_BYTES;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sV + VST * TILE_BYTES);
  uint64_t* q_full = bars;
  uint64_t* k_full = bars + 1;                    // [KST]
  uint64_t* k_empty = k_full + KST;               // [KST]
  uint64_t* v_full = k_empty + KST;               // [VST]
  uint64_t* v_empty = v_full + VST;               // [VST]
  uint64_t* s_full = v_empty + VST;               // [NQ]
  uint64_t* p_arr = s_full + NQ;                  // [NQ][4] P of kv chunk c (32 keys) released (PMASK)
  uint64_t* o_done = p_arr + 4 * NQ;              // [NQ]
  uint64_t* o_free = o_done + NQ;                 // [NQ] epilogue has read O (next work item may overwrite it)
  uint64_t* q_empty = o_free + NQ;                // last QK of a work item done (Q tiles reusable)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(q_empty + 1);
  uint32_t* tail_last = tmem_slot + 1;            // [NQ] split tail: this CTA merges the tile's parts

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int N = p.N;
  // ragged batch: request b's keys [seq_valid[b], N) are padding (masked; their K/V rows are
  // finite, so P = 0 contributes exactly nothing); query rows beyond are computed and ignored

  const int nqb = (N + NQ * BQ - 1) / (NQ * BQ);
  const int total = nqb * p.H * p.B;               // work items: (query block, head, request), block fastest

#ifndef ATTN_ROLE_BASE
#define ATTN_ROLE_BASE 2
#endif
  // producer / MMA warps: above every softmax warp (SMSP arbiter priority); ATTN_ROLE_BASE picks
  // which two of warps 8-11 (SMSPs 0-3) they take
#ifndef ATTN_ROLE_LOW
#define ATTN_ROLE_LOW 0
#endif
  // ATTN_ROLE_LOW = 1: the producer / MMA warpgroup takes warps 0-3 (LOWEST arbiter priority) and
  // the softmax warpgroups warps 4-11
  constexpr int SM_W0 = ATTN_ROLE_LOW ? 4 : 0;   // first softmax warp
  constexpr int W_LOAD = ATTN_ROLE_LOW ? ATTN_ROLE_BASE : NQ * SM_WARPS_PER_TILE + ATTN_ROLE_BASE, W_MMA = W_LOAD + 1;
  if (warp == W_LOAD && lane == 0) {
    tma_prefetch_desc(&maps.q);
    tma_prefetch_desc(&maps.k);
    tma_prefetch_desc(&maps.v);
    mbar_init(q_full, 1);
    mbar_init(q_empty, 1);
    for (int i = 0; i < KST; ++i) {
      mbar_init(&k_full[i], 1);
      mbar_init(&k_empty[i], 1);
    }
    for (int i = 0; i < VST; ++i) {
      mbar_init(&v_full[i], 1);
      mbar_init(&v_empty[i], 1);
    }
    for (int i = 0; i < NQ; ++i) {
      mbar_init(&s_full[i], 1);
      for (int c = 0; c < 4; ++c) mbar_init(&p_arr[4 * i + c], SM_WARPS_PER_TILE);
      mbar_init(&o_done[i], 1);
      mbar_init(&o_free[i], SM_WARPS_PER_TILE);
    }
    fence_barrier_init();
  }
  if (warp == W_MMA) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  if (ATTN_ROLE_LOW ? warp < SM_W0 : warp >= NQ * SM_WARPS_PER_TILE) {
   asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(ATTN_REG_OTHER));
   long long* const trace = TRACE_PTR;   // loaded after setmaxnreg (no spill)
   if (warp == W_LOAD) {
    if (lane == 0) {
      const TailSched<SPLIT> sched(p);   // (built after setmaxnreg: no spills)
      int g = 0, it = 0;                           // kv-tile counter (ring position), item counter
      for (int w = 0, part = 0; sched.unit(it, w, part); ++it) {
        const int bh = w / nqb, q0 = (w - bh * nqb) * (NQ * BQ);
        const int nkv_all = kv_tiles<RAGGED>(p, bh / p.H);
        const int j0 = sched.split(w) ? sched.kv0(part, nkv_all) : 0;
        const int nkv = sched.split(w) ? sched.kv1(part, nkv_all) - j0 : nkv_all;
        if (it > 0) mbar_wait(q_empty, (it - 1) & 1);
        mbar_expect_tx(q_full, NQ * TILE_BYTES);
        for (int t = 0; t < NQ; ++t)
          for (int pn = 0; pn < NPANEL; ++pn)
            tma_load_3d(&maps.q, q_full, sQ + t * TILE_BYTES + pn * PANEL, pn * 64, q0 + t * BQ, bh);
        for (int j = 0; j < nkv; ++j, ++g) {
          const int st = g % KST, sv = g % VST;
          const uint32_t ph = (g / KST) & 1, pv = (g / VST) & 1;
          mbar_wait(&k_empty[st], ph ^ 1);
          if (it == 0) TRACE(0, j);
          mbar_expect_tx(&k_full[st], TILE_BYTES);
          for (int pn = 0; pn < NPANEL; ++pn)
            tma_load_3d(&maps.k, &k_full[st], sK + st * TILE_BYTES + pn * PANEL, pn * 64, (j0 + j) * BKV, bh);
          mbar_wait(&v_empty[sv], pv ^ 1);
          if (it == 0) TRACE(1, j);
          mbar_expect_tx(&v_full[sv], TILE_BYTES);
          for (int pn = 0; pn < NPANEL; ++pn)
            tma_load_3d(&maps.v, &v_full[sv], sV + sv * TILE_BYTES + pn * PANEL, pn * 64, (j0 + j) * BKV, bh);
        }
      }
    }
  } else if (warp == W_MMA) {
    // The whole warp walks the schedule (waits included); inside each MMA/commit asm block
    // one lane is elected, so every operand is warp-uniform (see tc_mma_ss_k128_warp).
    constexpr uint32_t idesc_qk = idesc_bf16_f32(BQ, BKV);
    constexpr uint32_t idesc_pv = idesc_bf16_f32(BQ, HD) | (1u << 16);   // B (V) MN-major
    const uint32_t tm = __shfl_sync(0xffffffffu, tmem, 0);
    bool tr = false;
    // g: global kv-tile index (K/V ring stage + phase, and the s/p/o barrier phases)
    auto issue_qk = [&](int t, int g, int j) {
      const int st = g % KST;
      if (t == 0 && lane == 0 && tr) TRACE(14, j);
      if (t == 0) mbar_wait(&k_full[st], (g / KST) & 1);
      if (t == 0 && lane == 0 && tr) TRACE(2, j);
      tc_fence_after();
      if constexpr (HD == 128)
        tc_mma_ss_k128_warp<PANEL>(tm + COL_S + t * 128, smem_desc_k_sw128(smem_u32(sQ + t * TILE_BYTES)),
                                   smem_desc_k_sw128(smem_u32(sK + st * TILE_BYTES)), idesc_qk, 0);
      else
        tc_mma_ss_k64_warp(tm + COL_S + t * 128, smem_desc_k_sw128(smem_u32(sQ + t * TILE_BYTES)),
                           smem_desc_k_sw128(smem_u32(sK + st * TILE_BYTES)), idesc_qk, 0);
      tc_commit_warp(&s_full[t]);
      if (t == NQ - 1) tc_commit_warp(&k_empty[st]);
    };
    auto issue_pv = [&](int t, int g, int j, int it, int nkv) {
      const int st = g % VST;
      if (lane == 0 && tr) TRACE(15 + t, j);
      constexpr int c_first = (PMASK & 1) ? 0 : (PMASK & 2) ? 1 : (PMASK & 4) ? 2 : 3;
      mbar_wait(&p_arr[4 * t + c_first], g & 1);
      if (lane == 0 && tr) TRACE(3 + t, j);
      if (j == 0 && it > 0) mbar_wait(&o_free[t], (it - 1) & 1);   // previous item's O read out
      if (t == 0) mbar_wait(&v_full[st], (g / VST) & 1);
      if (t == 0 && lane == 0 && tr) TRACE(5, j);
      tc_fence_after();
      {
        // P is released in chunks of 32 keys (PMASK); each chunk's two K = 16 MMAs wait for it
        const uint64_t vdesc = desc_mn_sw128(smem_u32(sV + st * TILE_BYTES), PANEL);
        const uint32_t od = tm + COL_O + t * HD, pa = tm + COL_S + t * 128;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          if (c > c_first && (c == 3 || ((PMASK >> (c - 1)) & 1))) {   // a new release point covers chunk c
            int e = c;
            while (e < 3 && !((PMASK >> e) & 1)) ++e;
            mbar_wait(&p_arr[4 * t + e], g & 1);
            tc_fence_after();
          }
#pragma unroll
          for (int kk = 2 * c; kk < 2 * c + 2; ++kk)
            tc_mma_ts_warp(od, pa + kk * 8, vdesc + (uint64_t)(kk * 128), idesc_pv, (j | kk) != 0);
        }
      }
      // O of this work item is final after its last PV: the only phase anyone waits on (the
      // epilogue).  Earlier PVs need no barrier: the commit of the next QK into S_t covers them.
      if (j == nkv - 1) tc_commit_warp(&o_done[t]);
      if (t == NQ - 1) tc_commit_warp(&v_empty[st]);
    };
    const TailSched<SPLIT> sched(p);
    int g = 0, it = 0;
    for (int w = 0, part = 0; sched.unit(it, w, part); ++it) {
      const int nkv_all = kv_tiles<RAGGED>(p, (w / nqb) / p.H);
      const int nkv = sched.split(w) ? sched.kv1(part, nkv_all) - sched.kv0(part, nkv_all) : nkv_all;
      tr = trace != nullptr && it == 0;
      mbar_wait(q_full, it & 1);
      issue_qk(0, g, 0);
      issue_qk(1, g, 0);
      if (nkv == 1) tc_commit_warp(q_empty);
      for (int j = 0; j < nkv; ++j) {
        issue_pv(0, g + j, j, it, nkv);
        if (j + 1 < nkv) issue_qk(0, g + j + 1, j + 1);
        issue_pv(1, g + j, j, it, nkv);
        if (j + 1 < nkv) {
          issue_qk(1, g + j + 1, j + 1);
          if (j + 2 == nkv) tc_commit_warp(q_empty);   // last QK of this item issued
        }
      }
      g += nkv;
    }
   }
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(ATTN_REG_SOFTMAX));
    long long* const trace = TRACE_PTR;
    // softmax: warps 0-3 own query tile 0, warps 4-7 tile 1; one query row per thread
    // (TMEM lane = row), all 128 score columns of it in registers: no cross-warp exchange.
    const int t = (warp - SM_W0) >> 2;
    const int wq = warp & 3;                       // TMEM lane quarter
    const int row = wq * 32 + lane;
    const uint32_t lane_base = (uint32_t)(wq * 32) << 16;
    const uint32_t colS = tmem + lane_base + COL_S + t * 128;
    const uint32_t colO = tmem + lane_base + COL_O + t * HD;
    const float sl2 = p.scale_log2;
    const TailSched<SPLIT> sched(p);
    int g = 0, it = 0;
    for (int w = 0, part = 0; sched.unit(it, w, part); ++it) {
      const bool tr = trace != nullptr && it == 0 && lane == 0 && wq == 0;
      const int bh = w / nqb, q0 = (w - bh * nqb) * (NQ * BQ);
      const int b = bh / p.H, h = bh - b * p.H;
      const int nkv_all = kv_tiles<RAGGED>(p, b);
      const bool split = sched.split(w);
      const int j0 = split ? sched.kv0(part, nkv_all) : 0;
      const int Nv = seq_len_of<RAGGED>(p, b) - j0 * BKV, nkv = split ? sched.kv1(part, nkv_all) - j0 : nkv_all;
      float m_used = -INFINITY, l = 0.f;
      for (int j = 0; j < nkv; ++j, ++g) {
        mbar_wait(&s_full[t], g & 1);
        if (tr) TRACE(6 + t, j);
        tc_fence_after();
#if ATTN_FAKE
        {  // timing experiment: no softmax math (ATTN_FAKE=1: no S read either)
          uint32_t z[16];
#pragma unroll
          for (int e = 0; e < 16; ++e) z[e] = 0x3f803f80u;
          if (ATTN_FAKE == 2) {
            uint32_t sr[32];
            for (int c = 0; c < 4; ++c) tmem_ld32(colS + c * 32, sr);
            tmem_ld_wait();
            if (sr[lane] == 0x12345678u) z[0] = 0;
          }
#pragma unroll
          for (int c = 0; c < 4; ++c) tmem_st16(colS + c * 16, z);
          tmem_st_wait();
          tc_fence_before();
          __syncwarp();
          if (tr) TRACE(8 + t, j);
          for (int c = 0; c < 4; ++c)
            if (lane == 0 && (c == 3 || ((PMASK >> c) & 1))) mbar_arrive(&p_arr[4 * t + c]);
          l = 1.f;
          continue;
        }
#endif
        uint32_t sr[128];
#pragma unroll
        for (int c = 0; c < 4; ++c) tmem_ld32(colS + c * 32, *reinterpret_cast<uint32_t(*)[32]>(&sr[32 * c]));
        tmem_ld_wait();
        if (tr) TRACE(10 + t, j);
        const int kv_valid = Nv - j * BKV;   // (Nv counts from this unit's first key tile)
        if (kv_valid < BKV) {
#pragma unroll
          for (int e = 0; e < 128; ++e)
            if (e >= kv_valid) sr[e] = __float_as_uint(-INFINITY);
        }
        float m8[8];
#pragma unroll
        for (int a = 0; a < 8; ++a) m8[a] = fmaxf(__uint_as_float(sr[2 * a]), __uint_as_float(sr[2 * a + 1]));
#pragma unroll
        for (int e = 16; e < 128; e += 16)
#pragma unroll
          for (int a = 0; a < 8; ++a)
            m8[a] = fmaxf(m8[a], fmaxf(__uint_as_float(sr[e + 2 * a]), __uint_as_float(sr[e + 2 * a + 1])));
        const float mx = fmaxf(fmaxf(fmaxf(m8[0], m8[1]), fmaxf(m8[2], m8[3])),
                               fmaxf(fmaxf(m8[4], m8[5]), fmaxf(m8[6], m8[7]))) * sl2;
        if (tr) TRACE(12 + t, j);
        const bool need = mx > m_used + RESCALE_THRESH;
        const float m_new = need ? mx : m_used;
        if (j > 0 && __any_sync(0xffffffff, need)) {
          const float alpha = need ? mufu_exp2(m_used - m_new) : 1.0f;
          // O_t holds PV(t, j-1): complete, since S_t(j) (waited above) was committed after it
#pragma unroll 1
          for (int c = 0; c < HD / 16; ++c) {
            uint32_t r[16];
            tmem_ld16(colO + c * 16, r);
            tmem_ld_wait();
#pragma unroll
            for (int e = 0; e < 16; ++e) r[e] = __float_as_uint(__uint_as_float(r[e]) * alpha);
            tmem_st16(colO + c * 16, r);
          }
          tmem_st_wait();
          l *= alpha;
        }
        m_used = m_new;
        const float2 sl2v = make_float2(sl2, sl2), nm = make_float2(-m_used, -m_used);
        // exponentials (kept in sr as fp32 for the row sum); P (bf16 pairs) over the first 64
        // columns of this row's S, 16 at a time
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          uint32_t r[16];
#pragma unroll
          for (int e = 0; e < 16; ++e) {
            const float2 x = __ffma2_rn(make_float2(__uint_as_float(sr[32 * c + 2 * e]), __uint_as_float(sr[32 * c + 2 * e + 1])), sl2v, nm);
            float2 pp;
            constexpr int PM = HD == 64 ? ATTN_POLY_MOD64 : POLY_MOD, PR = HD == 64 ? ATTN_POLY_RES64 : POLY_RES;
            if ((e % PM) >= PM - PR) {
              pp = poly_exp2x2(x);                   // POLY_RES/POLY_MOD of the pairs on the FMA pipe
            } else {
              pp.x = mufu_exp2(x.x);
              pp.y = mufu_exp2(x.y);
            }
            sr[32 * c + 2 * e] = __float_as_uint(pp.x);
            sr[32 * c + 2 * e + 1] = __float_as_uint(pp.y);
            r[e] = pack_bf16(pp.x, pp.y);
          }
          tmem_st16(colS + c * 16, r);
          if (c < 3 && ((PMASK >> c) & 1)) {   // kv [0, 32 (c + 1)) of P are in TMEM: let the PV MMA start on them
            tmem_st_wait();
            tc_fence_before();
            __syncwarp();
            if (tr) TRACE(8 + t, j);
            if (trace != nullptr && it == 0 && lane == 0 && t == 0 && wq > 0) TRACE(16 + wq, j);   // arrive skew
            if (lane == 0) mbar_arrive(&p_arr[4 * t + c]);
          }
        }
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        uint64_t tok = 0;
        if (lane == 0)
          asm volatile("mbarrier.arrive.shared::cta.b64 %0, [%1];" : "=l"(tok) : "r"(smem_u32(&p_arr[4 * t + 3])) : "memory");
        // row sum off the critical path (the PV MMA is already running): seeded with a zero
        // derived from the arrive's state token, so ptxas cannot hoist it above the arrive
        tok = __shfl_sync(0xffffffffu, tok, 0);
        const float z = tok == ~0ull ? 1.0f : 0.0f;
        float2 acc0 = make_float2(z, z), acc1 = make_float2(z, z);
#pragma unroll
        for (int e = 0; e < 128; e += 4) {
          acc0 = __fadd2_rn(acc0, make_float2(__uint_as_float(sr[e]), __uint_as_float(sr[e + 1])));
          acc1 = __fadd2_rn(acc1, make_float2(__uint_as_float(sr[e + 2]), __uint_as_float(sr[e + 3])));
        }
        l += (acc0.x + acc0.y) + (acc1.x + acc1.y);
      }
      // epilogue: read O out of TMEM, release it to the next work item, then O / l -> bf16
      // (one 256-byte output row per thread)
      // (the output address first: its temporaries die before the 128 O registers go live)
      const int n = q0 + t * BQ + row;
      uint4* dst = n < N ? reinterpret_cast<uint4*>(attn_out_addr(p, b, n, h, HD)) : nullptr;
      mbar_wait(&o_done[t], it & 1);   // one phase per work item
      tc_fence_after();
      uint32_t o[HD];
#pragma unroll
      for (int c = 0; c < HD / 32; ++c) tmem_ld32(colO + c * 32, *reinterpret_cast<uint32_t(*)[32]>(&o[32 * c]));
      tmem_ld_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&o_free[t]);
      if (split) {
        // split tail: leave this part's O (unnormalised, relative to m_used) and (m_used, l), then
        // the last of the S parts of this query tile merges them in part order
        const int ti = (w - sched.full) * NQ + t;
        float* mine = p.tail_ws + ((size_t)((w - sched.full) * sched.S + part) * NQ + t) * BQ * (HD + 4) + (size_t)row * (HD + 4);
#pragma unroll
        for (int q = 0; q < HD / 4; ++q)
          reinterpret_cast<float4*>(mine)[q] = make_float4(__uint_as_float(o[4 * q]), __uint_as_float(o[4 * q + 1]),
                                                           __uint_as_float(o[4 * q + 2]), __uint_as_float(o[4 * q + 3]));
        reinterpret_cast<float4*>(mine)[HD / 4] = make_float4(m_used, l, 0.f, 0.f);
        __threadfence();
        named_bar_sync(1 + t, BQ);
        if (row == 0) tail_last[t] = atomicAdd(p.tail_cnt + ti, 1u) == (uint32_t)sched.S - 1 ? 1u : 0u;
        named_bar_sync(1 + t, BQ);
        if (tail_last[t] == 0u) continue;
        __threadfence();
        if (row == 0) p.tail_cnt[ti] = 0;   // (next launch)
        const float* base = p.tail_ws + ((size_t)((w - sched.full) * sched.S) * NQ + t) * BQ * (HD + 4) + (size_t)row * (HD + 4);
        const size_t pstride = (size_t)NQ * BQ * (HD + 4);   // floats between consecutive parts
        float f[4], M = -INFINITY, lt = 0.f;
#pragma unroll
        for (int s2 = 0; s2 < 4; ++s2) {
          f[s2] = -INFINITY;
          if (s2 < sched.S) {
            const float4 ml = __ldcg(reinterpret_cast<const float4*>(base + s2 * pstride) + HD / 4);
            f[s2] = ml.x;
            M = fmaxf(M, ml.x);
          }
        }
#pragma unroll
        for (int s2 = 0; s2 < 4; ++s2) {
          f[s2] = f[s2] == -INFINITY ? 0.f : exp2f(f[s2] - M);
          if (s2 < sched.S) lt = fmaf(f[s2], __ldcg(base + s2 * pstride + HD + 1), lt);
        }
#pragma unroll
        for (int q = 0; q < HD / 4; ++q) {
          float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
          for (int s2 = 0; s2 < 4; ++s2) {
            if (s2 < sched.S) {
              const float4 v4 = __ldcg(reinterpret_cast<const float4*>(base + s2 * pstride) + q);
              acc.x = fmaf(f[s2], v4.x, acc.x);
              acc.y = fmaf(f[s2], v4.y, acc.y);
              acc.z = fmaf(f[s2], v4.z, acc.z);
              acc.w = fmaf(f[s2], v4.w, acc.w);
            }
          }
          o[4 * q] = __float_as_uint(acc.x);
          o[4 * q + 1] = __float_as_uint(acc.y);
          o[4 * q + 2] = __float_as_uint(acc.z);
          o[4 * q + 3] = __float_as_uint(acc.w);
        }
        l = lt;
      }
      if (dst != nullptr) {
        const float inv = 1.0f / l;
#pragma unroll
        for (int q = 0; q < HD / 8; ++q) {
          uint4 u;
          u.x = pack_bf16(__uint_as_float(o[8 * q + 0]) * inv, __uint_as_float(o[8 * q + 1]) * inv);
          u.y = pack_bf16(__uint_as_float(o[8 * q + 2]) * inv, __uint_as_float(o[8 * q + 3]) * inv);
          u.z = pack_bf16(__uint_as_float(o[8 * q + 4]) * inv, __uint_as_float(o[8 * q + 5]) * inv);
          u.w = pack_bf16(__uint_as_float(o[8 * q + 6]) * inv, __uint_as_float(o[8 * q + 7]) * inv);
          dst[q] = u;
        }
        if (p.split == 3) __threadfence_system();   // fused exchange: peer stores, system scope
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == W_MMA) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

}  // namespace attn_tc


cudaError_t attention_set_trace(long long* buf) {
  return cudaMemcpyToSymbol(attn_tc::g_attn_trace, &buf, sizeof(buf));
}

template <int HD, bool RAGGED>
static cudaError_t attention_tc_launch_hd(const AttnParams& p, cudaStream_t s) {
  using namespace attn_tc;
  constexpr int SMEM = smem_bytes<HD>();
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(attn_tc_kernel<HD, RAGGED, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
    if (e == cudaSuccess && !RAGGED)
      e = cudaFuncSetAttribute(attn_tc_kernel<HD, RAGGED, !RAGGED>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
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
  static int sms = 0;
  if (sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  // persistent: one CTA per SM walks work items (query block fastest, so the CTAs running at
  // the same time share each head's K/V in L2)
  const int total = (p.N + NQ * BQ - 1) / (NQ * BQ) * p.H * p.B;
  const int G = std::min(total, sms);
  // split tail (opt-in): when the last round is at most half full (S >= 2 key parts per tail item);
  // the split instantiation runs the full rounds as fast as the plain one (measured: d = 128
  // 1341 vs 1341 TF/s at B = 8, H = 24, N = 4608) and shortens the tail round S-fold
  bool split = false;
  if (!RAGGED && p.split_tail && p.tail_ws && p.tail_cnt && total > G && total % G != 0) {
    const int rem = total % G, nkv = (p.N + BKV - 1) / BKV;
    const int S = std::min(std::min(4, G / rem), nkv);
    split = S >= 2 && rem * S <= ATTN_TAIL_UNITS;
  }
  if (split)
    attn_tc_kernel<HD, RAGGED, !RAGGED><<<dim3(G), THREADS, SMEM, s>>>(m, p);
  else
    attn_tc_kernel<HD, RAGGED, false><<<dim3(G), THREADS, SMEM, s>>>(m, p);
  return cudaGetLastError();
}

cudaError_t attention_tc_launch(const AttnParams& p, cudaStream_t s) {
  if (p.seq_valid != nullptr)
    return p.d == 64 ? attention_tc_launch_hd<64, true>(p, s) : attention_tc_launch_hd<128, true>(p, s);
  return p.d == 64 ? attention_tc_launch_hd<64, false>(p, s) : attention_tc_launch_hd<128, false>(p, s);
}

cudaError_t attention_tc_preload() { return preload_module_of(reinterpret_cast<const void*>(&attn_tc::attn_tc_kernel<128, false, false>)); }

}  // namespace dit
