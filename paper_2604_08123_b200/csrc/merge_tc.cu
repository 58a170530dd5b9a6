// merge_tc.cu -- LoRA weight patching on the tensor cores:
//   W'[o][i] = bf16(W[o][i] + scale * sum_k B[o][k] A[k][i])
// One CTA per 128 x 128 tile of W: TMA brings the B rows (K-major), the A columns (MN-major)
// and the W tile (all SWIZZLE_128B) into shared memory, one thread issues the rank-r product
// as tcgen05 MMAs into 128 TMEM columns, every thread then owns one tile row: it reads its
// accumulator row from TMEM, adds it into the W row in shared memory, and one thread TMA-stores
// the patched tile.  Global traffic is the W read + W' write (the factors are L2-resident), all
// of it as TMA bulk copies; the product costs no CUDA-core time.
#include <algorithm>

#include "common.cuh"
#include "kernels.h"

namespace dit {
namespace merge_tc {

constexpr int TILE = 128, THREADS = 128;

// MN-major SWIZZLE_128B descriptor (64-element rows along N, 8-row core groups along K 1024 B
// apart, next 64-wide N panel at LBO).
DEVI uint64_t desc_mn_sw128(uint32_t saddr, uint32_t lbo_bytes) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo_bytes >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

DEVI void tma_store_2d(const void* desc, const void* smem, int c0, int c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(desc)),
               "r"(smem_u32(smem)), "r"(c0), "r"(c1)
               : "memory");
}

struct Maps {
  CUtensorMap w, out;   // [out][in], box {64, 128}
  CUtensorMap b;        // B factor [out][ra], box {64, 128}
  CUtensorMap a;        // A factor [ra][in], box {64, ra}
};

template <int RA>
constexpr int smem_bytes() { return (RA / 64) * 16384 + 2 * RA * 128 + 32768 + 1024 + 64; }

// One adapted linear of the merge: its maps live in device memory (64-byte aligned, written
// by the host before the launch), tiles [tile_begin, tile_begin + tiles) of the global list.
// elem_base: index of this linear's element [0][0] in the concatenation of all adapted linears
// (the in-place merge's undo-log address space); w: the linear's weights (exception restore).
struct alignas(64) Job {
  Maps m;
  int tile_begin, tiles, tiles_n;
  float scale;
  long long elem_base;
  uint16_t* w;
  int cols;
};

// Modes of the one kernel (DESIGN.md §7 "in-place hot patch"):
//   MERGE_COPY    W' = bf16(W + s BA) stored to the job's `out` map (a second copy)
//   COUNT         no store: count the elements whose W the inverse below cannot recover
//   MERGE_INPLACE W' stored over W itself, and each unrecoverable element logged as
//                 (value W << 48 | element index) into the undo log
//   RESTORE       W = bf16(W' - s BA) over W' (the logged elements are then rewritten exactly
//                 by restore_log_kernel)
// The inverse is exact except where rounding W + d to bf16 lost bits -- W' in a higher binade
// than W (small |W| against |d|) or a rounding tie; the log holds exactly those elements, so
// MERGE_INPLACE + RESTORE returns every weight bit for bit.  d = s * acc is the same fp32 product in
// every mode (the tensor-core product of a tile is deterministic).
enum Mode { MERGE_COPY = 0, COUNT = 1, MERGE_INPLACE = 2, RESTORE = 3 };

DEVI uint16_t bf16_bits_rn(float x) { return (uint16_t)(pack_bf16(x, 0.f) & 0xffffu); }

// Persistent: each CTA walks the global tile list of ALL adapted linears (one launch per
// merge: no per-module launch tails), one TMEM allocation and one barrier pair per CTA,
// phases tracked per tile.
template <int RA, int MODE>
__global__ void __launch_bounds__(THREADS) merge_tc_kernel(const Job* __restrict__ jobs, int njobs, int total,
                                                           unsigned long long* __restrict__ log,
                                                           unsigned long long* __restrict__ log_count) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  constexpr int KP = RA / 64;
  uint8_t* sB = smem;                    // KP x [128 rows][64 k]
  uint8_t* sA = sB + KP * 16384;         // 2 x [RA k][64 cols]
  uint8_t* sW = sA + 2 * RA * 128;       // 2 x [128 rows][64 cols]
  uint64_t* bars = reinterpret_cast<uint64_t*>(sW + 32768);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + 2);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc<128>(tslot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;
  int it = 0;
  for (int t = blockIdx.x; t < total; t += gridDim.x, ++it) {
    int lo = 0, hi = njobs - 1;           // the job holding tile t
    while (lo < hi) {
      const int mid = (lo + hi + 1) / 2;
      if (jobs[mid].tile_begin <= t) lo = mid; else hi = mid - 1;
    }
    const Job& J = jobs[lo];
    const int lt = t - J.tile_begin;
    const int c0 = (lt % J.tiles_n) * TILE, r0 = (lt / J.tiles_n) * TILE;
    const float scale = J.scale;
    if (threadIdx.x == 0) {
      mbar_expect_tx(&bars[0], KP * 16384 + 2 * RA * 128 + 32768);
      for (int p = 0; p < KP; ++p) tma_load_2d(&J.m.b, &bars[0], sB + p * 16384, p * 64, r0);
      for (int p = 0; p < 2; ++p) tma_load_2d(&J.m.a, &bars[0], sA + p * RA * 128, c0 + p * 64, 0);
      for (int p = 0; p < 2; ++p) tma_load_2d(&J.m.w, &bars[0], sW + p * 16384, c0 + p * 64, r0);
      mbar_wait(&bars[0], it & 1);
      tc_fence_after();
      constexpr uint32_t idesc = idesc_bf16_f32(TILE, TILE) | (1u << 16);   // A K-major, B MN-major
      const uint64_t bdesc = desc_mn_sw128(smem_u32(sA), RA * 128);
#pragma unroll
      for (int k = 0; k < RA / 16; ++k)
        tc_mma_f16(tmem, smem_desc_k_sw128(smem_u32(sB + (k / 4) * 16384)) + 2 * (k % 4),
                   bdesc + (uint64_t)(k * 128), idesc, k > 0);
      tc_commit(&bars[1]);
    }
    __syncwarp();
    // every thread: one tile row (TMEM lane), 4 x 32 accumulator columns into the swizzled W row
    mbar_wait(&bars[1], it & 1);
    tc_fence_after();
    const int row = warp * 32 + lane;
    const uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16);
    unsigned exc = 0;   // unrecoverable elements of this thread's row
    unsigned long long lbase = 0;
    if (MODE == MERGE_INPLACE) {
      // count this row's log entries first (the same arithmetic as below, nothing written), so a
      // warp reserves its log range with ONE atomic per tile instead of one per entry
#pragma unroll 1
      for (int cc = 0; cc < 4; ++cc) {
        uint32_t acc[32];
        tmem_ld32(taddr + cc * 32, acc);
        tmem_ld_wait();
        const uint8_t* prow = sW + (cc / 2) * 16384 + row * 128;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int j = (cc % 2) * 4 + q;
          const uint4 w = *reinterpret_cast<const uint4*>(prow + ((j ^ (row & 7)) << 4));
          const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float d0 = scale * __uint_as_float(acc[q * 8 + 2 * e]);
            const float d1 = scale * __uint_as_float(acc[q * 8 + 2 * e + 1]);
            const uint32_t np = pack_bf16(__fadd_rn(bf16_lo(ws[e]), d0), __fadd_rn(bf16_hi(ws[e]), d1));
            const uint32_t inv = pack_bf16(__fsub_rn(bf16_lo(np), d0), __fsub_rn(bf16_hi(np), d1));
            exc += ((inv & 0xffffu) != (ws[e] & 0xffffu)) + ((inv >> 16) != (ws[e] >> 16));
          }
        }
      }
      unsigned incl = exc;   // inclusive warp scan
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
      }
      const unsigned total = __shfl_sync(0xffffffffu, incl, 31);
      unsigned long long wb = 0;
      if (lane == 31 && total) wb = atomicAdd(log_count, (unsigned long long)total);
      lbase = __shfl_sync(0xffffffffu, wb, 31) + (incl - exc);
    }
#pragma unroll
    for (int cc = 0; cc < 4; ++cc) {
      uint32_t acc[32];
      tmem_ld32(taddr + cc * 32, acc);
      tmem_ld_wait();
      uint8_t* prow = sW + (cc / 2) * 16384 + row * 128;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int j = (cc % 2) * 4 + q;                                       // logical 16-byte chunk
        uint4* pc = reinterpret_cast<uint4*>(prow + ((j ^ (row & 7)) << 4));   // SWIZZLE_128B
        uint4 w = *pc;
        uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float d0 = scale * __uint_as_float(acc[q * 8 + 2 * e]);
          const float d1 = scale * __uint_as_float(acc[q * 8 + 2 * e + 1]);
          if (MODE == RESTORE) {
            ws[e] = pack_bf16(__fsub_rn(bf16_lo(ws[e]), d0), __fsub_rn(bf16_hi(ws[e]), d1));
          } else {
            const uint32_t np = pack_bf16(__fadd_rn(bf16_lo(ws[e]), d0), __fadd_rn(bf16_hi(ws[e]), d1));
            if (MODE == COUNT || MODE == MERGE_INPLACE) {
              // what RESTORE will compute from W' -- differs from W only where bits were lost
              const uint32_t inv = pack_bf16(__fsub_rn(bf16_lo(np), d0), __fsub_rn(bf16_hi(np), d1));
#pragma unroll
              for (int h = 0; h < 2; ++h) {
                const uint32_t wv = (ws[e] >> (16 * h)) & 0xffffu;
                if (((inv >> (16 * h)) & 0xffffu) != wv) {
                  if (MODE == COUNT) {
                    ++exc;
                  } else {
                    const int col = c0 + (cc / 2) * 64 + j * 8 + 2 * e + h;
                    const long long idx = J.elem_base + (long long)(r0 + row) * J.cols + col;
                    log[lbase++] = ((unsigned long long)wv << 48) | (unsigned long long)idx;
                  }
                }
              }
            }
            ws[e] = np;
          }
        }
        if (MODE != COUNT) *pc = make_uint4(ws[0], ws[1], ws[2], ws[3]);
      }
    }
    if (MODE == COUNT) {
      exc = __reduce_add_sync(0xffffffffu, exc);
      if (lane == 0 && exc) atomicAdd(log_count, (unsigned long long)exc);
    }
    fence_async_shared();   // the patched rows (generic proxy) -> the TMA store (async proxy)
    tc_fence_before();
    __syncthreads();        // (also: every thread's TMEM reads are done before the next MMA)
    if (MODE != COUNT && threadIdx.x == 0) {
      for (int p = 0; p < 2; ++p) tma_store_2d(&J.m.out, sW + p * 16384, c0 + p * 64, r0);
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");   // sW reusable
    }
    __syncthreads();
    tc_fence_after();
  }
  if (warp == 0) tmem_dealloc<128>(tmem);
}

// Rewrite the logged elements (after RESTORE): entry = value << 48 | global element index.
__global__ void restore_log_kernel(const Job* __restrict__ jobs, int njobs, const unsigned long long* __restrict__ log,
                                   unsigned long long n) {
  for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < n;
       i += (unsigned long long)gridDim.x * blockDim.x) {
    const unsigned long long e = log[i];
    const long long idx = (long long)(e & ((1ull << 48) - 1));
    int lo = 0, hi = njobs - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) / 2;
      if (jobs[mid].elem_base <= idx) lo = mid; else hi = mid - 1;
    }
    jobs[lo].w[idx - jobs[lo].elem_base] = (uint16_t)(e >> 48);
  }
}

}  // namespace merge_tc

size_t merge_job_bytes() { return sizeof(merge_tc::Job); }

bool merge_job_fill(void* job, const CUtensorMap& w_map, const CUtensorMap& out_map, const void* A, const void* Bm,
                    int rows, int cols, int ra, float scale, int tile_begin, const void* w, long long elem_base) {
  using namespace merge_tc;
  Job* J = static_cast<Job*>(job);
  J->m.w = w_map;
  J->m.out = out_map;
  J->w = static_cast<uint16_t*>(const_cast<void*>(w));
  J->elem_base = elem_base;
  J->cols = cols;
  if (!make_tmap_2d(&J->m.b, Bm, ra, rows, (uint64_t)ra * 2, 64, 128) ||
      !make_tmap_2d(&J->m.a, A, cols, ra, (uint64_t)cols * 2, 64, ra))
    return false;
  J->tiles_n = (cols + TILE - 1) / TILE;
  J->tiles = J->tiles_n * ((rows + TILE - 1) / TILE);
  J->tile_begin = tile_begin;
  J->scale = scale;
  return true;
}

int merge_job_tiles(const void* job) { return static_cast<const merge_tc::Job*>(job)->tiles; }

template <int RA, int MODE>
static cudaError_t merge_launch_ra(const merge_tc::Job* jobs, int njobs, int total_tiles, int grid,
                                   unsigned long long* log, unsigned long long* log_count, cudaStream_t s) {
  using namespace merge_tc;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(merge_tc_kernel<RA, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         smem_bytes<RA>());
    if (e != cudaSuccess) return e;
    attr = true;
  }
  merge_tc_kernel<RA, MODE><<<grid, THREADS, smem_bytes<RA>(), s>>>(jobs, njobs, total_tiles, log, log_count);
  return cudaGetLastError();
}

cudaError_t lora_merge_tc_launch(const void* jobs_dev, int njobs, int total_tiles, int ra, int num_sms,
                                 cudaStream_t s, int mode, unsigned long long* log, unsigned long long* log_count) {
  using namespace merge_tc;
  if ((ra != 64 && ra != 128) || njobs < 1 || total_tiles < 1 || mode < 0 || mode > 3) return cudaErrorInvalidValue;
  const Job* jobs = static_cast<const Job*>(jobs_dev);
  const int per_sm = ra == 64 ? 3 : 2;
  const int grid = std::min(total_tiles, num_sms * per_sm);
#define MERGE_CASE(R, M) \
  if (ra == R && mode == M) return merge_launch_ra<R, M>(jobs, njobs, total_tiles, grid, log, log_count, s);
  MERGE_CASE(64, 0) MERGE_CASE(64, 1) MERGE_CASE(64, 2) MERGE_CASE(64, 3)
  MERGE_CASE(128, 0) MERGE_CASE(128, 1) MERGE_CASE(128, 2) MERGE_CASE(128, 3)
#undef MERGE_CASE
  return cudaErrorInvalidValue;
}

cudaError_t restore_log_launch(const void* jobs_dev, int njobs, const unsigned long long* log, unsigned long long n,
                               int num_sms, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  const unsigned long long blocks = std::min<unsigned long long>((n + 255) / 256, (unsigned long long)num_sms * 8);
  merge_tc::restore_log_kernel<<<(unsigned)blocks, 256, 0, s>>>(static_cast<const merge_tc::Job*>(jobs_dev), njobs,
                                                                 log, n);
  return cudaGetLastError();
}

cudaError_t merge_preload() { return preload_module_of(reinterpret_cast<const void*>(&merge_tc::restore_log_kernel)); }

}  // namespace dit
