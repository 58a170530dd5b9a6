// merge_tc.cu -- LoRA weight patching on the tensor cores:
//   W'[o][i] = bf16(W[o][i] + scale * sum_k B[o][k] A[k][i])
// One CTA per 128 x 128 tile of W: TMA brings the B rows (K-major), the A columns (MN-major)
// and the W tile (all SWIZZLE_128B) into shared memory, one thread issues the rank-r product
// as tcgen05 MMAs into 128 TMEM columns, every thread then owns one tile row: it reads its
// accumulator row from TMEM, adds it into the W row in shared memory, and one thread TMA-stores
// the patched tile.  Global traffic is the W read + W' write (the factors are L2-resident), all
// of it as TMA bulk copies; the product costs no CUDA-core time.
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

template <int RA>
__global__ void __launch_bounds__(THREADS) merge_tc_kernel(const __grid_constant__ Maps m, float scale) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  constexpr int KP = RA / 64;
  uint8_t* sB = smem;                    // KP x [128 rows][64 k]
  uint8_t* sA = sB + KP * 16384;         // 2 x [RA k][64 cols]
  uint8_t* sW = sA + 2 * RA * 128;       // 2 x [128 rows][64 cols]
  uint64_t* bars = reinterpret_cast<uint64_t*>(sW + 32768);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + 2);
  const int c0 = blockIdx.x * TILE, r0 = blockIdx.y * TILE;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    tma_prefetch_desc(&m.w);
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc<128>(tslot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;
  if (threadIdx.x == 0) {
    mbar_expect_tx(&bars[0], KP * 16384 + 2 * RA * 128 + 32768);
    for (int p = 0; p < KP; ++p) tma_load_2d(&m.b, &bars[0], sB + p * 16384, p * 64, r0);
    for (int p = 0; p < 2; ++p) tma_load_2d(&m.a, &bars[0], sA + p * RA * 128, c0 + p * 64, 0);
    for (int p = 0; p < 2; ++p) tma_load_2d(&m.w, &bars[0], sW + p * 16384, c0 + p * 64, r0);
    mbar_wait(&bars[0], 0);
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
  mbar_wait(&bars[1], 0);
  tc_fence_after();
  const int row = warp * 32 + lane;
  const uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16);
#pragma unroll
  for (int cc = 0; cc < 4; ++cc) {
    uint32_t acc[32];
    tmem_ld32(taddr + cc * 32, acc);
    tmem_ld_wait();
    uint8_t* prow = sW + (cc / 2) * 16384 + row * 128;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int j = (cc % 2) * 4 + q;                                   // logical 16-byte chunk
      uint4* pc = reinterpret_cast<uint4*>(prow + ((j ^ (row & 7)) << 4));   // SWIZZLE_128B
      uint4 w = *pc;
      uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
      for (int e = 0; e < 4; ++e)
        ws[e] = pack_bf16(bf16_lo(ws[e]) + scale * __uint_as_float(acc[q * 8 + 2 * e]),
                          bf16_hi(ws[e]) + scale * __uint_as_float(acc[q * 8 + 2 * e + 1]));
      *pc = make_uint4(ws[0], ws[1], ws[2], ws[3]);
    }
  }
  fence_async_shared();   // the patched rows (generic proxy) -> the TMA store (async proxy)
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int p = 0; p < 2; ++p) tma_store_2d(&m.out, sW + p * 16384, c0 + p * 64, r0);
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
  }
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<128>(tmem);
  }
}

}  // namespace merge_tc

cudaError_t lora_merge_tc_launch(const CUtensorMap& w_map, const CUtensorMap& out_map, const void* A, const void* Bm,
                                 int rows, int cols, int ra, float scale, cudaStream_t s) {
  using namespace merge_tc;
  if (ra != 64 && ra != 128) return cudaErrorInvalidValue;
  Maps m;
  m.w = w_map;
  m.out = out_map;
  if (!make_tmap_2d(&m.b, Bm, ra, rows, (uint64_t)ra * 2, 64, 128) ||
      !make_tmap_2d(&m.a, A, cols, ra, (uint64_t)cols * 2, 64, ra))
    return cudaErrorInvalidValue;
  static bool attr64 = false, attr128 = false;
  dim3 grid((cols + TILE - 1) / TILE, (rows + TILE - 1) / TILE);
  if (ra == 64) {
    if (!attr64) {
      cudaError_t e = cudaFuncSetAttribute(merge_tc_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           smem_bytes<64>());
      if (e != cudaSuccess) return e;
      attr64 = true;
    }
    merge_tc_kernel<64><<<grid, THREADS, smem_bytes<64>(), s>>>(m, scale);
  } else {
    if (!attr128) {
      cudaError_t e = cudaFuncSetAttribute(merge_tc_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           smem_bytes<128>());
      if (e != cudaSuccess) return e;
      attr128 = true;
    }
    merge_tc_kernel<128><<<grid, THREADS, smem_bytes<128>(), s>>>(m, scale);
  }
  return cudaGetLastError();
}

}  // namespace dit
