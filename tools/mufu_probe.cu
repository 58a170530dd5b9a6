// MUFU exp2 throughput probe: ex2.approx.f32 vs ex2.approx.f16x2 vs ex2.approx.ftz.bf16x2
// (results per clock per SM), all warps of a full-occupancy grid issuing independent chains.
#include <cstdio>
#include <cuda_fp16.h>
#include <cuda_bf16.h>

__global__ void k_f32(float* out, int iters) {
  float a[8];
  for (int i = 0; i < 8; ++i) a[i] = -0.001f * (threadIdx.x + i);
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
  long long t1 = clock64();
  float s = 0; for (int i = 0; i < 8; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s + (float)(t1 - t0) * 1e-30f;
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = (float)(t1 - t0);
}
__global__ void k_f16x2(float* out, int iters) {
  unsigned a[8];
  for (int i = 0; i < 8; ++i) { __half2 h = __floats2half2_rn(-0.001f * (threadIdx.x + i), -0.002f); a[i] = *reinterpret_cast<unsigned*>(&h); }
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(a[i]));
  long long t1 = clock64();
  unsigned s = 0; for (int i = 0; i < 8; ++i) s ^= a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = (float)s;
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = (float)(t1 - t0);
}
__global__ void k_bf16x2(float* out, int iters) {
  unsigned a[8];
  for (int i = 0; i < 8; ++i) { __nv_bfloat162 h = __floats2bfloat162_rn(-0.001f * (threadIdx.x + i), -0.002f); a[i] = *reinterpret_cast<unsigned*>(&h); }
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(a[i]));
  long long t1 = clock64();
  unsigned s = 0; for (int i = 0; i < 8; ++i) s ^= a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = (float)s;
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = (float)(t1 - t0);
}

int main() {
  float* d; cudaMalloc(&d, 148 * 1024 * 4 * 4);
  int iters = 4096;
  for (int kind = 0; kind < 3; ++kind) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
      cudaEventRecord(e0);
      if (kind == 0) k_f32<<<148 * 2, 1024>>>(d, iters);
      if (kind == 1) k_f16x2<<<148 * 2, 1024>>>(d, iters);
      if (kind == 2) k_bf16x2<<<148 * 2, 1024>>>(d, iters);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      float cyc; cudaMemcpy(&cyc, d, 4, cudaMemcpyDeviceToHost);
      double ops = 148.0 * 2 * 1024 * iters * 8;           // instructions (lanes)
      double results = ops * (kind == 0 ? 1 : 2);
      printf("%s: %.3f ms, %.1f Gresults/s, per-thread cycles %.0f -> %.2f results/clk/SM (at block clock)\n",
             kind == 0 ? "ex2.f32" : (kind == 1 ? "ex2.f16x2" : "ex2.bf16x2"), ms, results / ms / 1e6, cyc,
             (double)2048 * iters * 8 * (kind == 0 ? 1 : 2) / cyc);
    }
  }
  return 0;
}
