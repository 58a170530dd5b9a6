// MUFU.EX2 issue rate by warps per SMSP: one CTA of 128 / 256 / 512 threads (1 / 2 / 4 warps per
// SMSP), each thread 64 independent exp2 per iteration (FFMA2 input, so nothing is hoisted),
// clocks per iteration.  KIND 0: results consumed at the end; KIND 1: each pair packed to bf16x2
// right after its two MUFUs (short scoreboard released early); KIND 2: KIND 1 + every 4th pair
// on the FMA-pipe polynomial.  Question: how fast can ONE warp (the attention softmax has one warp
// per SMSP per query tile) stream MUFU ops?
#include <cstdio>

__device__ __forceinline__ float ex2(float x) { float y; asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ __forceinline__ unsigned pk(float a, float b) { unsigned r; asm("cvt.rn.bf16x2.f32 %0, %2, %1;" : "=r"(r) : "f"(a), "f"(b)); return r; }
__device__ __forceinline__ float2 poly2(float2 x) {
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

template <int KIND>
__global__ void k(float* out, long long* cyc, int iters) {
  float s[64];
  for (int i = 0; i < 64; ++i) s[i] = out[(threadIdx.x * 64 + i) & 16383] * 1e-3f;
  float m = 0.f;
  unsigned acc = 0;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    float y[64];
    unsigned r[32];
#pragma unroll
    for (int e = 0; e < 64; e += 2) {
      float2 x = __ffma2_rn(make_float2(s[e], s[e + 1]), make_float2(1.4427f, 1.4427f), make_float2(-m, -m));
      if (KIND == 2 && (e / 2) % 4 == 3) {
        const float2 pp = poly2(x);
        y[e] = pp.x; y[e + 1] = pp.y;
      } else {
        y[e] = ex2(x.x); y[e + 1] = ex2(x.y);
      }
      if (KIND >= 1) r[e / 2] = pk(y[e], y[e + 1]);
    }
    m = y[63] * 1e-30f + y[0] * 1e-30f;
    if (KIND >= 1) {
#pragma unroll
      for (int e = 0; e < 32; ++e) acc += r[e];
    } else {
#pragma unroll
      for (int e = 0; e < 64; ++e) s[e] = __int_as_float(__float_as_int(s[e]) ^ (__float_as_int(y[e]) & 1));
    }
  }
  long long t1 = clock64();
  float a = m + (float)acc;
  for (int i = 0; i < 64; ++i) a += s[i];
  out[threadIdx.x] = a;
  if (threadIdx.x == 0) cyc[0] = (t1 - t0);
}

int main() {
  float* d; long long* c; cudaMalloc(&d, 16384 * 4); cudaMalloc(&c, 8); cudaMemset(d, 0, 16384 * 4);
  int iters = 2000;
  const char* names[] = {"consume late", "pack per pair", "pack + 1/4 poly"};
  for (int kind = 0; kind < 3; ++kind)
    for (int thr = 128; thr <= 512; thr *= 2) {
      if (kind == 0) k<0><<<1, thr>>>(d, c, iters);
      if (kind == 1) k<1><<<1, thr>>>(d, c, iters);
      if (kind == 2) k<2><<<1, thr>>>(d, c, iters);
      cudaDeviceSynchronize();
      long long cy; cudaMemcpy(&cy, c, 8, cudaMemcpyDeviceToHost);
      const double per_it = (double)cy / iters;
      const int mufu = kind == 2 ? 48 : 64;
      printf("%-16s %d warps/SMSP: %7.1f clk per iteration per SMSP (%d MUFU per warp) -> %.2f clk per MUFU\n",
             names[kind], thr / 128, per_it, mufu, per_it / (mufu * thr / 128.0));
    }
  return 0;
}
