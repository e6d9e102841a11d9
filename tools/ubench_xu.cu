// Microbenchmark (measurement only): which pipe runs the bf16x2 pack (cvt.rn.bf16x2.f32) relative to
// MUFU.EX2, and the FMA-pipe exp2 emulation rate.  nvcc -gencode arch=compute_100a,code=sm_100a
// -I paper_2601_17654_b200/csrc tools/ubench_xu.cu -o tools/ubench_xu && tools/ubench_xu
#include "sm100.cuh"
using namespace kpo::sm100;
using kpo::pack_bf16x2;

__device__ __forceinline__ float ex2_fma(float x) {
  // round-to-nearest via the 1.5*2^23 magic constant (FADD on the FMA pipe, no FRND / F2I)
  const float j = x + 12582912.f;
  const float f = x - (j - 12582912.f);  // [-0.5, 0.5]
  float p = fmaf(fmaf(fmaf(fmaf(0.0013333558f, f, 0.0096181291f), f, 0.0555041087f), f, 0.2402265070f), f, 0.6931471806f);
  p = fmaf(p, f, 1.0f);
  return __int_as_float(__float_as_int(p) + (__float_as_int(j) << 23));
}

__device__ __forceinline__ uint32_t ex2_h2(uint32_t x) {
  uint32_t y;
  asm volatile("ex2.approx.f16x2 %0, %1;" : "=r"(y) : "r"(x));
  return y;
}

template <int MODE>
__global__ void k(int iters, float* out) {
  float a[8], acc = 0.f;
  uint32_t u = 0;
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3f + i * 0.01f - 4.f;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (MODE == 0 || MODE == 2) a[i] = ex2(a[i]) - 4.f;
      if (MODE == 1 || MODE == 2) u ^= pack_bf16x2(a[i], a[(i + 1) & 7]);
      if (MODE == 3) a[i] = ex2_fma(a[i]) - 4.f;
      if (MODE == 4) {
        if (i & 1) a[i] = ex2_fma(a[i]) - 4.f;
        else a[i] = ex2(a[i]) - 4.f;
      }
      if (MODE == 1) a[i] += 1e-7f;
      if (MODE == 5) u = ex2_h2(u ^ (uint32_t)i) ^ 0x3c003c00u;  // 2 exponentials per instruction
      if (MODE == 6) {  // the full f16x2 softmax path per pair: pack args, ex2.f16x2, unpack, bf16x2 pack
        uint32_t h;
        asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(h) : "f"(a[i]), "f"(a[(i + 1) & 7]));
        h = ex2_h2(h);
        float lo, hi;
        asm("{.reg .f16 l, h; mov.b32 {l, h}, %2; cvt.f32.f16 %0, l; cvt.f32.f16 %1, h;}" : "=f"(lo), "=f"(hi) : "r"(h));
        u ^= pack_bf16x2(lo, hi);
        a[i] = lo + hi - 4.f;
      }
    }
  }
  long long t1 = clock64();
  for (int i = 0; i < 8; ++i) acc += a[i];
  if (threadIdx.x == 0) out[blockIdx.x] = (float)(t1 - t0);
  if (acc == 1234.5f || u == 0x12345u) out[1000 + blockIdx.x] = acc + u;
}

int main() {
  float* d;
  cudaMalloc(&d, 4096 * 4);
  const char* names[] = {"ex2 (MUFU)", "cvt.rn.bf16x2 pack", "ex2 + pack", "ex2 on FMA pipe", "half MUFU half FMA",
                         "ex2.f16x2 (per instr, 2 exps)", "f16x2 softmax pair path (per pair)"};
  for (int m = 0; m < 7; ++m) {
    const int iters = 2048, threads = 512;
    auto run = [&]() {
      if (m == 0) k<0><<<148, threads>>>(iters, d);
      if (m == 1) k<1><<<148, threads>>>(iters, d);
      if (m == 2) k<2><<<148, threads>>>(iters, d);
      if (m == 3) k<3><<<148, threads>>>(iters, d);
      if (m == 4) k<4><<<148, threads>>>(iters, d);
      if (m == 5) k<5><<<148, threads>>>(iters, d);
      if (m == 6) k<6><<<148, threads>>>(iters, d);
    };
    run();
    cudaDeviceSynchronize();
    run();
    float h[148];
    cudaMemcpy(h, d, 148 * 4, cudaMemcpyDeviceToHost);
    double c = 0;
    for (int i = 0; i < 148; ++i) c += h[i];
    c /= 148;
    printf("%-22s %.2f ops/clk/SM\n", names[m], (double)threads * iters * 8 / c);
  }
  // accuracy of ex2_fma vs exp2f on [-30, 0]
  return 0;
}
