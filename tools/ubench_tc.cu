// Microbenchmark (measurement only, not part of libkpo): tcgen05.ld / tcgen05.st throughput and
// tcgen05.mma dispatch rate for the attention tile shapes.  nvcc -gencode arch=compute_100a,code=sm_100a
// -I paper_2601_17654_b200/csrc tools/ubench_tc.cu -o tools/ubench_tc && tools/ubench_tc
#include "sm100.cuh"
using namespace kpo::sm100;

__global__ void __launch_bounds__(512, 1) k_ld(int warps_active, int iters, unsigned long long* out) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) tmem_alloc(smem_u32(&slot), 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  uint32_t acc = 0;
  long long t0 = clock64();
  if (warp < warps_active) {
    const uint32_t a = tmem + ((uint32_t)((warp & 3) * 32) << 16) + (warp >> 2) * 32;
    for (int i = 0; i < iters; ++i) {
      uint32_t r[32];
      tmem_ld32_nowait(a + ((i & 3) * 128 & 511), r);
      tmem_wait_ld();
#pragma unroll
      for (int j = 0; j < 32; ++j) acc += r[j];
    }
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = (unsigned long long)(t1 - t0);
  if (acc == 0x12345678u) out[1000] = acc;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, 512);
}

__global__ void __launch_bounds__(512, 1) k_st(int warps_active, int iters, unsigned long long* out) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) tmem_alloc(smem_u32(&slot), 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  long long t0 = clock64();
  if (warp < warps_active) {
    const uint32_t a = tmem + ((uint32_t)((warp & 3) * 32) << 16) + (warp >> 2) * 32;
    uint32_t r[32];
    for (int j = 0; j < 32; ++j) r[j] = j * threadIdx.x;
    for (int i = 0; i < iters; ++i) {
      tmem_st32(a + ((i & 3) * 128 & 511), r);
      tmem_wait_st();
    }
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = (unsigned long long)(t1 - t0);
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, 512);
}

// mode 0: SS (A,B smem), mode 1: TS (A from TMEM)
__global__ void __launch_bounds__(128, 1) k_mma(int N, int mode, int iters, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* s = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm) + 1023) & ~uintptr_t(1023));
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(s)[i] = 0;
  if (threadIdx.x == 0) {
    mbar_init(smem_u32(&bar), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) tmem_alloc(smem_u32(&slot), 512);
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  long long t0 = clock64();
  if (threadIdx.x == 0) {
    const uint32_t sa = smem_u32(s), sb = smem_u32(s + 32768);
    const uint32_t id = idesc_bf16(128, N, false, false);
    if (mode >= 2 && mode <= 4) {
      // independent accumulators round-robin (2 / 4) or unrolled same accumulator (mode 4)
      const int nacc = mode == 2 ? 2 : (mode == 3 ? 4 : 1);
      const uint32_t step = N <= 64 ? 64 : 128;
      const uint64_t a0 = smem_desc(sa, 16, 1024), b0 = smem_desc(sb, 16, 1024);
      for (int i = 0; i < iters; i += 8) {
#pragma unroll
        for (int u = 0; u < 8; ++u)
          tc_mma(tmem + (nacc == 1 ? 0 : ((u % nacc) * step) % 512), a0 + 2 * (u & 3), b0 + 2 * (u & 3), id, 1u);
      }
    } else {
      for (int i = 0; i < iters; ++i) {
        const int k = i & 3;
        if (mode == 0)
          tc_mma(tmem + 256, smem_desc(sa + k * 32, 16, 1024), smem_desc(sb + k * 32, 16, 1024), id, 1u);
        else
          tc_mma_ts(tmem + 256, tmem + 0 + k * 8, smem_desc(sb + k * 32, 16, 1024), id, 1u);
      }
    }
    tc_commit(smem_u32(&bar));
    mbar_wait(smem_u32(&bar), 0);
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = (unsigned long long)(t1 - t0);
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, 512);
}

static double avg(unsigned long long* h, int n) {
  double s = 0;
  for (int i = 0; i < n; ++i) s += h[i];
  return s / n;
}

int main() {
  unsigned long long *d, h[1024];
  cudaMalloc(&d, 1024 * 8 + 8 * 8);
  const int G = 148;
  const int iters = 4096;
  for (int w : {1, 4, 8, 16}) {
    k_ld<<<G, 512>>>(w, iters, d);
    cudaDeviceSynchronize();
    k_ld<<<G, 512>>>(w, iters, d);
    cudaMemcpy(h, d, G * 8, cudaMemcpyDeviceToHost);
    double cyc = avg(h, G);
    printf("tcgen05.ld 32x32b.x32  warps=%2d  %.1f cyc/ld/warp  %.1f B/clk/SM\n", w, cyc / iters,
           (double)w * iters * 4096 / cyc);
  }
  for (int w : {4, 8, 16}) {
    k_st<<<G, 512>>>(w, iters, d);
    cudaDeviceSynchronize();
    k_st<<<G, 512>>>(w, iters, d);
    cudaMemcpy(h, d, G * 8, cudaMemcpyDeviceToHost);
    double cyc = avg(h, G);
    printf("tcgen05.st 32x32b.x32  warps=%2d  %.1f cyc/st/warp  %.1f B/clk/SM\n", w, cyc / iters,
           (double)w * iters * 4096 / cyc);
  }
  cudaFuncSetAttribute(k_mma, cudaFuncAttributeMaxDynamicSharedMemorySize, 66 * 1024);
  for (int mode : {0, 1, 2, 3, 4})
    for (int N : {64, 128, 256}) {
      if (mode == 3 && N == 256) continue;
      k_mma<<<G, 128, 66 * 1024>>>(N, mode, iters, d);
      cudaDeviceSynchronize();
      k_mma<<<G, 128, 66 * 1024>>>(N, mode, iters, d);
      cudaMemcpy(h, d, G * 8, cudaMemcpyDeviceToHost);
      double cyc = avg(h, G);
      printf("tcgen05.mma %s M=128 N=%3d K=16  %.1f cyc/mma (floor %d)  %.0f flop/clk/SM\n", (const char*[]){"SS", "TS", "SS-2acc", "SS-4acc", "SS-unroll"}[mode], N,
             cyc / iters, 128 * N / 256, 2.0 * 128 * N * 16 * iters / cyc);
    }
  cudaError_t e = cudaGetLastError();
  printf("status %s\n", cudaGetErrorString(e));
  return 0;
}
