// Microbenchmark (measurement only): per-CTA copy bandwidth, LSU 16-byte loads/stores vs TMA bulk
// copies (cp.async.bulk G2S -> S2G through a shared-memory ring).  One CTA per SM.
// nvcc -gencode arch=compute_100a,code=sm_100a -I paper_2601_17654_b200/csrc tools/ubench_copy.cu -o tools/ubench_copy
#include "sm100.cuh"
using namespace kpo::sm100;

__global__ void __launch_bounds__(512, 1) copy_lsu(const uint4* __restrict__ src, uint4* __restrict__ dst, size_t n) {
  const size_t per = (n + gridDim.x - 1) / gridDim.x;
  const size_t b = per * blockIdx.x, e = min(n, b + per);
  size_t i = b + threadIdx.x;
  constexpr int U = 16;
  for (; i + (U - 1) * 512 < e; i += U * 512) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = kpo::ld_weak_v4(src + i + u * 512);
#pragma unroll
    for (int u = 0; u < U; ++u) kpo::st_v4(dst + i + u * 512, v[u]);
  }
  for (; i < e; i += 512) kpo::st_v4(dst + i, kpo::ld_weak_v4(src + i));
}

template <int CHUNK, int STAGES>
__global__ void __launch_bounds__(32, 1) copy_tma(const char* __restrict__ src, char* __restrict__ dst, size_t bytes) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ __align__(8) uint64_t bar[STAGES];
  const size_t per = (bytes / CHUNK + gridDim.x - 1) / gridDim.x * CHUNK;
  const size_t b = per * blockIdx.x, e = min(bytes, b + per);
  if (threadIdx.x != 0) return;
  for (int s = 0; s < STAGES; ++s) mbar_init(smem_u32(&bar[s]), 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  const int nchunks = (int)((e > b ? e - b : 0) / CHUNK);
  // prologue: fill the ring
  for (int c = 0; c < STAGES - 1 && c < nchunks; ++c) {
    mbar_arrive_expect_tx(smem_u32(&bar[c]), CHUNK);
    bulk_load(smem_u32(smem + c * CHUNK), src + b + (size_t)c * CHUNK, CHUNK, smem_u32(&bar[c]));
  }
  for (int c = 0; c < nchunks; ++c) {
    const int s = c % STAGES;
    mbar_wait(smem_u32(&bar[s]), (c / STAGES) & 1);
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst + b + (size_t)c * CHUNK),
                 "r"(smem_u32(smem + s * CHUNK)), "r"(CHUNK)
                 : "memory");
    bulk_commit();
    // refill the stage of chunk c-1 (its store was committed one iteration ago): at most one store
    // group (chunk c's) may still be reading shared memory
    const int pc = c - 1, nc = pc + STAGES;
    if (c == 0 && STAGES - 1 < nchunks) {  // last prologue chunk goes into the one free stage
      mbar_arrive_expect_tx(smem_u32(&bar[STAGES - 1]), CHUNK);
      bulk_load(smem_u32(smem + (STAGES - 1) * CHUNK), src + b + (size_t)(STAGES - 1) * CHUNK, CHUNK,
                smem_u32(&bar[STAGES - 1]));
    }
    if (pc >= 0 && nc < nchunks) {
      asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
      const int ps = pc % STAGES;
      mbar_arrive_expect_tx(smem_u32(&bar[ps]), CHUNK);
      bulk_load(smem_u32(smem + ps * CHUNK), src + b + (size_t)nc * CHUNK, CHUNK, smem_u32(&bar[ps]));
    }
  }
  bulk_wait0();
}

int main() {
  const size_t bytes = 256ull << 20;
  char *src, *dst;
  cudaMalloc(&src, bytes);
  cudaMalloc(&dst, bytes);
  cudaMemset(src, 1, bytes);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto timeit = [&](auto fn) {
    fn();
    cudaDeviceSynchronize();
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) fn();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    return ms / 5;
  };
  constexpr int CH = 16384, ST = 13;
  cudaFuncSetAttribute(copy_tma<CH, ST>, cudaFuncAttributeMaxDynamicSharedMemorySize, CH * ST);
  cudaFuncSetAttribute(copy_lsu, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (int g : {1, 4, 8, 16, 32, 64, 148}) {
    float a = timeit([&] { copy_lsu<<<g, 512, 200 * 1024>>>((const uint4*)src, (uint4*)dst, bytes / 16); });
    float t = timeit([&] { copy_tma<CH, ST><<<g, 32, CH * ST>>>(src, dst, bytes); });
    printf("ctas %3d  lsu %7.1f GB/s (%.1f per CTA)   tma-bulk %7.1f GB/s (%.1f per CTA)\n", g, bytes / a / 1e6,
           bytes / a / 1e6 / g, bytes / t / 1e6, bytes / t / 1e6 / g);
  }
  // verify the last TMA copy
  cudaMemset(dst, 0, bytes);
  {
    unsigned char* h = (unsigned char*)malloc(bytes);
    for (size_t i = 0; i < bytes; ++i) h[i] = (unsigned char)(i * 131 + 7);
    cudaMemcpy(src, h, bytes, cudaMemcpyHostToDevice);
    copy_tma<CH, ST><<<16, 32, CH * ST>>>(src, dst, bytes);
    unsigned char* g = (unsigned char*)malloc(bytes);
    cudaMemcpy(g, dst, bytes, cudaMemcpyDeviceToHost);
    size_t bad = 0;
    for (size_t i = 0; i < bytes; ++i) bad += g[i] != h[i];
    printf("tma copy verify: %zu bad bytes\n", bad);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
