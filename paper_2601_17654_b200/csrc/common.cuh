// common.cuh — status/error plumbing and small device helpers shared by every kpo kernel file.
#pragma once
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>
#include <stdio.h>
#include <stdarg.h>
#include <string>
#include <utility>
#include <cstdlib>

#include "../../include/kpo.h"

namespace kpo {

// Thread-local last-error string (kpo_last_error).  Defined in capi.cu.
void set_error(const char* fmt, ...);

#define KPO_CHECK_ARG(cond, ...)                 \
  do {                                           \
    if (!(cond)) {                               \
      ::kpo::set_error(__VA_ARGS__);             \
      return KPO_ERR_INVALID;                    \
    }                                            \
  } while (0)

#define KPO_CUDA(call)                                                                  \
  do {                                                                                  \
    cudaError_t _e = (call);                                                            \
    if (_e != cudaSuccess) {                                                            \
      ::kpo::set_error("%s:%d %s -> %s", __FILE__, __LINE__, #call, cudaGetErrorString(_e)); \
      return KPO_ERR_CUDA;                                                              \
    }                                                                                   \
  } while (0)

#define KPO_LAUNCH_CHECK() KPO_CUDA(cudaGetLastError())

inline int num_sms(int device = -1) {
  static int cached[64] = {0};
  if (device < 0) cudaGetDevice(&device);
  if (device >= 0 && device < 64 && cached[device]) return cached[device];
  int n = 0;
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, device);
  if (device >= 0 && device < 64) cached[device] = n;
  return n;
}

// ------------------------------------------------------------------ programmatic dependent launch
// Every compute kernel is launched with programmatic stream serialization: it lets the next kernel
// of the stream launch once all of its CTAs have started (griddepcontrol.launch_dependents), and the
// next kernel waits for this one's completion and memory flush (griddepcontrol.wait) before it
// touches global memory.  The dependent's launch latency and prologue (barrier init, TMEM
// allocation, tensor-map prefetch) then overlap the tail of the previous kernel.  Both
// instructions are no-ops for a kernel launched without the attribute.
// Opt-in (KPO_PDL=1): measured on the layer step it is SLOWER (5.73 -> 6.06 ms per iteration, A/B in
// one session), most likely because early-launched dependents take SMs the SM-budgeted collective
// on the other stream needs; the launch path and the kernel-side waits are kept for that experiment.
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
#define KPO_PDL_ENTRY()             \
  do {                              \
    ::kpo::pdl_launch_dependents(); \
    ::kpo::pdl_wait();              \
  } while (0)

inline bool pdl_enabled() {
  static const bool on = [] {
    const char* e = getenv("KPO_PDL");
    return e && e[0] == '1';
  }();
  return on;
}

template <typename... KArgs, typename... Args>
inline cudaError_t pdl_launch(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                              Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

// ------------------------------------------------------------------ device helpers
__device__ __forceinline__ float bf2f(__nv_bfloat16 v) { return __bfloat162float(v); }
__device__ __forceinline__ __nv_bfloat16 f2bf(float v) { return __float2bfloat16_rn(v); }

// 8 x bf16 <-> uint4
__device__ __forceinline__ void unpack8(const uint4& u, float* f) {
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    float2 t = __bfloat1622float2(h[i]);
    f[2 * i] = t.x;
    f[2 * i + 1] = t.y;
  }
}
__device__ __forceinline__ uint4 pack8(const float* f) {
  uint4 u;
  __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
  for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(f[2 * i], f[2 * i + 1]);
  return u;
}

__device__ __forceinline__ uint4 ld_nc_v4(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
// Volatile (uncached in L1) 16-byte load: peer memory written by another device.
__device__ __forceinline__ uint4 ld_volatile_v4(const void* p) {
  uint4 r;
  asm volatile("ld.volatile.global.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
// weak 16-byte load that skips L1: for peer / symmetric buffers read after an acquire barrier
// (ld.volatile compiles to LDG.STRONG.SYS, which measured ~2x slower per CTA for bulk copies)
__device__ __forceinline__ uint4 ld_weak_v4(const void* p) {
  uint4 r;
  asm volatile("ld.global.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p)
               : "memory");
  return r;
}
__device__ __forceinline__ void st_v4(void* p, const uint4& v) {
  asm volatile("st.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}

__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
  __nv_bfloat162 h = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&h);
}

// logistic sigmoid for the SwiGLU kernels and the fused GEMM epilogues (one definition, so the fused
// and separate paths are bit-identical): MUFU ex2 + MUFU rcp (__fdividef), no IEEE division.  For
// x < -87 the denominator overflows and the result is 0, the correctly rounded limit.
__device__ __forceinline__ float kpo_sigmoid(float x) { return __fdividef(1.f, 1.f + __expf(-x)); }

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ uint32_t smid() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t r;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(r));
  return r;
}

}  // namespace kpo
