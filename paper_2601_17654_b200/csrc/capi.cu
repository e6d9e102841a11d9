// capi.cu — library-level C ABI: error convention, version, device facts.
#include "common.cuh"

namespace kpo {
static thread_local char g_last_error[1024] = "";
void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_last_error, sizeof(g_last_error), fmt, ap);
  va_end(ap);
}
}  // namespace kpo

extern "C" const char* kpo_last_error(void) { return kpo::g_last_error; }

extern "C" int kpo_version(void) { return 1; }

extern "C" int kpo_device_info(int device, int* num_sms, int* smem_optin_bytes, int* cc_major, int* cc_minor) {
  KPO_CHECK_ARG(num_sms && smem_optin_bytes && cc_major && cc_minor, "device_info: null output");
  KPO_CUDA(cudaDeviceGetAttribute(num_sms, cudaDevAttrMultiProcessorCount, device));
  KPO_CUDA(cudaDeviceGetAttribute(smem_optin_bytes, cudaDevAttrMaxSharedMemoryPerBlockOptin, device));
  KPO_CUDA(cudaDeviceGetAttribute(cc_major, cudaDevAttrComputeCapabilityMajor, device));
  KPO_CUDA(cudaDeviceGetAttribute(cc_minor, cudaDevAttrComputeCapabilityMinor, device));
  return KPO_OK;
}

// Launch-completion-event probe: one empty kernel launched with
// cudaLaunchAttributeLaunchCompletionEvent.  The partition executor's launch gate (executor.py) uses
// this attribute on every overlapped collective; some tools (e.g. a profiler replaying kernels)
// reject it, so the executor probes once and falls back to an ungated fork when it fails.
__global__ void kpo_probe_kernel() {}

extern "C" int kpo_probe_launch_completion(void* event, void* stream) {
  KPO_CHECK_ARG(event, "probe_launch_completion: null event");
  cudaLaunchConfig_t cfg = {};
  // the same attribute set as the collectives' launches (comm.cu): 2-CTA clusters + the completion event
  cfg.gridDim = dim3(2);
  cfg.blockDim = dim3(32);
  cfg.stream = (cudaStream_t)stream;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeLaunchCompletionEvent;
  attr[1].val.launchCompletionEvent.event = (cudaEvent_t)event;
  attr[1].val.launchCompletionEvent.flags = 0;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  KPO_CUDA(cudaLaunchKernelEx(&cfg, kpo_probe_kernel));
  KPO_CUDA(cudaStreamSynchronize((cudaStream_t)stream));
  KPO_CUDA(cudaEventQuery((cudaEvent_t)event));
  return KPO_OK;
}

// SM blocker: `ncta` CTAs, each holding the whole opt-in shared memory (so exactly one per SM and no
// other CTA can share its SM), spinning on the global timer for `spin_ns`.  Measures a kernel's time
// on (num_sms - ncta) SMs without touching the kernel (reference kernel_duration(k, f, sms),
// simgpu.py:144-168, tools/unit_sm_sweep.py).  `launched_event` (cudaEvent_t, may be null) is
// recorded with cudaLaunchAttributeLaunchCompletionEvent: once it completes, every blocker CTA is
// resident.
__global__ void kpo_sm_blocker_kernel(unsigned long long spin_ns) {
  extern __shared__ uint8_t kpo_blocker_smem[];
  unsigned long long t0, t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  if (threadIdx.x == 0) kpo_blocker_smem[0] = 0;
  do {
    __nanosleep(500);
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  } while (t - t0 < spin_ns);
}

extern "C" int kpo_sm_blocker(int ncta, int64_t spin_ns, void* launched_event, void* stream) {
  KPO_CHECK_ARG(ncta >= 0 && spin_ns >= 0, "sm_blocker: ncta and spin_ns must be >= 0");
  if (ncta == 0) return KPO_OK;
  int dev = 0, smem = 0;
  KPO_CUDA(cudaGetDevice(&dev));
  KPO_CUDA(cudaDeviceGetAttribute(&smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  KPO_CUDA(cudaFuncSetAttribute(kpo_sm_blocker_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)ncta);
  cfg.blockDim = dim3(32);
  cfg.dynamicSmemBytes = (size_t)smem;
  cfg.stream = (cudaStream_t)stream;
  // like the collectives (comm.cu): an even count is launched as 2-CTA clusters, so it takes whole
  // TPCs and leaves whole TPCs to the CTA-pair GEMMs
  cudaLaunchAttribute attr[2];
  int na = 0;
  if (ncta % 2 == 0) {
    attr[na].id = cudaLaunchAttributeClusterDimension;
    attr[na].val.clusterDim.x = 2;
    attr[na].val.clusterDim.y = 1;
    attr[na].val.clusterDim.z = 1;
    ++na;
  }
  if (launched_event) {
    attr[na].id = cudaLaunchAttributeLaunchCompletionEvent;
    attr[na].val.launchCompletionEvent.event = (cudaEvent_t)launched_event;
    attr[na].val.launchCompletionEvent.flags = 0;
    ++na;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  KPO_CUDA(cudaLaunchKernelEx(&cfg, kpo_sm_blocker_kernel, (unsigned long long)spin_ns));
  return KPO_OK;
}
