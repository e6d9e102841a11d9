// comm.cu — SM-budgeted peer-to-peer collectives over NVLink 5 / NVSwitch (or loopback).
//
// Replaces the reference's abstract communication kernel ("allreduce", workloads.py:50,64,74,90)
// whose cost model is `comm_bytes / (net_bw * min(1, sm/sat))` (simgpu.py:81-82,162-163) and
// whose SM budget `config.sm_alloc` (domain.py:152) the simulator charges against the compute
// kernels (simgpu.py:221).  Here the budget is physical:
//
//   * grid = exactly `ncta` CTAs, and every CTA requests the device's full opt-in shared memory,
//     so no other CTA (of any kernel) can be co-resident on its SM — the collective owns
//     `ncta` SMs while it runs, the compute kernels get the rest;
//   * data moves with 16-byte vector loads from each peer's symmetric buffer (mapped through
//     CUDA IPC) and 16-byte local stores; reductions accumulate in fp32 in a fixed rank order
//     (0..world-1), so results are deterministic and bit-identical to the CPU oracle;
//   * synchronisation is per CTA: CTA c of every rank exchanges epoch flags with CTA c of every
//     peer (release/acquire at system scope), so no grid-wide barrier is needed and the epoch
//     counters live on the device — a captured CUDA graph can be replayed indefinitely.
#include "sm100.cuh"
#include <vector>
#include <cstring>

#define KPO_MAX_WORLD 8
#define KPO_MAX_CTAS 256

struct kpo_comm {
  int rank = 0, world = 1, device = 0, loopback = 0;
  size_t sym_bytes = 0, flag_off = 0, alloc_bytes = 0;
  char* local = nullptr;                       // this rank's allocation (symmetric + flags)
  char* virt[KPO_MAX_WORLD] = {nullptr};       // loopback: virtual peers' allocations
  char* peer[KPO_MAX_WORLD] = {nullptr};       // every rank's allocation as mapped here
  bool opened = false;
  uint32_t* epoch = nullptr;                   // local [KPO_MAX_CTAS] per-CTA epoch counters
  int smem_bytes = 0;                          // full-SM reservation
  int64_t* trace = nullptr;
  int trace_slots = 0;
  int trace_next = 0;
  cudaEvent_t launch_evt = nullptr;
  cudaIpcMemHandle_t handle;
};

namespace kpo {

struct CommArgs {
  char* peer[KPO_MAX_WORLD];   // base of every rank's allocation
  uint32_t* my_flags;          // flags[src][cta] in my allocation
  uint32_t* peer_flags[KPO_MAX_WORLD];
  uint32_t* epoch;
  int rank, world, loopback;
  int bulk;                    // copy phases through TMA bulk copies (else 16-byte LSU copies)
  int64_t* trace;              // [ncta*4] or null
};

// TMA bulk copies beat the 16-byte LSU copies from 0.5 MB per CTA up (measured A/B with
// tools/comm_ab.sh: all-gather +8% at 1 MB per CTA, +27-38% at 4-16 MB per CTA; all-reduce +10-22%);
// tiny messages keep the LSU path (no ring fill latency).  KPO_COMM_BULK=0/1 forces either path.
inline int choose_bulk(size_t bytes_per_cta) {
  const char* env = getenv("KPO_COMM_BULK");
  if (env) return atoi(env) != 0;
  return bytes_per_cta >= ((size_t)256 << 10);
}

__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Per-CTA cross-rank barrier (CTA c of every rank).  Threads [0, world) each own one peer.
__device__ __forceinline__ void cta_barrier(const CommArgs& a, uint32_t e) {
  __syncthreads();
  const int t = threadIdx.x;
  if (t < a.world && t != a.rank) {
    __threadfence_system();
    // tell peer t that this rank's CTA blockIdx.x reached epoch e
    st_release_sys(a.peer_flags[t] + (size_t)a.rank * KPO_MAX_CTAS + blockIdx.x, e);
    if (!a.loopback) {
      const uint32_t* mine = a.my_flags + (size_t)t * KPO_MAX_CTAS + blockIdx.x;
      while ((int32_t)(ld_acquire_sys(mine) - e) < 0) {
      }
    }
  }
  __syncthreads();
}

__device__ __forceinline__ void trace_enter(const CommArgs& a) {
  if (a.trace && threadIdx.x == 0) {
    a.trace[blockIdx.x * 4 + 0] = smid();
    a.trace[blockIdx.x * 4 + 1] = (int64_t)globaltimer();
  }
}
__device__ __forceinline__ void trace_exit(const CommArgs& a) {
  if (a.trace && threadIdx.x == 0) {
    a.trace[blockIdx.x * 4 + 2] = (int64_t)globaltimer();
    a.trace[blockIdx.x * 4 + 3] = 1;
  }
}

// [begin, end) vector range of this CTA within n vectors.
__device__ __forceinline__ void cta_slice(size_t n, size_t& b, size_t& e) {
  const size_t per = (n + gridDim.x - 1) / gridDim.x;
  b = per * blockIdx.x;
  e = b + per < n ? b + per : n;
  if (b > n) b = n;
}

constexpr int kCommThreads = 512;
// 16 x 16 B loads in flight per thread = 128 KB per CTA: a CTA's copy rate is in-flight bytes /
// latency (measured with 4 in flight: ~28 GB/s per CTA on loopback HBM, i.e. latency-bound)
constexpr int kUnroll = 16;

// Copy n 16-byte vectors src -> dst, kUnroll loads in flight per thread.
__device__ __forceinline__ void copy_vecs(uint4* __restrict__ dst, const uint4* __restrict__ src, size_t b,
                                          size_t e) {
  size_t i = b + threadIdx.x;
  for (; i + (kUnroll - 1) * kCommThreads < e; i += kUnroll * kCommThreads) {
    uint4 v[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) v[u] = ld_weak_v4(src + i + u * kCommThreads);
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) st_v4(dst + i + u * kCommThreads, v[u]);
  }
  for (; i < e; i += kCommThreads) st_v4(dst + i, ld_weak_v4(src + i));
}

// ---------------------------------------------------------------- TMA bulk copies
// Copies move through a shared-memory ring with cp.async.bulk (global -> shared, completing on an
// mbarrier; shared -> global, tracked by a bulk group), issued by one thread.  Measured per CTA
// (tools/ubench_copy.cu): ~50 GB/s against ~35 GB/s with 16-byte loads / stores, so a collective
// needs fewer SMs for the same bandwidth.  The ring is the CTA's dynamic shared memory, which it
// reserves anyway to own its SM.
constexpr int kBulkChunk = 16384;
constexpr int kBulkStages = 12;
struct BulkSeg {
  char* dst;
  const char* src;
  size_t bytes;
};

// Thread 0 only.  Copies segs[0..n) (bytes multiples of 16, 16-byte aligned) through the ring.
__device__ void bulk_copy_segs(const BulkSeg* segs, int n, uint8_t* ring, uint64_t* full) {
  using namespace kpo::sm100;
  // chunk enumeration over the segments
  int seg = 0;
  size_t off = 0;
  auto next = [&](const char*& src, char*& dst, uint32_t& len) -> bool {
    while (seg < n && off >= segs[seg].bytes) {
      ++seg;
      off = 0;
    }
    if (seg >= n) return false;
    const size_t rem = segs[seg].bytes - off;
    len = (uint32_t)(rem < (size_t)kBulkChunk ? rem : (size_t)kBulkChunk);
    src = segs[seg].src + off;
    dst = segs[seg].dst + off;
    off += len;
    return true;
  };
  char* dsts[kBulkStages];
  uint32_t lens[kBulkStages];
  int loaded = 0;
  // async-proxy reads must observe the generic-proxy writes the acquire barrier made visible
  asm volatile("fence.proxy.async.global;" ::: "memory");
  for (; loaded < kBulkStages; ++loaded) {
    const char* src;
    if (!next(src, dsts[loaded], lens[loaded])) break;
    mbar_arrive_expect_tx(smem_u32(&full[loaded]), lens[loaded]);
    bulk_load(smem_u32(ring + loaded * kBulkChunk), src, lens[loaded], smem_u32(&full[loaded]));
  }
  for (int c = 0; c < loaded; ++c) {
    const int st = c % kBulkStages;
    mbar_wait(smem_u32(&full[st]), (uint32_t)(c / kBulkStages) & 1u);
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dsts[st]),
                 "r"(smem_u32(ring + st * kBulkChunk)), "r"(lens[st])
                 : "memory");
    bulk_commit();
    // refill the stage of chunk c-1 once its store has read shared memory (at most chunk c's
    // store group may still be reading)
    if (c >= 1) {
      const int ps = (c - 1) % kBulkStages;
      const char* src;
      char* d;
      uint32_t len;
      if (next(src, d, len)) {
        asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
        dsts[ps] = d;
        lens[ps] = len;
        mbar_arrive_expect_tx(smem_u32(&full[ps]), len);
        bulk_load(smem_u32(ring + ps * kBulkChunk), src, len, smem_u32(&full[ps]));
        ++loaded;
      }
    }
  }
  bulk_wait0();  // every store performed (and every load consumed) before the CTA's release barrier
}

// dst[i] = sum_p src_p[i] (bf16, fp32 accumulate, p = 0..world-1 in order); optional 2nd dst.
template <int W>
__device__ __forceinline__ void reduce_vecs(uint4* __restrict__ dst, uint4* __restrict__ dst2,
                                            const CommArgs& a, size_t src_off_bytes, size_t b, size_t e) {
  // R independent vectors per thread per iteration: R * W loads in flight
  constexpr int R = W <= 2 ? 8 : (W <= 4 ? 4 : 2);
  size_t i = b + threadIdx.x;
  for (; i + (R - 1) * kCommThreads < e; i += R * kCommThreads) {
    uint4 v[R][W];
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
      for (int p = 0; p < W; ++p)
        v[r][p] = ld_weak_v4(reinterpret_cast<const uint4*>(a.peer[p] + src_off_bytes) + i + r * kCommThreads);
#pragma unroll
    for (int r = 0; r < R; ++r) {
      float acc[8], f[8];
      unpack8(v[r][0], acc);
#pragma unroll
      for (int p = 1; p < W; ++p) {
        unpack8(v[r][p], f);
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[j] += f[j];
      }
      const uint4 o = pack8(acc);
      st_v4(dst + i + r * kCommThreads, o);
      if (dst2) st_v4(dst2 + i + r * kCommThreads, o);
    }
  }
  for (; i < e; i += kCommThreads) {
    uint4 v[W];
#pragma unroll
    for (int p = 0; p < W; ++p)
      v[p] = ld_weak_v4(reinterpret_cast<const uint4*>(a.peer[p] + src_off_bytes) + i);
    float acc[8], f[8];
    unpack8(v[0], acc);
#pragma unroll
    for (int p = 1; p < W; ++p) {
      unpack8(v[p], f);
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[j] += f[j];
    }
    const uint4 r = pack8(acc);
    st_v4(dst + i, r);
    if (dst2) st_v4(dst2 + i, r);
  }
}

__device__ __forceinline__ void reduce_vecs_dyn(uint4* __restrict__ dst, uint4* __restrict__ dst2,
                                                const CommArgs& a, size_t src_off_bytes, size_t b, size_t e) {
  switch (a.world) {
    case 1: reduce_vecs<1>(dst, dst2, a, src_off_bytes, b, e); break;
    case 2: reduce_vecs<2>(dst, dst2, a, src_off_bytes, b, e); break;
    case 3: reduce_vecs<3>(dst, dst2, a, src_off_bytes, b, e); break;
    case 4: reduce_vecs<4>(dst, dst2, a, src_off_bytes, b, e); break;
    case 5: reduce_vecs<5>(dst, dst2, a, src_off_bytes, b, e); break;
    case 6: reduce_vecs<6>(dst, dst2, a, src_off_bytes, b, e); break;
    case 7: reduce_vecs<7>(dst, dst2, a, src_off_bytes, b, e); break;
    default: reduce_vecs<8>(dst, dst2, a, src_off_bytes, b, e); break;
  }
}

__shared__ __align__(8) uint64_t bulk_bars[kBulkStages];
__device__ __forceinline__ uint8_t* bulk_ring() {
  extern __shared__ __align__(1024) uint8_t comm_dyn_smem[];
  return comm_dyn_smem;
}
__device__ __forceinline__ void bulk_init() {
  if (threadIdx.x == 0) {
    for (int i = 0; i < kBulkStages; ++i) kpo::sm100::mbar_init(kpo::sm100::smem_u32(&bulk_bars[i]), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
}

__global__ void __launch_bounds__(kCommThreads, 1)
    all_gather_kernel(CommArgs a, size_t sym_off, char* __restrict__ out, size_t bytes_per_rank) {
  trace_enter(a);
  bulk_init();
  __shared__ uint32_t base_epoch;
  if (threadIdx.x == 0) base_epoch = a.epoch[blockIdx.x];
  __syncthreads();
  const uint32_t e0 = base_epoch;
  cta_barrier(a, e0 + 1);  // every rank's shard is in its symmetric buffer
  const size_t nvec = bytes_per_rank / 16;
  size_t b, e;
  cta_slice(nvec, b, e);
  if (a.bulk) {
    if (threadIdx.x == 0 && e > b) {
      BulkSeg segs[KPO_MAX_WORLD];
      for (int k = 0; k < a.world; ++k) {
        const int p = (a.rank + k) % a.world;  // stagger peers across ranks
        segs[k] = {out + (size_t)p * bytes_per_rank + b * 16, a.peer[p] + sym_off + b * 16, (e - b) * 16};
      }
      bulk_copy_segs(segs, a.world, bulk_ring(), bulk_bars);
    }
  } else {
    for (int k = 0; k < a.world; ++k) {
      const int p = (a.rank + k) % a.world;  // stagger peers across ranks
      copy_vecs(reinterpret_cast<uint4*>(out + (size_t)p * bytes_per_rank),
                reinterpret_cast<const uint4*>(a.peer[p] + sym_off), b, e);
    }
  }
  cta_barrier(a, e0 + 2);  // nobody reuses its shard buffer before every peer has read it
  if (threadIdx.x == 0) a.epoch[blockIdx.x] = e0 + 2;
  trace_exit(a);
}

__global__ void __launch_bounds__(kCommThreads, 1)
    reduce_scatter_kernel(CommArgs a, size_t sym_off, char* __restrict__ out, size_t count) {
  trace_enter(a);
  __shared__ uint32_t base_epoch;
  if (threadIdx.x == 0) base_epoch = a.epoch[blockIdx.x];
  __syncthreads();
  const uint32_t e0 = base_epoch;
  cta_barrier(a, e0 + 1);
  const size_t nvec = count / 8;
  size_t b, e;
  cta_slice(nvec, b, e);
  reduce_vecs_dyn(reinterpret_cast<uint4*>(out), nullptr, a, sym_off + (size_t)a.rank * count * 2, b, e);
  cta_barrier(a, e0 + 2);
  if (threadIdx.x == 0) a.epoch[blockIdx.x] = e0 + 2;
  trace_exit(a);
}

__global__ void __launch_bounds__(kCommThreads, 1)
    all_reduce_kernel(CommArgs a, size_t sym_off, size_t stage_off, char* __restrict__ out, size_t count) {
  trace_enter(a);
  bulk_init();
  __shared__ uint32_t base_epoch;
  if (threadIdx.x == 0) base_epoch = a.epoch[blockIdx.x];
  __syncthreads();
  const uint32_t e0 = base_epoch;
  cta_barrier(a, e0 + 1);
  const size_t chunk = count / a.world;  // elements per rank chunk
  const size_t nvec = chunk / 8;
  size_t b, e;
  cta_slice(nvec, b, e);
  // phase 1: reduce my chunk from every rank -> my stage buffer and my output
  const size_t my_chunk_bytes = (size_t)a.rank * chunk * 2;
  reduce_vecs_dyn(reinterpret_cast<uint4*>(a.peer[a.rank] + stage_off + my_chunk_bytes),
                  reinterpret_cast<uint4*>(out + my_chunk_bytes), a, sym_off + my_chunk_bytes, b, e);
  cta_barrier(a, e0 + 2);  // slice blockIdx.x of every rank's chunk is reduced
  // phase 2: gather the other ranks' reduced chunks (same slice) from their stage buffers
  if (a.bulk) {
    if (threadIdx.x == 0 && e > b) {
      BulkSeg segs[KPO_MAX_WORLD];
      for (int k = 1; k < a.world; ++k) {
        const int p = (a.rank + k) % a.world;
        const size_t off = (size_t)p * chunk * 2 + b * 16;
        segs[k - 1] = {out + off, a.peer[p] + stage_off + off, (e - b) * 16};
      }
      bulk_copy_segs(segs, a.world - 1, bulk_ring(), bulk_bars);
    }
  } else {
    for (int k = 1; k < a.world; ++k) {
      const int p = (a.rank + k) % a.world;
      const size_t off = (size_t)p * chunk * 2;
      copy_vecs(reinterpret_cast<uint4*>(out + off),
                reinterpret_cast<const uint4*>(a.peer[p] + stage_off + off), b, e);
    }
  }
  cta_barrier(a, e0 + 3);
  if (threadIdx.x == 0) a.epoch[blockIdx.x] = e0 + 3;
  trace_exit(a);
}

}  // namespace kpo

using namespace kpo;

static size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

extern "C" int kpo_comm_create(int rank, int world, int device, size_t sym_bytes, int loopback, kpo_comm** out) {
  KPO_CHECK_ARG(out, "comm_create: null out");
  KPO_CHECK_ARG(world >= 1 && world <= KPO_MAX_WORLD, "comm_create: world must be in [1, %d]", KPO_MAX_WORLD);
  KPO_CHECK_ARG(rank >= 0 && rank < world, "comm_create: rank out of range");
  KPO_CHECK_ARG(sym_bytes > 0, "comm_create: sym_bytes must be > 0");
  KPO_CUDA(cudaSetDevice(device));
  kpo_comm* c = new kpo_comm();
  c->rank = rank;
  c->world = world;
  c->device = device;
  c->loopback = loopback ? 1 : 0;
  c->sym_bytes = align_up(sym_bytes, 256);
  c->flag_off = c->sym_bytes;
  c->alloc_bytes = c->flag_off + align_up(sizeof(uint32_t) * KPO_MAX_WORLD * KPO_MAX_CTAS, 256);
  auto fail = [&](cudaError_t e, const char* what) {
    set_error("comm_create: %s: %s", what, cudaGetErrorString(e));
    delete c;
    return KPO_ERR_CUDA;
  };
  cudaError_t e = cudaMalloc(&c->local, c->alloc_bytes);
  if (e != cudaSuccess) return fail(e, "cudaMalloc");
  cudaMemset(c->local + c->flag_off, 0, c->alloc_bytes - c->flag_off);
  e = cudaMalloc(&c->epoch, sizeof(uint32_t) * KPO_MAX_CTAS);
  if (e != cudaSuccess) return fail(e, "cudaMalloc(epoch)");
  cudaMemset(c->epoch, 0, sizeof(uint32_t) * KPO_MAX_CTAS);
  c->peer[rank] = c->local;
  if (c->loopback || world == 1) {
    for (int p = 0; p < world; ++p) {
      if (p == rank) continue;
      e = cudaMalloc(&c->virt[p], c->alloc_bytes);
      if (e != cudaSuccess) return fail(e, "cudaMalloc(loopback peer)");
      cudaMemset(c->virt[p], 0, c->alloc_bytes);
      c->peer[p] = c->virt[p];
    }
    c->opened = true;
  } else {
    e = cudaIpcGetMemHandle(&c->handle, c->local);
    if (e != cudaSuccess) return fail(e, "cudaIpcGetMemHandle");
  }
  int optin = 0;
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
  // full-SM reservation: static + dynamic shared memory == the per-block opt-in maximum, which
  // together with the 1 KB per-CTA system reservation is the whole SM's shared memory.
  const void* kernels[] = {(const void*)all_gather_kernel, (const void*)reduce_scatter_kernel,
                           (const void*)all_reduce_kernel};
  size_t max_static = 0;
  for (const void* k : kernels) {
    cudaFuncAttributes fa;
    e = cudaFuncGetAttributes(&fa, k);
    if (e != cudaSuccess) return fail(e, "cudaFuncGetAttributes");
    if (fa.sharedSizeBytes > max_static) max_static = fa.sharedSizeBytes;
  }
  c->smem_bytes = optin - (int)max_static;
  for (const void* k : kernels) {
    e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, c->smem_bytes);
    if (e != cudaSuccess) return fail(e, "cudaFuncSetAttribute(smem)");
  }
  e = cudaDeviceSynchronize();
  if (e != cudaSuccess) return fail(e, "sync");
  *out = c;
  return KPO_OK;
}

extern "C" int kpo_comm_ipc_handle(kpo_comm* c, void* handle_out) {
  KPO_CHECK_ARG(c && handle_out, "comm_ipc_handle: null");
  if (c->loopback || c->world == 1) {
    memset(handle_out, 0, KPO_IPC_HANDLE_BYTES);
    return KPO_OK;
  }
  static_assert(sizeof(cudaIpcMemHandle_t) == KPO_IPC_HANDLE_BYTES, "IPC handle size");
  memcpy(handle_out, &c->handle, KPO_IPC_HANDLE_BYTES);
  return KPO_OK;
}

extern "C" int kpo_comm_open_peers(kpo_comm* c, const void* handles) {
  KPO_CHECK_ARG(c && handles, "comm_open_peers: null");
  if (c->opened) return KPO_OK;
  KPO_CUDA(cudaSetDevice(c->device));
  const char* h = (const char*)handles;
  for (int p = 0; p < c->world; ++p) {
    if (p == c->rank) continue;
    cudaIpcMemHandle_t hp;
    memcpy(&hp, h + (size_t)p * KPO_IPC_HANDLE_BYTES, KPO_IPC_HANDLE_BYTES);
    void* ptr = nullptr;
    KPO_CUDA(cudaIpcOpenMemHandle(&ptr, hp, cudaIpcMemLazyEnablePeerAccess));
    c->peer[p] = (char*)ptr;
  }
  c->opened = true;
  return KPO_OK;
}

extern "C" void* kpo_comm_sym_ptr(kpo_comm* c) { return c ? c->local : nullptr; }
extern "C" void* kpo_comm_peer_ptr(kpo_comm* c, int p) {
  if (!c || p < 0 || p >= c->world) return nullptr;
  return c->peer[p];
}
extern "C" int kpo_comm_max_ctas(kpo_comm* c) {
  (void)c;
  int n = num_sms();
  return n < KPO_MAX_CTAS ? n : KPO_MAX_CTAS;
}

extern "C" int kpo_comm_destroy(kpo_comm* c) {
  if (!c) return KPO_OK;
  cudaSetDevice(c->device);
  cudaDeviceSynchronize();
  for (int p = 0; p < c->world; ++p) {
    if (p == c->rank) continue;
    if (c->virt[p]) cudaFree(c->virt[p]);
    else if (c->peer[p]) cudaIpcCloseMemHandle(c->peer[p]);
  }
  if (c->local) cudaFree(c->local);
  if (c->epoch) cudaFree(c->epoch);
  delete c;
  return KPO_OK;
}

extern "C" int kpo_comm_trace(kpo_comm* c, int64_t* buf, int n_slots) {
  KPO_CHECK_ARG(c, "comm_trace: null comm");
  c->trace = buf;
  c->trace_slots = buf ? n_slots : 0;
  c->trace_next = 0;
  return KPO_OK;
}

extern "C" int kpo_set_launch_completion_event(kpo_comm* c, void* ev) {
  KPO_CHECK_ARG(c, "set_launch_completion_event: null comm");
  c->launch_evt = (cudaEvent_t)ev;
  return KPO_OK;
}

static int prep_args(kpo_comm* c, int ncta, CommArgs& a) {
  KPO_CHECK_ARG(c, "collective: null comm");
  if (!c->opened) {
    set_error("collective: peers not opened (call kpo_comm_open_peers)");
    return KPO_ERR_STATE;
  }
  KPO_CHECK_ARG(ncta >= 1 && ncta <= kpo_comm_max_ctas(c), "collective: ncta %d out of [1, %d]", ncta,
                kpo_comm_max_ctas(c));
  a.bulk = 0;
  for (int p = 0; p < KPO_MAX_WORLD; ++p) {
    a.peer[p] = p < c->world ? c->peer[p] : nullptr;
    a.peer_flags[p] = p < c->world ? (uint32_t*)(c->peer[p] + c->flag_off) : nullptr;
  }
  a.my_flags = (uint32_t*)(c->local + c->flag_off);
  a.epoch = c->epoch;
  a.rank = c->rank;
  a.world = c->world;
  a.loopback = (c->loopback || c->world == 1) ? 1 : 0;
  a.trace = nullptr;
  if (c->trace && c->trace_next < c->trace_slots) {
    a.trace = c->trace + (size_t)c->trace_next * KPO_MAX_CTAS * 4;
    c->trace_next++;
  }
  return KPO_OK;
}

template <typename... KArgs, typename... Args>
static int launch_comm(kpo_comm* c, void (*kernel)(KArgs...), int ncta, cudaStream_t s, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(ncta);
  cfg.blockDim = dim3(kCommThreads);
  cfg.dynamicSmemBytes = (size_t)c->smem_bytes;  // full-SM reservation: owns ncta SMs
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  int na = 0;
  if (ncta % 2 == 0) {
    // pack the collective's CTAs two per TPC so whole TPCs stay free for the CTA-pair GEMM
    attr[na].id = cudaLaunchAttributeClusterDimension;
    attr[na].val.clusterDim.x = 2;
    attr[na].val.clusterDim.y = 1;
    attr[na].val.clusterDim.z = 1;
    ++na;
  }
  if (c->launch_evt) {
    attr[na].id = cudaLaunchAttributeLaunchCompletionEvent;
    attr[na].val.launchCompletionEvent.event = c->launch_evt;
    attr[na].val.launchCompletionEvent.flags = 0;
    ++na;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  KPO_CUDA(cudaLaunchKernelEx(&cfg, kernel, args...));
  return KPO_OK;
}

extern "C" int kpo_all_gather(kpo_comm* c, size_t sym_off, void* out, size_t bytes_per_rank, int ncta,
                              void* stream) {
  CommArgs a;
  int st = prep_args(c, ncta, a);
  if (st) return st;
  KPO_CHECK_ARG(out && bytes_per_rank % 16 == 0 && sym_off % 16 == 0, "all_gather: 16B alignment required");
  KPO_CHECK_ARG(sym_off + bytes_per_rank <= c->sym_bytes, "all_gather: source exceeds symmetric buffer");
  a.bulk = choose_bulk(bytes_per_rank * (size_t)c->world / (size_t)ncta);
  return launch_comm(c, all_gather_kernel, ncta, (cudaStream_t)stream, a, sym_off, (char*)out, bytes_per_rank);
}

extern "C" int kpo_reduce_scatter(kpo_comm* c, size_t sym_off, void* out, size_t count, int ncta, void* stream) {
  CommArgs a;
  int st = prep_args(c, ncta, a);
  if (st) return st;
  KPO_CHECK_ARG(out && count % 8 == 0 && sym_off % 16 == 0, "reduce_scatter: count %% 8 and 16B alignment");
  KPO_CHECK_ARG(sym_off + count * 2 * c->world <= c->sym_bytes, "reduce_scatter: source exceeds symmetric buffer");
  return launch_comm(c, reduce_scatter_kernel, ncta, (cudaStream_t)stream, a, sym_off, (char*)out, count);
}

extern "C" int kpo_all_reduce(kpo_comm* c, size_t sym_off, size_t stage_off, void* out, size_t count, int ncta,
                              void* stream) {
  CommArgs a;
  int st = prep_args(c, ncta, a);
  if (st) return st;
  KPO_CHECK_ARG(out && count % (8 * (size_t)c->world) == 0 && sym_off % 16 == 0 && stage_off % 16 == 0,
                "all_reduce: count must be a multiple of 8*world, offsets 16B aligned");
  KPO_CHECK_ARG(sym_off + count * 2 <= c->sym_bytes && stage_off + count * 2 <= c->sym_bytes,
                "all_reduce: buffers exceed symmetric buffer");
  KPO_CHECK_ARG(stage_off >= sym_off + count * 2 || sym_off >= stage_off + count * 2,
                "all_reduce: stage and input regions overlap");
  a.bulk = choose_bulk(count * 2 / (size_t)ncta);
  return launch_comm(c, all_reduce_kernel, ncta, (cudaStream_t)stream, a, sym_off, stage_off, (char*)out, count);
}
