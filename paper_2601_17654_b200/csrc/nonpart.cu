// nonpart.cu — the non-partition work of a microbatch: token embedding (fwd gather / bwd
// scatter-add) and the fused softmax cross-entropy over the LM-head logits (loss + dlogits in one
// kernel).  The LM-head GEMMs themselves are gemm_sm100.cu.
//
// These replace the reference's analytic non-partition cost table (cli.py:227-241, fed into
// MicrobatchSpec.non_partition_costs, compose.py:79-102): the engine measures them on hardware
// (nonpartition.py).  All three are HBM-bound; roofline = algorithmic bytes / copy bandwidth.
#include "common.cuh"

namespace kpo {

// ===================================================================== embedding
// out[t, :] = table[ids[t], :]  — one warp per token row, 16-byte vectors.
__global__ void __launch_bounds__(256) embedding_fwd_kernel(const int32_t* __restrict__ ids,
                                                            const __nv_bfloat16* __restrict__ table,
                                                            __nv_bfloat16* __restrict__ out, int64_t T, int64_t h,
                                                            int64_t vocab, int* __restrict__ bad) {
  KPO_PDL_ENTRY();
  const int64_t t = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (t >= T) return;
  const int32_t id = ids[t];
  uint4* o = reinterpret_cast<uint4*>(out + t * h);
  if (id < 0 || id >= vocab) {  // out-of-range token: zero row, flag it (reported by the host)
    for (int64_t c = lane; c < h / 8; c += 32) o[c] = make_uint4(0, 0, 0, 0);
    if (lane == 0) atomicOr(bad, 1);
    return;
  }
  const uint4* src = reinterpret_cast<const uint4*>(table + (int64_t)id * h);
#pragma unroll 4
  for (int64_t c = lane; c < h / 8; c += 32) o[c] = ld_nc_v4(src + c);
}

// dtable[ids[t], :] += dy[t, :]  (fp32 gradient table) — one warp per token row, v4 fp32 reductions
// straight into L2 (repeated tokens reduce in arbitrary order: fp32 rounding differs by ulps).
__global__ void __launch_bounds__(256) embedding_bwd_kernel(const int32_t* __restrict__ ids,
                                                            const __nv_bfloat16* __restrict__ dy,
                                                            float* __restrict__ dtable, int64_t T, int64_t h,
                                                            int64_t vocab) {
  KPO_PDL_ENTRY();
  const int64_t t = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (t >= T) return;
  const int32_t id = ids[t];
  if (id < 0 || id >= vocab) return;
  const uint4* src = reinterpret_cast<const uint4*>(dy + t * h);
  float* dst = dtable + (int64_t)id * h;
#pragma unroll 2
  for (int64_t c = lane; c < h / 8; c += 32) {
    float f[8];
    unpack8(ld_nc_v4(src + c), f);
    float* p = dst + c * 8;
    asm volatile("red.global.add.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(f[0]), "f"(f[1]), "f"(f[2]), "f"(f[3])
                 : "memory");
    asm volatile("red.global.add.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p + 4), "f"(f[4]), "f"(f[5]), "f"(f[6]),
                 "f"(f[7])
                 : "memory");
  }
}

// ===================================================================== fused cross-entropy
// One CTA per token row of logits [T, V] (row stride ld):
//   pass 1: online (max, sum of 2^(x*log2e - max)) over the row, 8 bf16 per 16-byte load;
//   loss[t] = ln(sum) + max*ln2 - x[label]   (natural-log units, i.e. -log softmax(x)[label])
//   pass 2: dlogits = (softmax(x) - onehot(label)) * grad_scale, written in bf16 (may alias logits:
//           every element is read before it is overwritten by the same thread).
// The row (V = 128256 -> 250 KB) is re-read from L2 in pass 2: 148 resident rows ~ 37 MB << 126 MB.
constexpr int kCeThreads = 512;
constexpr float kLog2eF = 1.4426950408889634f;
constexpr float kLn2F = 0.6931471805599453f;

__device__ __forceinline__ void ms_merge(float& m, float& s, float m2, float s2) {
  const float mn = fmaxf(m, m2);
  if (mn == -INFINITY) return;
  s = s * exp2f(m - mn) + s2 * exp2f(m2 - mn);
  m = mn;
}

__global__ void __launch_bounds__(kCeThreads) cross_entropy_kernel(const __nv_bfloat16* logits,
                                                                    __nv_bfloat16* dlogits,
                                                                    const int32_t* __restrict__ labels,
                                                                    float* __restrict__ loss, int64_t V,
                                                                    int64_t ld, float grad_scale,
                                                                    int ignore_index) {
  KPO_PDL_ENTRY();
  const int64_t t = blockIdx.x;
  const __nv_bfloat16* row = logits + t * ld;
  __nv_bfloat16* drow = dlogits + t * ld;
  const int32_t label = labels[t];
  const int64_t nv = V / 8;  // V % 8 == 0 (checked by the host)
  const uint4* rv = reinterpret_cast<const uint4*>(row);
  // ---- pass 1 (values in log2 units)
  float m = -INFINITY, s = 0.f;
  for (int64_t c = threadIdx.x; c < nv; c += kCeThreads) {
    float f[8];
    unpack8(rv[c], f);
    float cm = f[0];
#pragma unroll
    for (int i = 1; i < 8; ++i) cm = fmaxf(cm, f[i]);
    cm *= kLog2eF;
    const float mn = fmaxf(m, cm);
    float cs = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i) cs += exp2f(fmaf(f[i], kLog2eF, -mn));
    s = s * exp2f(m - mn) + cs;
    m = mn;
  }
  // warp then block reduction of (m, s)
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float m2 = __shfl_xor_sync(0xffffffffu, m, o), s2 = __shfl_xor_sync(0xffffffffu, s, o);
    ms_merge(m, s, m2, s2);
  }
  __shared__ float sm[kCeThreads / 32], ss[kCeThreads / 32];
  __shared__ float lse2_sh;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) {
    sm[warp] = m;
    ss[warp] = s;
  }
  __syncthreads();
  if (warp == 0) {
    m = lane < kCeThreads / 32 ? sm[lane] : -INFINITY;
    s = lane < kCeThreads / 32 ? ss[lane] : 0.f;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float m2 = __shfl_xor_sync(0xffffffffu, m, o), s2 = __shfl_xor_sync(0xffffffffu, s, o);
      ms_merge(m, s, m2, s2);
    }
    if (lane == 0) {
      const float lse2 = m + log2f(s);  // log2 of the partition function
      lse2_sh = lse2;
      const bool valid = label != ignore_index && label >= 0 && label < V;
      loss[t] = valid ? (lse2 - bf2f(row[label]) * kLog2eF) * kLn2F : 0.f;
    }
  }
  __syncthreads();
  const float lse2 = lse2_sh;
  const bool valid = label != ignore_index && label >= 0 && label < V;
  const float gs = valid ? grad_scale : 0.f;
  // ---- pass 2
  uint4* dv = reinterpret_cast<uint4*>(drow);
  for (int64_t c = threadIdx.x; c < nv; c += kCeThreads) {
    float f[8];
    unpack8(rv[c], f);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const float p = exp2f(fmaf(f[i], kLog2eF, -lse2));
      f[i] = (p - ((c * 8 + i) == label ? 1.f : 0.f)) * gs;
    }
    dv[c] = pack8(f);
  }
}

}  // namespace kpo

using namespace kpo;

extern "C" int kpo_embedding_fwd(const int32_t* ids, const void* table, void* out, int64_t tokens, int64_t hidden,
                                 int64_t vocab, int* bad_flag, void* stream) {
  KPO_CHECK_ARG(ids && table && out && bad_flag, "embedding_fwd: null pointer");
  KPO_CHECK_ARG(hidden > 0 && hidden % 8 == 0 && vocab > 0 && tokens >= 0,
                "embedding_fwd: hidden must be a positive multiple of 8");
  KPO_CHECK_ARG(((uintptr_t)table & 15) == 0 && ((uintptr_t)out & 15) == 0, "embedding_fwd: 16B alignment");
  if (tokens == 0) return KPO_OK;
  KPO_CUDA(::kpo::pdl_launch(embedding_fwd_kernel, (unsigned)((tokens + 7) / 8), 256, 0, (cudaStream_t)stream, 
      ids, (const __nv_bfloat16*)table, (__nv_bfloat16*)out, tokens, hidden, vocab, bad_flag));
  KPO_LAUNCH_CHECK();
  return KPO_OK;
}

extern "C" int kpo_embedding_bwd(const int32_t* ids, const void* dy, float* dtable, int64_t tokens, int64_t hidden,
                                 int64_t vocab, void* stream) {
  KPO_CHECK_ARG(ids && dy && dtable, "embedding_bwd: null pointer");
  KPO_CHECK_ARG(hidden > 0 && hidden % 8 == 0 && vocab > 0 && tokens >= 0,
                "embedding_bwd: hidden must be a positive multiple of 8");
  KPO_CHECK_ARG(((uintptr_t)dy & 15) == 0 && ((uintptr_t)dtable & 15) == 0, "embedding_bwd: 16B alignment");
  if (tokens == 0) return KPO_OK;
  KPO_CUDA(::kpo::pdl_launch(embedding_bwd_kernel, (unsigned)((tokens + 7) / 8), 256, 0, (cudaStream_t)stream, 
      ids, (const __nv_bfloat16*)dy, dtable, tokens, hidden, vocab));
  KPO_LAUNCH_CHECK();
  return KPO_OK;
}

extern "C" int kpo_cross_entropy(const void* logits, void* dlogits, const int32_t* labels, float* loss,
                                 int64_t tokens, int64_t vocab, int64_t ld, float grad_scale, int ignore_index,
                                 void* stream) {
  KPO_CHECK_ARG(logits && dlogits && labels && loss, "cross_entropy: null pointer");
  KPO_CHECK_ARG(vocab > 0 && vocab % 8 == 0 && ld >= vocab && ld % 8 == 0,
                "cross_entropy: vocab and row stride must be positive multiples of 8");
  KPO_CHECK_ARG(((uintptr_t)logits & 15) == 0 && ((uintptr_t)dlogits & 15) == 0, "cross_entropy: 16B alignment");
  if (tokens == 0) return KPO_OK;
  KPO_CUDA(::kpo::pdl_launch(cross_entropy_kernel, (unsigned)tokens, kCeThreads, 0, (cudaStream_t)stream, 
      (const __nv_bfloat16*)logits, (__nv_bfloat16*)dlogits, labels, loss, vocab, ld, grad_scale, ignore_index));
  KPO_LAUNCH_CHECK();
  return KPO_OK;
}
