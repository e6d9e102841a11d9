// attention.cu — causal GQA flash attention forward/backward (bf16, fp32 softmax statistics).
//
// Replaces the reference's abstract compute-bound "attention_core" kernel (workloads.py:47).
// Round-1 implementation: register-tiled flash attention on the warp-level tensor-core path
// (mma.sync m16n8k16, ldmatrix from XOR-swizzled shared memory, cp.async double buffering).
// Forward: one CTA = 128 query rows of one q head (8 warps x 16 rows), 64-key blocks.
// Backward: one CTA = 64 keys of one kv head (4 warps x 16 keys); it loops over every q head of
// the GQA group and every causal query block, so dK/dV accumulate in registers without atomics;
// dQ accumulates in fp32 through atomics and is converted by a small epilogue kernel.
#include "common.cuh"

namespace kpo {
int attn_fwd_tcgen05(const void* q, const void* k, const void* v, void* o, float* lse, int64_t T, int hq, int hkv,
                     int d, int64_t qs, int64_t ks, int64_t vs, int64_t os, float scale, int causal, cudaStream_t st);
int attn_bwd_tcgen05_main(const void* q, const void* k, const void* v, const void* dout, const float* lse,
                          const float* dvec, float* dq_acc, void* dk, void* dv, int64_t T, int hq, int hkv, int d,
                          int64_t qs, int64_t ks, int64_t vs, int64_t os, int64_t dks, int64_t dvs, float scale,
                          int causal, float* dkv_acc, int split_group, int qsplit_tiles, int qchunks,
                          cudaStream_t st, const float* rope_table);
int attn_bwd_tcgen05_split(const void* q, const void* k, const void* v, const void* o, const void* dout,
                           const float* lse, float* dvec, void* dq, void* dk, void* dv, int64_t T, int hq, int hkv,
                           int d, int64_t qs, int64_t ks, int64_t vs, int64_t os, int64_t dqs, int64_t dks,
                           int64_t dvs, float scale, int causal, float* dkv_acc, int split_group, int qsplit_tiles,
                           int qchunks, cudaStream_t st, const float* rope_table);
}

namespace kpo {
namespace attn {

__device__ __forceinline__ uint32_t s_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, bool valid) {
  const int n = valid ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(n) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__device__ __forceinline__ void mma16816(float* c, const uint32_t* a, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 h = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&h);
}

// Byte offset of (row, col) in a [rows][COLS] bf16 tile with 16-byte chunks XOR-swizzled by row.
template <int COLS>
__device__ __forceinline__ uint32_t swz(int row, int col) {
  return (uint32_t)(row * COLS * 2 + ((((col >> 3) ^ (row & 7))) << 4) + (col & 7) * 2);
}

// Async load of a [ROWS][D] tile whose rows are tokens row0.. (stride `stride` elements).
template <int ROWS, int D, int NT>
__device__ __forceinline__ void load_tile(uint32_t sbase, const __nv_bfloat16* g, int64_t stride, int row0, int T) {
  constexpr int CH = D / 8;
  for (int i = threadIdx.x; i < ROWS * CH; i += NT) {
    const int r = i / CH, c = i % CH;
    const int tok = row0 + r;
    const bool ok = tok < T;
    const __nv_bfloat16* src = g + (int64_t)(ok ? tok : 0) * stride + c * 8;
    cp_async16(sbase + swz<D>(r, c * 8), src, ok);
  }
}

constexpr float kLog2e = 1.4426950408889634f;

// ============================================================================ forward
template <int D>
struct FwdCfg {
  static constexpr int BM = 128, BN = 64, WARPS = 8, NT = WARPS * 32;
  static constexpr int Q_BYTES = BM * D * 2, KV_BYTES = BN * D * 2;
  static constexpr int SMEM = Q_BYTES + 4 * KV_BYTES;
};

template <int D>
__global__ void __launch_bounds__(256, 1)
    attn_fwd_kernel(const __nv_bfloat16* __restrict__ q, const __nv_bfloat16* __restrict__ k,
                    const __nv_bfloat16* __restrict__ v, __nv_bfloat16* __restrict__ o, float* __restrict__ lse,
                    int T, int hq, int hkv, int64_t qs, int64_t ks, int64_t vs, int64_t os, float scale_log2,
                    int causal) {
  KPO_PDL_ENTRY();
  using CF = FwdCfg<D>;
  constexpr int BM = CF::BM, BN = CF::BN, NT = CF::NT;
  extern __shared__ __align__(128) uint8_t smem[];
  const uint32_t sQ = s_u32(smem);
  const uint32_t sK0 = sQ + CF::Q_BYTES;
  const uint32_t sV0 = sK0 + 2 * CF::KV_BYTES;

  const int mblk = gridDim.x - 1 - blockIdx.x;  // longest causal rows first
  const int h = blockIdx.y;
  const int kvh = h / (hq / hkv);
  const int m0 = mblk * BM;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  const __nv_bfloat16* qg = q + (int64_t)h * D;
  const __nv_bfloat16* kg = k + (int64_t)kvh * D;
  const __nv_bfloat16* vg = v + (int64_t)kvh * D;

  int nblocks = (T + BN - 1) / BN;
  if (causal) nblocks = min(nblocks, (m0 + BM + BN - 1) / BN);

  load_tile<BM, D, NT>(sQ, qg, qs, m0, T);
  load_tile<BN, D, NT>(sK0, kg, ks, 0, T);
  load_tile<BN, D, NT>(sV0, vg, vs, 0, T);
  cp_commit();

  float o_acc[D / 8][4];
#pragma unroll
  for (int i = 0; i < D / 8; ++i) o_acc[i][0] = o_acc[i][1] = o_acc[i][2] = o_acc[i][3] = 0.f;
  float row_m[2] = {-INFINITY, -INFINITY}, row_l[2] = {0.f, 0.f};
  uint32_t qf[D / 16][4];
  const int wr0 = warp * 16;  // warp's first row within the tile
  const int qrow[2] = {m0 + wr0 + (lane >> 2), m0 + wr0 + (lane >> 2) + 8};

  for (int j = 0; j < nblocks; ++j) {
    const int buf = j & 1;
    if (j + 1 < nblocks) {
      load_tile<BN, D, NT>(sK0 + (buf ^ 1) * CF::KV_BYTES, kg, ks, (j + 1) * BN, T);
      load_tile<BN, D, NT>(sV0 + (buf ^ 1) * CF::KV_BYTES, vg, vs, (j + 1) * BN, T);
    }
    cp_commit();
    cp_wait<1>();
    __syncthreads();
    if (j == 0) {
#pragma unroll
      for (int kk = 0; kk < D / 16; ++kk) {
        const int r = wr0 + (lane & 7) + ((lane >> 3) & 1) * 8;
        const int c = kk * 16 + (lane >> 4) * 8;
        ldsm_x4(sQ + swz<D>(r, c), qf[kk][0], qf[kk][1], qf[kk][2], qf[kk][3]);
      }
    }
    const uint32_t sK = sK0 + buf * CF::KV_BYTES, sV = sV0 + buf * CF::KV_BYTES;
    // S = Q K^T : 16 rows x 64 keys per warp
    float s[BN / 8][4];
#pragma unroll
    for (int i = 0; i < BN / 8; ++i) s[i][0] = s[i][1] = s[i][2] = s[i][3] = 0.f;
#pragma unroll
    for (int kk = 0; kk < D / 16; ++kk) {
#pragma unroll
      for (int np = 0; np < BN / 16; ++np) {
        uint32_t b0, b1, b2, b3;
        const int r = np * 16 + (lane & 7) + (lane >> 4) * 8;
        const int c = kk * 16 + ((lane >> 3) & 1) * 8;
        ldsm_x4(sK + swz<D>(r, c), b0, b1, b2, b3);
        mma16816(s[2 * np], qf[kk], b0, b1);
        mma16816(s[2 * np + 1], qf[kk], b2, b3);
      }
    }
    // scale, mask, online softmax (log2 domain)
    const int kbase = j * BN;
    const bool need_mask = (causal && kbase + BN > m0 + wr0) || (kbase + BN > T);
#pragma unroll
    for (int i = 0; i < BN / 8; ++i) {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        float x = s[i][e] * scale_log2;
        if (need_mask) {
          const int key = kbase + i * 8 + (lane & 3) * 2 + (e & 1);
          const int qr = qrow[e >> 1];
          if (key >= T || (causal && key > qr)) x = -INFINITY;
        }
        s[i][e] = x;
      }
    }
    float mnew[2], corr[2];
#pragma unroll
    for (int hh = 0; hh < 2; ++hh) {
      float mx = row_m[hh];
#pragma unroll
      for (int i = 0; i < BN / 8; ++i) mx = fmaxf(mx, fmaxf(s[i][2 * hh], s[i][2 * hh + 1]));
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
      mnew[hh] = mx;
      corr[hh] = (row_m[hh] == -INFINITY) ? 0.f : exp2f(row_m[hh] - mx);
      row_m[hh] = mx;
    }
    float lsum[2] = {0.f, 0.f};
#pragma unroll
    for (int i = 0; i < BN / 8; ++i) {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float mm = mnew[e >> 1];
        const float p = (mm == -INFINITY) ? 0.f : exp2f(s[i][e] - mm);
        s[i][e] = p;
        lsum[e >> 1] += p;
      }
    }
#pragma unroll
    for (int hh = 0; hh < 2; ++hh) row_l[hh] = row_l[hh] * corr[hh] + lsum[hh];
#pragma unroll
    for (int i = 0; i < D / 8; ++i) {
      o_acc[i][0] *= corr[0];
      o_acc[i][1] *= corr[0];
      o_acc[i][2] *= corr[1];
      o_acc[i][3] *= corr[1];
    }
    // O += P V
#pragma unroll
    for (int kk = 0; kk < BN / 16; ++kk) {
      uint32_t pa[4];
      pa[0] = pack_bf16(s[2 * kk][0], s[2 * kk][1]);
      pa[1] = pack_bf16(s[2 * kk][2], s[2 * kk][3]);
      pa[2] = pack_bf16(s[2 * kk + 1][0], s[2 * kk + 1][1]);
      pa[3] = pack_bf16(s[2 * kk + 1][2], s[2 * kk + 1][3]);
#pragma unroll
      for (int np = 0; np < D / 16; ++np) {
        uint32_t b0, b1, b2, b3;
        const int r = kk * 16 + (lane & 7) + ((lane >> 3) & 1) * 8;
        const int c = np * 16 + (lane >> 4) * 8;
        ldsm_x4_t(sV + swz<D>(r, c), b0, b1, b2, b3);
        mma16816(o_acc[2 * np], pa, b0, b1);
        mma16816(o_acc[2 * np + 1], pa, b2, b3);
      }
    }
    __syncthreads();
  }
  // finalize
#pragma unroll
  for (int hh = 0; hh < 2; ++hh) {
    float l = row_l[hh];
    l += __shfl_xor_sync(0xffffffffu, l, 1);
    l += __shfl_xor_sync(0xffffffffu, l, 2);
    row_l[hh] = l;
  }
#pragma unroll
  for (int hh = 0; hh < 2; ++hh) {
    const int r = qrow[hh];
    if (r >= T) continue;
    const float inv = 1.f / row_l[hh];
    __nv_bfloat16* orow = o + (int64_t)r * os + (int64_t)h * D;
#pragma unroll
    for (int i = 0; i < D / 8; ++i) {
      const int c = i * 8 + (lane & 3) * 2;
      *reinterpret_cast<uint32_t*>(orow + c) = pack_bf16(o_acc[i][2 * hh] * inv, o_acc[i][2 * hh + 1] * inv);
    }
    if ((lane & 3) == 0) lse[(int64_t)h * T + r] = (row_m[hh] + log2f(row_l[hh])) / kLog2e;
  }
}

// ============================================================================ backward
// Dv[h][t] = sum_d dO*O ; dq_acc zeroed.
template <int D>
__global__ void attn_bwd_pre_kernel(const __nv_bfloat16* __restrict__ o, const __nv_bfloat16* __restrict__ dout,
                                    float* __restrict__ dvec, float* __restrict__ dq_acc, int T, int hq,
                                    int64_t os) {
  // D[h][t] = sum_d O[t,h,d] dO[t,h,d] and zero the fp32 dQ accumulator: one thread per 8 elements,
  // D/8 consecutive lanes per (t, h) row, reduced with shuffles inside the lane group
  KPO_PDL_ENTRY();
  constexpr int G = D / 8;  // lanes per row (16 for D = 128, 8 for D = 64)
  const int64_t gt = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t row = gt / G;
  const int c = (int)(gt % G) * 8;
  const bool ok = row < (int64_t)T * hq;
  const int t = ok ? (int)(row / hq) : 0, h = ok ? (int)(row % hq) : 0;
  float acc = 0.f;
  if (ok) {
    float a[8], b[8];
    unpack8(*reinterpret_cast<const uint4*>(o + (int64_t)t * os + (int64_t)h * D + c), a);
    unpack8(*reinterpret_cast<const uint4*>(dout + (int64_t)t * os + (int64_t)h * D + c), b);
#pragma unroll
    for (int j = 0; j < 8; ++j) acc += a[j] * b[j];
  }
#pragma unroll
  for (int off = G / 2; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
  if (!ok) return;
  if (c == 0) dvec[(int64_t)h * T + t] = acc;
  float4* dq = reinterpret_cast<float4*>(dq_acc + ((int64_t)t * hq + h) * D + c);
  dq[0] = make_float4(0.f, 0.f, 0.f, 0.f);
  dq[1] = make_float4(0.f, 0.f, 0.f, 0.f);
}

template <int D>
__global__ void attn_bwd_post_kernel(const float* __restrict__ dq_acc, __nv_bfloat16* __restrict__ dq, int T, int hq,
                                     int64_t dqs) {
  KPO_PDL_ENTRY();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;  // one thread per 8 elements
  const int64_t total = (int64_t)T * hq * D / 8;
  if (i >= total) return;
  const int64_t e = i * 8;
  const int64_t th = e / D;
  const int c = (int)(e % D);
  const int t = (int)(th / hq), h = (int)(th % hq);
  const float4* src = reinterpret_cast<const float4*>(dq_acc + e);
  float4 a = src[0], b = src[1];
  float f[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
  *reinterpret_cast<uint4*>(dq + (int64_t)t * dqs + (int64_t)h * D + c) = pack8(f);
}

// fp32 accumulator -> bf16 with the inverse rotary embedding of token t (pairs (i, i + D/2));
// one thread per 8 pairs.  Used for dQ (and split-mode dK) when the forward rotated q / k in the
// QKV GEMM epilogue.
template <int D>
__global__ void attn_bwd_post_rope_kernel(const float* __restrict__ acc, __nv_bfloat16* __restrict__ out, int T,
                                          int heads, int64_t os, const float2* __restrict__ cs) {
  KPO_PDL_ENTRY();
  constexpr int H = D / 2;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t total = (int64_t)T * heads * (H / 8);
  if (i >= total) return;
  const int64_t th = i / (H / 8);
  const int i0 = (int)(i % (H / 8)) * 8;
  const int t = (int)(th / heads), h = (int)(th % heads);
  const float* src = acc + th * D;
  const float4 a0 = *reinterpret_cast<const float4*>(src + i0), a1 = *reinterpret_cast<const float4*>(src + i0 + 4);
  const float4 b0 = *reinterpret_cast<const float4*>(src + H + i0), b1 = *reinterpret_cast<const float4*>(src + H + i0 + 4);
  const float xa[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
  const float xb[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
  float oa[8], ob[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const float2 r = cs[(int64_t)t * H + i0 + j];
    oa[j] = xa[j] * r.x + xb[j] * r.y;
    ob[j] = xb[j] * r.x - xa[j] * r.y;
  }
  __nv_bfloat16* dst = out + (int64_t)t * os + (int64_t)h * D;
  *reinterpret_cast<uint4*>(dst + i0) = pack8(oa);
  *reinterpret_cast<uint4*>(dst + H + i0) = pack8(ob);
}

template <int D>
struct BwdCfg {
  static constexpr int BN = 64, BM = 64, WARPS = 4, NT = WARPS * 32;
  static constexpr int KV_BYTES = BN * D * 2, QB = BM * D * 2, DS_BYTES = BN * BM * 2;
  static constexpr int OFF_K = 0, OFF_V = KV_BYTES, OFF_Q = 2 * KV_BYTES, OFF_DO = OFF_Q + 2 * QB;
  static constexpr int OFF_DS = OFF_DO + 2 * QB, OFF_STAT = OFF_DS + DS_BYTES;
  static constexpr int SMEM = OFF_STAT + 2 * 2 * BM * 4;
};

template <int D>
__global__ void __launch_bounds__(128, 2)
    attn_bwd_kernel(const __nv_bfloat16* __restrict__ q, const __nv_bfloat16* __restrict__ k,
                    const __nv_bfloat16* __restrict__ v, const __nv_bfloat16* __restrict__ dout,
                    const float* __restrict__ lse, const float* __restrict__ dvec, float* __restrict__ dq_acc,
                    __nv_bfloat16* __restrict__ dk, __nv_bfloat16* __restrict__ dv, int T, int hq, int hkv,
                    int64_t qs, int64_t ks, int64_t vs, int64_t os, int64_t dks, int64_t dvs, float scale,
                    int causal) {
  KPO_PDL_ENTRY();
  using CF = BwdCfg<D>;
  constexpr int BN = CF::BN, BM = CF::BM, NT = CF::NT;
  extern __shared__ __align__(128) uint8_t smem[];
  const uint32_t sbase = s_u32(smem);
  const uint32_t sK = sbase + CF::OFF_K, sV = sbase + CF::OFF_V;
  const uint32_t sQ0 = sbase + CF::OFF_Q, sDO0 = sbase + CF::OFF_DO, sDS = sbase + CF::OFF_DS;
  float* sstat = reinterpret_cast<float*>(smem + CF::OFF_STAT);  // [2 buf][lse2 BM | dvec BM]

  const int nblk = gridDim.x - 1 - blockIdx.x;  // causal: early key blocks have the most work
  const int kvh = blockIdx.y;
  const int group = hq / hkv;
  const int n0 = nblk * BN;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const float scale_log2 = scale * kLog2e;

  load_tile<BN, D, NT>(sK, k + (int64_t)kvh * D, ks, n0, T);
  load_tile<BN, D, NT>(sV, v + (int64_t)kvh * D, vs, n0, T);

  const int mb_first = causal ? (n0 / BM) : 0;
  const int mb_count = (T + BM - 1) / BM - mb_first;
  const int steps = group * mb_count;

  auto issue = [&](int step, int buf) {
    const int h = kvh * group + step / mb_count;
    const int m0 = (mb_first + step % mb_count) * BM;
    load_tile<BM, D, NT>(sQ0 + buf * CF::QB, q + (int64_t)h * D, qs, m0, T);
    load_tile<BM, D, NT>(sDO0 + buf * CF::QB, dout + (int64_t)h * D, os, m0, T);
    float* st = sstat + buf * 2 * BM;
    for (int i = threadIdx.x; i < BM; i += NT) {
      const int t = m0 + i;
      st[i] = t < T ? lse[(int64_t)h * T + t] * kLog2e : INFINITY;
      st[BM + i] = t < T ? dvec[(int64_t)h * T + t] : 0.f;
    }
  };

  float dk_acc[D / 8][4], dv_acc[D / 8][4];
#pragma unroll
  for (int i = 0; i < D / 8; ++i)
#pragma unroll
    for (int e = 0; e < 4; ++e) dk_acc[i][e] = dv_acc[i][e] = 0.f;

  const int wk0 = warp * 16;  // warp's keys within the block
  const int key_of[2] = {n0 + wk0 + (lane >> 2), n0 + wk0 + (lane >> 2) + 8};

  if (steps > 0) issue(0, 0);
  cp_commit();
  for (int step = 0; step < steps; ++step) {
    const int buf = step & 1;
    if (step + 1 < steps) issue(step + 1, buf ^ 1);
    cp_commit();
    cp_wait<1>();
    __syncthreads();
    const int h = kvh * group + step / mb_count;
    const int m0 = (mb_first + step % mb_count) * BM;
    const uint32_t sQ = sQ0 + buf * CF::QB, sDO = sDO0 + buf * CF::QB;
    const float* st = sstat + buf * 2 * BM;

    // S^T = K Q^T (16 keys x 64 queries) and dP^T = V dO^T
    float s[BM / 8][4], dp[BM / 8][4];
#pragma unroll
    for (int i = 0; i < BM / 8; ++i)
#pragma unroll
      for (int e = 0; e < 4; ++e) s[i][e] = dp[i][e] = 0.f;
#pragma unroll
    for (int kk = 0; kk < D / 16; ++kk) {
      uint32_t ka[4], va[4];
      {
        const int r = wk0 + (lane & 7) + ((lane >> 3) & 1) * 8;
        const int c = kk * 16 + (lane >> 4) * 8;
        ldsm_x4(sK + swz<D>(r, c), ka[0], ka[1], ka[2], ka[3]);
        ldsm_x4(sV + swz<D>(r, c), va[0], va[1], va[2], va[3]);
      }
#pragma unroll
      for (int np = 0; np < BM / 16; ++np) {
        const int r = np * 16 + (lane & 7) + (lane >> 4) * 8;
        const int c = kk * 16 + ((lane >> 3) & 1) * 8;
        uint32_t b0, b1, b2, b3;
        ldsm_x4(sQ + swz<D>(r, c), b0, b1, b2, b3);
        mma16816(s[2 * np], ka, b0, b1);
        mma16816(s[2 * np + 1], ka, b2, b3);
        ldsm_x4(sDO + swz<D>(r, c), b0, b1, b2, b3);
        mma16816(dp[2 * np], va, b0, b1);
        mma16816(dp[2 * np + 1], va, b2, b3);
      }
    }
    // P^T and dS^T
#pragma unroll
    for (int i = 0; i < BM / 8; ++i) {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int qi = i * 8 + (lane & 3) * 2 + (e & 1);
        const int key = key_of[e >> 1];
        const int qtok = m0 + qi;
        float p = exp2f(s[i][e] * scale_log2 - st[qi]);
        if (key >= T || qtok >= T || (causal && qtok < key)) p = 0.f;
        s[i][e] = p;
        dp[i][e] = p * (dp[i][e] - st[BM + qi]);
      }
    }
    // dV += P^T dO ; dK += dS^T Q
#pragma unroll
    for (int kk = 0; kk < BM / 16; ++kk) {
      uint32_t pa[4], da[4];
      pa[0] = pack_bf16(s[2 * kk][0], s[2 * kk][1]);
      pa[1] = pack_bf16(s[2 * kk][2], s[2 * kk][3]);
      pa[2] = pack_bf16(s[2 * kk + 1][0], s[2 * kk + 1][1]);
      pa[3] = pack_bf16(s[2 * kk + 1][2], s[2 * kk + 1][3]);
      da[0] = pack_bf16(dp[2 * kk][0], dp[2 * kk][1]);
      da[1] = pack_bf16(dp[2 * kk][2], dp[2 * kk][3]);
      da[2] = pack_bf16(dp[2 * kk + 1][0], dp[2 * kk + 1][1]);
      da[3] = pack_bf16(dp[2 * kk + 1][2], dp[2 * kk + 1][3]);
#pragma unroll
      for (int np = 0; np < D / 16; ++np) {
        const int r = kk * 16 + (lane & 7) + ((lane >> 3) & 1) * 8;
        const int c = np * 16 + (lane >> 4) * 8;
        uint32_t b0, b1, b2, b3;
        ldsm_x4_t(sDO + swz<D>(r, c), b0, b1, b2, b3);
        mma16816(dv_acc[2 * np], pa, b0, b1);
        mma16816(dv_acc[2 * np + 1], pa, b2, b3);
        ldsm_x4_t(sQ + swz<D>(r, c), b0, b1, b2, b3);
        mma16816(dk_acc[2 * np], da, b0, b1);
        mma16816(dk_acc[2 * np + 1], da, b2, b3);
      }
    }
    // dS^T -> smem [key][query]
#pragma unroll
    for (int i = 0; i < BM / 8; ++i) {
      const int c = i * 8 + (lane & 3) * 2;
      const int r0 = wk0 + (lane >> 2);
      *reinterpret_cast<uint32_t*>(smem + CF::OFF_DS + swz<BM>(r0, c)) = pack_bf16(dp[i][0], dp[i][1]);
      *reinterpret_cast<uint32_t*>(smem + CF::OFF_DS + swz<BM>(r0 + 8, c)) = pack_bf16(dp[i][2], dp[i][3]);
    }
    __syncthreads();
    // dQ (16 queries per warp x D) += dS K, accumulated through fp32 atomics
    {
      const int wq0 = warp * 16;
      uint32_t dsa[BN / 16][4];
#pragma unroll
      for (int kk = 0; kk < BN / 16; ++kk) {
        const int j = lane >> 3;
        const int r = kk * 16 + (lane & 7) + (j >> 1) * 8;  // key (row of stored dS^T)
        const int c = wq0 + (j & 1) * 8;                      // query
        ldsm_x4_t(sDS + swz<BM>(r, c), dsa[kk][0], dsa[kk][1], dsa[kk][2], dsa[kk][3]);
      }
#pragma unroll
      for (int nc = 0; nc < D / 32; ++nc) {
        float acc[4][4];
#pragma unroll
        for (int i = 0; i < 4; ++i) acc[i][0] = acc[i][1] = acc[i][2] = acc[i][3] = 0.f;
#pragma unroll
        for (int kk = 0; kk < BN / 16; ++kk) {
#pragma unroll
          for (int np = 0; np < 2; ++np) {
            const int r = kk * 16 + (lane & 7) + ((lane >> 3) & 1) * 8;
            const int c = nc * 32 + np * 16 + (lane >> 4) * 8;
            uint32_t b0, b1, b2, b3;
            ldsm_x4_t(sK + swz<D>(r, c), b0, b1, b2, b3);
            mma16816(acc[2 * np], dsa[kk], b0, b1);
            mma16816(acc[2 * np + 1], dsa[kk], b2, b3);
          }
        }
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          const int qtok = m0 + wq0 + (lane >> 2) + hh * 8;
          if (qtok >= T) continue;
          float* dst = dq_acc + ((int64_t)qtok * hq + h) * D + nc * 32 + (lane & 3) * 2;
#pragma unroll
          for (int i = 0; i < 4; ++i)
            atomicAdd(reinterpret_cast<float2*>(dst + i * 8),
                      make_float2(acc[i][2 * hh] * scale, acc[i][2 * hh + 1] * scale));
        }
      }
    }
    __syncthreads();
  }
  // write dK (scaled), dV
#pragma unroll
  for (int hh = 0; hh < 2; ++hh) {
    const int key = key_of[hh];
    if (key >= T) continue;
    __nv_bfloat16* dkr = dk + (int64_t)key * dks + (int64_t)kvh * D;
    __nv_bfloat16* dvr = dv + (int64_t)key * dvs + (int64_t)kvh * D;
#pragma unroll
    for (int i = 0; i < D / 8; ++i) {
      const int c = i * 8 + (lane & 3) * 2;
      *reinterpret_cast<uint32_t*>(dkr + c) = pack_bf16(dk_acc[i][2 * hh] * scale, dk_acc[i][2 * hh + 1] * scale);
      *reinterpret_cast<uint32_t*>(dvr + c) = pack_bf16(dv_acc[i][2 * hh], dv_acc[i][2 * hh + 1]);
    }
  }
}

template <int D>
static int fwd_launch(const void* q, const void* k, const void* v, void* o, float* lse, int64_t T, int hq, int hkv,
                      int64_t qs, int64_t ks, int64_t vs, int64_t os, float scale, int causal, cudaStream_t s) {
  using CF = FwdCfg<D>;
  static bool set = false;
  if (!set) {
    KPO_CUDA(cudaFuncSetAttribute(attn_fwd_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, CF::SMEM));
    set = true;
  }
  dim3 grid((unsigned)((T + CF::BM - 1) / CF::BM), (unsigned)hq);
  KPO_CUDA(::kpo::pdl_launch(attn_fwd_kernel<D>, grid, CF::NT, CF::SMEM, s, (const __nv_bfloat16*)q, (const __nv_bfloat16*)k,
                                                    (const __nv_bfloat16*)v, (__nv_bfloat16*)o, lse, (int)T, hq, hkv,
                                                    qs, ks, vs, os, scale * kLog2e, causal));
  KPO_LAUNCH_CHECK();
  return KPO_OK;
}

template <int D>
static int bwd_launch(const void* q, const void* k, const void* v, const void* o, const void* dout, const float* lse,
                      void* dq, void* dk, void* dv, int64_t T, int hq, int hkv, int64_t qs, int64_t ks, int64_t vs,
                      int64_t os, int64_t dqs, int64_t dks, int64_t dvs, float scale, int causal, void* ws,
                      cudaStream_t s, bool use_tc, const float* rope_table = nullptr) {
  const float2* rope_cs = reinterpret_cast<const float2*>(rope_table);
  using CF = BwdCfg<D>;
  float* dq_acc = (float*)ws;
  float* dvec = dq_acc + T * hq * D;
  // KPO_ATTN_BWD: unset = the single-kernel tcgen05 backward (64-query steps for head_dim 128, 128-query
  // steps for 64); 2 / 3 force one of them; 4 = two kernels (dQ, then dK / dV: no cross-CTA dQ
  // reduction, so dQ is bitwise deterministic, and no pre / post kernels; measured 1.33x slower at
  // config 1); 1 = mma.sync (A/B baseline)
  static const int variant = getenv("KPO_ATTN_BWD") ? atoi(getenv("KPO_ATTN_BWD")) : 0;
  const bool two_kernels = use_tc && T % 8 == 0 && variant == 4;
  if (!two_kernels) {
    const int64_t threads = T * hq * (D / 8);
    KPO_CUDA(::kpo::pdl_launch(attn_bwd_pre_kernel<D>, (unsigned)((threads + 255) / 256), 256, 0, s, 
        (const __nv_bfloat16*)o, (const __nv_bfloat16*)dout, dvec, dq_acc, (int)T, hq, os));
    KPO_LAUNCH_CHECK();
  }
  if (use_tc && T % 8 == 0) {  // tcgen05 path (bulk-copied softmax stats need 16 B rows)
    // split-group mode when kv heads x key tiles cannot fill the GPU (e.g. TP8: one kv head per rank):
    // one CTA per (q head, key tile), dK/dV reduced in fp32 then converted
    const int64_t ntiles = (T + 127) / 128;
    static const int force_split = getenv("KPO_ATTN_BWD_SPLIT") ? atoi(getenv("KPO_ATTN_BWD_SPLIT")) : -1;
    const bool split = force_split >= 0 ? (force_split != 0 && hq > hkv) : (hq > hkv && hkv * ntiles < num_sms());
    // causal load balance: query chunks (grid z).  Split-group mode chunks every key tile (~2 CTAs per
    // SM).  Grouped mode can halve its first KPO_ATTN_BWD_QSPLIT key tiles (their dK / dV then go
    // through the fp32 accumulators); measured slower at config 1 for 6..12 tiles (0.298 -> 0.35-0.38
    // ms: the chunk-1 CTAs dispatch last, as a tail, and add 128 KB of fp32 reductions each), so off.
    int qchunks = 1, qsplit_tiles = 0;
    if (causal) {
      if (split) {
        const int sms = num_sms() > 0 ? num_sms() : 148;
        static const int env_q = getenv("KPO_ATTN_BWD_QCHUNKS") ? atoi(getenv("KPO_ATTN_BWD_QCHUNKS")) : 0;
        qchunks = env_q > 0 ? env_q : (int)((2 * sms) / (hq * ntiles));
        qchunks = qchunks < 1 ? 1 : (qchunks > 8 ? 8 : qchunks);
        qsplit_tiles = (int)ntiles;
      } else {
        static const int env_t = getenv("KPO_ATTN_BWD_QSPLIT") ? atoi(getenv("KPO_ATTN_BWD_QSPLIT")) : 0;
        qsplit_tiles = env_t < ntiles ? env_t : (int)ntiles;
        if (qsplit_tiles > 0) qchunks = 2;
      }
    }
    // key rows whose dK / dV are reduced through the fp32 accumulators (a prefix of the T rows)
    const int64_t acc_rows = split ? T : (qchunks > 1 ? std::min<int64_t>(T, (int64_t)qsplit_tiles * 128) : 0);
    float* dkv_acc = acc_rows > 0 ? dvec + (int64_t)hq * T : nullptr;
    if (dkv_acc) {
      KPO_CUDA(cudaMemsetAsync(dkv_acc, 0, sizeof(float) * acc_rows * hkv * D, s));
      KPO_CUDA(cudaMemsetAsync(dkv_acc + T * hkv * D, 0, sizeof(float) * acc_rows * hkv * D, s));
    }
    int st = two_kernels
                 ? attn_bwd_tcgen05_split(q, k, v, o, dout, lse, dvec, dq, dk, dv, T, hq, hkv, D, qs, ks, vs, os, dqs,
                                          dks, dvs, scale, causal, dkv_acc, split ? 1 : 0, qsplit_tiles, qchunks, s,
                                          rope_table)
                 : attn_bwd_tcgen05_main(q, k, v, dout, lse, dvec, dq_acc, dk, dv, T, hq, hkv, D, qs, ks, vs, os,
                                         dks, dvs, scale, causal, dkv_acc, split ? 1 : 0, qsplit_tiles, qchunks, s,
                                         rope_table);
    if (st) return st;
    if (dkv_acc) {
      // convert the accumulated rows; the accumulator layout [T][hkv][D] makes them a prefix, so the
      // conversion kernels run on acc_rows "tokens" with the full-T offset for the dV half
      const int64_t n = acc_rows * hkv * D / 8;
      if (rope_cs)
        KPO_CUDA(::kpo::pdl_launch(attn_bwd_post_rope_kernel<D>, (unsigned)((n / 2 + 255) / 256), 256, 0, s, dkv_acc,
                                   (__nv_bfloat16*)dk, (int)acc_rows, hkv, dks, rope_cs));
      else
        KPO_CUDA(::kpo::pdl_launch(attn_bwd_post_kernel<D>, (unsigned)((n + 255) / 256), 256, 0, s, dkv_acc,
                                   (__nv_bfloat16*)dk, (int)acc_rows, hkv, dks));
      KPO_LAUNCH_CHECK();
      KPO_CUDA(::kpo::pdl_launch(attn_bwd_post_kernel<D>, (unsigned)((n + 255) / 256), 256, 0, s,
                                 dkv_acc + T * hkv * D, (__nv_bfloat16*)dv, (int)acc_rows, hkv, dvs));
      KPO_LAUNCH_CHECK();
    }
  } else {
  static bool set = false;
  if (!set) {
    KPO_CUDA(cudaFuncSetAttribute(attn_bwd_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, CF::SMEM));
    set = true;
  }
  dim3 grid((unsigned)((T + CF::BN - 1) / CF::BN), (unsigned)hkv);
  KPO_CUDA(::kpo::pdl_launch(attn_bwd_kernel<D>, grid, CF::NT, CF::SMEM, s, 
      (const __nv_bfloat16*)q, (const __nv_bfloat16*)k, (const __nv_bfloat16*)v, (const __nv_bfloat16*)dout, lse, dvec,
      dq_acc, (__nv_bfloat16*)dk, (__nv_bfloat16*)dv, (int)T, hq, hkv, qs, ks, vs, os, dks, dvs, scale, causal));
  KPO_LAUNCH_CHECK();
  }
  if (!two_kernels) {  // dQ accumulator -> bf16 (the two-kernel path writes dQ directly)
    const int64_t n = T * hq * D / 8;
    if (rope_cs)
      KPO_CUDA(::kpo::pdl_launch(attn_bwd_post_rope_kernel<D>, (unsigned)((n / 2 + 255) / 256), 256, 0, s, dq_acc,
                                 (__nv_bfloat16*)dq, (int)T, hq, dqs, rope_cs));
    else
      KPO_CUDA(::kpo::pdl_launch(attn_bwd_post_kernel<D>, (unsigned)((n + 255) / 256), 256, 0, s, dq_acc, (__nv_bfloat16*)dq, (int)T, hq, dqs));
    KPO_LAUNCH_CHECK();
  }
  return KPO_OK;
}

}  // namespace attn
}  // namespace kpo

using namespace kpo;

static bool attn_args_ok(int64_t T, int hq, int hkv, int d) {
  return T > 0 && hq > 0 && hkv > 0 && hq % hkv == 0 && (d == 64 || d == 128);
}

extern "C" int kpo_attn_fwd(const void* q, const void* k, const void* v, void* o, float* lse, int64_t T, int hq,
                            int hkv, int d, int64_t q_stride, int64_t k_stride, int64_t v_stride, int64_t o_stride,
                            float scale, int causal, void* stream) {
  KPO_CHECK_ARG(q && k && v && o && lse, "attn_fwd: null pointer");
  KPO_CHECK_ARG(attn_args_ok(T, hq, hkv, d), "attn_fwd: need hq %% hkv == 0 and head_dim in {64, 128}");
  KPO_CHECK_ARG(q_stride % 8 == 0 && k_stride % 8 == 0 && v_stride % 8 == 0 && o_stride % 8 == 0,
                "attn_fwd: token strides must be multiples of 8");
  KPO_CHECK_ARG(((uintptr_t)q & 15) == 0 && ((uintptr_t)k & 15) == 0 && ((uintptr_t)v & 15) == 0,
                "attn_fwd: q/k/v must be 16B aligned (TMA)");
  return attn_fwd_tcgen05(q, k, v, o, lse, T, hq, hkv, d, q_stride, k_stride, v_stride, o_stride, scale, causal,
                          (cudaStream_t)stream);
}

extern "C" int kpo_attn_fwd_mma(const void* q, const void* k, const void* v, void* o, float* lse, int64_t T, int hq,
                                int hkv, int d, int64_t q_stride, int64_t k_stride, int64_t v_stride, int64_t o_stride,
                                float scale, int causal, void* stream) {
  KPO_CHECK_ARG(q && k && v && o && lse, "attn_fwd_mma: null pointer");
  KPO_CHECK_ARG(attn_args_ok(T, hq, hkv, d), "attn_fwd_mma: need hq %% hkv == 0 and head_dim in {64, 128}");
  cudaStream_t s = (cudaStream_t)stream;
  if (d == 128)
    return attn::fwd_launch<128>(q, k, v, o, lse, T, hq, hkv, q_stride, k_stride, v_stride, o_stride, scale, causal, s);
  return attn::fwd_launch<64>(q, k, v, o, lse, T, hq, hkv, q_stride, k_stride, v_stride, o_stride, scale, causal, s);
}

extern "C" int64_t kpo_attn_bwd_workspace_bytes(int64_t T, int hq, int hkv, int d) {
  // dq_acc [T][hq][d] + D-vector [hq][T] + (split-group mode) dK/dV accumulators 2 x [T][hkv][d], fp32
  return T * hq * d * 4 + (int64_t)hq * T * 4 + 2 * T * hkv * d * 4 + 256;
}

extern "C" int kpo_attn_bwd(const void* q, const void* k, const void* v, const void* o, const void* dout,
                            const float* lse, void* dq, void* dk, void* dv, int64_t T, int hq, int hkv, int d,
                            int64_t q_stride, int64_t k_stride, int64_t v_stride, int64_t o_stride, int64_t dq_stride,
                            int64_t dk_stride, int64_t dv_stride, float scale, int causal, void* workspace,
                            void* stream) {
  KPO_CHECK_ARG(q && k && v && o && dout && lse && dq && dk && dv && workspace, "attn_bwd: null pointer");
  KPO_CHECK_ARG(attn_args_ok(T, hq, hkv, d), "attn_bwd: need hq %% hkv == 0 and head_dim in {64, 128}");
  KPO_CHECK_ARG(((uintptr_t)workspace & 15) == 0, "attn_bwd: workspace must be 16B aligned");
  cudaStream_t s = (cudaStream_t)stream;
  if (d == 128)
    return attn::bwd_launch<128>(q, k, v, o, dout, lse, dq, dk, dv, T, hq, hkv, q_stride, k_stride, v_stride,
                                 o_stride, dq_stride, dk_stride, dv_stride, scale, causal, workspace, s, true);
  // head_dim 64 (config 0): the 128-query tcgen05 kernel; KPO_ATTN_BWD=1 keeps the mma.sync kernel (A/B only)
  static const bool legacy64 = getenv("KPO_ATTN_BWD") && atoi(getenv("KPO_ATTN_BWD")) == 1;
  return attn::bwd_launch<64>(q, k, v, o, dout, lse, dq, dk, dv, T, hq, hkv, q_stride, k_stride, v_stride, o_stride,
                              dq_stride, dk_stride, dv_stride, scale, causal, workspace, s, !legacy64);
}

extern "C" int kpo_attn_bwd_rope(const void* q, const void* k, const void* v, const void* o, const void* dout,
                                 const float* lse, void* dq, void* dk, void* dv, int64_t T, int hq, int hkv, int d,
                                 int64_t q_stride, int64_t k_stride, int64_t v_stride, int64_t o_stride,
                                 int64_t dq_stride, int64_t dk_stride, int64_t dv_stride, float scale, int causal,
                                 void* workspace, const float* rope_table, void* stream) {
  KPO_CHECK_ARG(q && k && v && o && dout && lse && dq && dk && dv && workspace && rope_table,
                "attn_bwd_rope: null pointer");
  KPO_CHECK_ARG(attn_args_ok(T, hq, hkv, d) && d == 128 && T % 8 == 0,
                "attn_bwd_rope: the fused inverse rotary path needs head_dim 128 and T %% 8 == 0");
  KPO_CHECK_ARG(((uintptr_t)workspace & 15) == 0, "attn_bwd_rope: workspace must be 16B aligned");
  return attn::bwd_launch<128>(q, k, v, o, dout, lse, dq, dk, dv, T, hq, hkv, q_stride, k_stride, v_stride, o_stride,
                               dq_stride, dk_stride, dv_stride, scale, causal, workspace, (cudaStream_t)stream, true,
                               rope_table);
}
