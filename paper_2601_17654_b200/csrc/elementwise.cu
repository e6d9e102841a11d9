// elementwise.cu — HBM-bound launch units of a partition: RMSNorm fwd/bwd, RoPE fwd/bwd,
// SwiGLU fwd/bwd, fp32 column sums.
//
// These stand in for the reference's memory-bound KernelSpecs ("norm", "rope", "fused_norm";
// reference pkg/src/schedfront/workloads.py:44-46,60,87), which compose.py:48-76
// (`group_memory_bound`) treats as single logical launch units.  Roofline: HBM bytes
// (read + write) / measured copy bandwidth; all loads/stores are 16-byte vectors and every row is
// read from HBM once (held in registers across its reduction: a 128-thread CTA per row for the
// RMSNorm forward, a row block per CTA with next-row prefetch for the fused backward, one warp per
// row for the generic widths).  The SwiGLU kernels also serve the blocked gate|up layout of the fused
// GEMM epilogues (gemm_sm100.cu) and share their sigmoid (kpo_sigmoid).
#include "common.cuh"

namespace kpo {

// ===================================================================== RMSNorm forward
// One warp per row.  Rows of up to 32*8*NV elements are cached in registers (NV uint4 per lane).
// Register cap: 3 CTAs (24 row-warps) per SM for rows up to 3072 columns — unbounded, ptxas hoists the
// gamma loads and reaches 150 registers, i.e. 8 warps per SM and 3.5 waves of latency-bound rows.
template <int NV>
__global__ void __launch_bounds__(256, NV <= 12 ? 3 : 1) rmsnorm_fwd_cached(const __nv_bfloat16* __restrict__ x,
                                                          const __nv_bfloat16* __restrict__ w,
                                                          __nv_bfloat16* __restrict__ y,
                                                          float* __restrict__ rstd, int64_t rows,
                                                          int cols, float eps) {
  KPO_PDL_ENTRY();
  const int lane = threadIdx.x & 31;
  const int64_t row = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (row >= rows) return;
  const uint4* xr = reinterpret_cast<const uint4*>(x + row * cols);
  uint4 v[NV];
  float ss = 0.f;
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    v[i] = ld_nc_v4(xr + lane + 32 * i);
    float f[8];
    unpack8(v[i], f);
#pragma unroll
    for (int j = 0; j < 8; ++j) ss += f[j] * f[j];
  }
  ss = warp_sum(ss);
  const float r = rsqrtf(ss / (float)cols + eps);
  if (lane == 0 && rstd) rstd[row] = r;
  const uint4* wr = reinterpret_cast<const uint4*>(w);
  uint4* yr = reinterpret_cast<uint4*>(y + row * cols);
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    float f[8], g[8];
    unpack8(v[i], f);
    unpack8(wr[lane + 32 * i], g);
#pragma unroll
    for (int j = 0; j < 8; ++j) f[j] = f[j] * r * g[j];
    yr[lane + 32 * i] = pack8(f);
  }
}

// One 128-thread CTA per row for rows of 1024*NV columns (NV uint4 per thread): ~30 registers, 16
// rows resident per SM, and a finished row's SM slot is refilled at CTA granularity.
template <int NV>
__global__ void __launch_bounds__(128) rmsnorm_fwd_row(const __nv_bfloat16* __restrict__ x,
                                                       const __nv_bfloat16* __restrict__ w,
                                                       __nv_bfloat16* __restrict__ y, float* __restrict__ rstd,
                                                       int64_t rows, int cols, float eps) {
  KPO_PDL_ENTRY();
  __shared__ float red[4];
  const int64_t row = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const uint4* xr = reinterpret_cast<const uint4*>(x + row * cols);
  uint4 v[NV];
  float ss = 0.f;
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    v[i] = ld_nc_v4(xr + tid + 128 * i);
    float f[8];
    unpack8(v[i], f);
#pragma unroll
    for (int j = 0; j < 8; ++j) ss += f[j] * f[j];
  }
  ss = warp_sum(ss);
  if (lane == 0) red[wid] = ss;
  __syncthreads();
  ss = (red[0] + red[1]) + (red[2] + red[3]);
  const float r = rsqrtf(ss / (float)cols + eps);
  if (tid == 0 && rstd) rstd[row] = r;
  const uint4* wr = reinterpret_cast<const uint4*>(w);
  uint4* yr = reinterpret_cast<uint4*>(y + row * cols);
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    float f[8], g[8];
    unpack8(v[i], f);
    unpack8(wr[tid + 128 * i], g);
#pragma unroll
    for (int j = 0; j < 8; ++j) f[j] = f[j] * r * g[j];
    yr[tid + 128 * i] = pack8(f);
  }
  (void)rows;
}

// Generic fallback: two passes over the row (second pass served by L1/L2).
__global__ void __launch_bounds__(256) rmsnorm_fwd_generic(const __nv_bfloat16* __restrict__ x,
                                                           const __nv_bfloat16* __restrict__ w,
                                                           __nv_bfloat16* __restrict__ y,
                                                           float* __restrict__ rstd, int64_t rows,
                                                           int cols, float eps) {
  KPO_PDL_ENTRY();
  const int lane = threadIdx.x & 31;
  const int64_t row = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (row >= rows) return;
  const uint4* xr = reinterpret_cast<const uint4*>(x + row * cols);
  const int nv = cols / 8;
  float ss = 0.f;
#pragma unroll 4
  for (int i = lane; i < nv; i += 32) {
    float f[8];
    unpack8(ld_nc_v4(xr + i), f);
#pragma unroll
    for (int j = 0; j < 8; ++j) ss += f[j] * f[j];
  }
  ss = warp_sum(ss);
  const float r = rsqrtf(ss / (float)cols + eps);
  if (lane == 0 && rstd) rstd[row] = r;
  const uint4* wr = reinterpret_cast<const uint4*>(w);
  uint4* yr = reinterpret_cast<uint4*>(y + row * cols);
#pragma unroll 4
  for (int i = lane; i < nv; i += 32) {
    float f[8], g[8];
    unpack8(xr[i], f);
    unpack8(wr[i], g);
#pragma unroll
    for (int j = 0; j < 8; ++j) f[j] = f[j] * r * g[j];
    yr[i] = pack8(f);
  }
}

// ===================================================================== RMSNorm backward
// dx_i = r*w_i*dy_i - x_i * r^3/n * sum_j(w_j*dy_j*x_j)  (+ dres_i)     [rmsnorm_bwd_dx: one warp per row]
// dw_j = sum_rows dy_j*x_j*r, as fp32 partial sums over 16-row slabs   [rmsnorm_bwd_dw: column-parallel,
//        re-reads x / dy right after the dx kernel, while they are still resident in the 126 MB L2]
constexpr int kNormBwdSlab = 16;

template <int NV>
__global__ void __launch_bounds__(256)
    rmsnorm_bwd_dx_cached(const __nv_bfloat16* __restrict__ dy, const __nv_bfloat16* __restrict__ x,
                          const __nv_bfloat16* __restrict__ w, const float* __restrict__ rstd,
                          const __nv_bfloat16* __restrict__ dres, __nv_bfloat16* __restrict__ dx, int64_t rows,
                          int cols) {
  KPO_PDL_ENTRY();
  const int lane = threadIdx.x & 31;
  const int64_t row = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (row >= rows) return;
  const uint4* xr = reinterpret_cast<const uint4*>(x + row * cols);
  const uint4* dyr = reinterpret_cast<const uint4*>(dy + row * cols);
  const uint4* wr = reinterpret_cast<const uint4*>(w);
  const float r = rstd[row];
  uint4 xv[NV], dv[NV];
  float dot = 0.f;
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    xv[i] = ld_nc_v4(xr + lane + 32 * i);
    dv[i] = ld_nc_v4(dyr + lane + 32 * i);
  }
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    float a[8], b[8], g[8];
    unpack8(xv[i], a);
    unpack8(dv[i], b);
    unpack8(wr[lane + 32 * i], g);
#pragma unroll
    for (int j = 0; j < 8; ++j) dot += g[j] * b[j] * a[j];
  }
  dot = warp_sum(dot);
  const float c = dot * r * r * r / (float)cols;
  uint4* dxr = reinterpret_cast<uint4*>(dx + row * cols);
  const uint4* dresr = dres ? reinterpret_cast<const uint4*>(dres + row * cols) : nullptr;
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    float a[8], b[8], g[8], o[8];
    unpack8(xv[i], a);
    unpack8(dv[i], b);
    unpack8(wr[lane + 32 * i], g);
    float res[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    if (dresr) unpack8(ld_nc_v4(dresr + lane + 32 * i), res);
#pragma unroll
    for (int j = 0; j < 8; ++j) o[j] = r * g[j] * b[j] - a[j] * c + res[j];
    dxr[lane + 32 * i] = pack8(o);
  }
}

__global__ void __launch_bounds__(256)
    rmsnorm_bwd_dx_generic(const __nv_bfloat16* __restrict__ dy, const __nv_bfloat16* __restrict__ x,
                           const __nv_bfloat16* __restrict__ w, const float* __restrict__ rstd,
                           const __nv_bfloat16* __restrict__ dres, __nv_bfloat16* __restrict__ dx, int64_t rows,
                           int cols) {
  KPO_PDL_ENTRY();
  const int lane = threadIdx.x & 31;
  const int64_t row = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (row >= rows) return;
  const int nv = cols / 8;
  const uint4* xr = reinterpret_cast<const uint4*>(x + row * cols);
  const uint4* dyr = reinterpret_cast<const uint4*>(dy + row * cols);
  const uint4* wr = reinterpret_cast<const uint4*>(w);
  const float r = rstd[row];
  float dot = 0.f;
#pragma unroll 4
  for (int i = lane; i < nv; i += 32) {
    float a[8], b[8], g[8];
    unpack8(ld_nc_v4(xr + i), a);
    unpack8(ld_nc_v4(dyr + i), b);
    unpack8(wr[i], g);
#pragma unroll
    for (int j = 0; j < 8; ++j) dot += g[j] * b[j] * a[j];
  }
  dot = warp_sum(dot);
  const float c = dot * r * r * r / (float)cols;
  uint4* dxr = reinterpret_cast<uint4*>(dx + row * cols);
  const uint4* dresr = dres ? reinterpret_cast<const uint4*>(dres + row * cols) : nullptr;
#pragma unroll 4
  for (int i = lane; i < nv; i += 32) {
    float a[8], b[8], g[8], o[8];
    unpack8(xr[i], a);
    unpack8(dyr[i], b);
    unpack8(wr[i], g);
    float res[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    if (dresr) unpack8(dresr[i], res);
#pragma unroll
    for (int j = 0; j < 8; ++j) o[j] = r * g[j] * b[j] - a[j] * c + res[j];
    dxr[i] = pack8(o);
  }
}

// Fused single-pass backward for rows of 1024*NV columns (hidden 1024..4096).  A 256-thread CTA owns
// a contiguous block of rows; its two 128-thread groups take alternate rows, one row per group at a
// time, with the next row's x / dy / dres loads issued before the current row is reduced (two rows
// per group in flight).  Each thread owns the same 8*NV columns of every row, so its share of dgamma
// accumulates in registers; the groups combine through shared memory into ONE fp32 partial row per
// CTA.  x, dy and dres are read from HBM once.
template <int NV>
__global__ void __launch_bounds__(256)
    rmsnorm_bwd_rows(const __nv_bfloat16* __restrict__ dy, const __nv_bfloat16* __restrict__ x,
                     const __nv_bfloat16* __restrict__ w, const float* __restrict__ rstd,
                     const __nv_bfloat16* __restrict__ dres, __nv_bfloat16* __restrict__ dx,
                     float* __restrict__ dw_partial, int64_t rows, int rows_per_cta) {
  KPO_PDL_ENTRY();
  constexpr int cols = NV * 1024;
  __shared__ float red[2][2][4];            // [group][row parity][warp] partial dot products
  __shared__ __align__(16) float comb[cols];  // group 1's dgamma share, added by group 0
  const int tid = threadIdx.x & 127, grp = threadIdx.x >> 7, lane = threadIdx.x & 31, wid = tid >> 5;
  const int64_t r_begin = (int64_t)blockIdx.x * rows_per_cta;
  const int64_t r_end = min(rows, r_begin + rows_per_cta);
  float acc[NV][8];
  float g[NV][8];
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    unpack8(reinterpret_cast<const uint4*>(w)[tid + 128 * i], g[i]);
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;
  }
  uint4 cx[NV], cd[NV], cr[NV], nx[NV], nd[NV], nr[NV];
  auto load = [&](int64_t row, uint4* ox, uint4* od, uint4* orr) {
    const uint4* xr = reinterpret_cast<const uint4*>(x + row * cols);
    const uint4* dyr = reinterpret_cast<const uint4*>(dy + row * cols);
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      ox[i] = ld_nc_v4(xr + tid + 128 * i);
      od[i] = ld_nc_v4(dyr + tid + 128 * i);
    }
    if (dres) {
      const uint4* rr = reinterpret_cast<const uint4*>(dres + row * cols);
#pragma unroll
      for (int i = 0; i < NV; ++i) orr[i] = ld_nc_v4(rr + tid + 128 * i);
    }
  };
  int64_t row = r_begin + grp;
  if (row < r_end) load(row, cx, cd, cr);
  for (int k = 0; row < r_end; ++k, row += 2) {
    const bool more = row + 2 < r_end;
    if (more) load(row + 2, nx, nd, nr);
    const float r = rstd[row];
    float dot = 0.f;
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      float a[8], b[8];
      unpack8(cx[i], a);
      unpack8(cd[i], b);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        acc[i][j] += b[j] * a[j] * r;
        dot += g[i][j] * b[j] * a[j];
      }
    }
    dot = warp_sum(dot);
    if (lane == 0) red[grp][k & 1][wid] = dot;
    asm volatile("bar.sync %0, 128;" ::"r"(1 + grp) : "memory");
    dot = (red[grp][k & 1][0] + red[grp][k & 1][1]) + (red[grp][k & 1][2] + red[grp][k & 1][3]);
    const float c = dot * r * r * r / (float)cols;
    uint4* dxr = reinterpret_cast<uint4*>(dx + row * cols);
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      float a[8], b[8], o[8], res[8];
      unpack8(cx[i], a);
      unpack8(cd[i], b);
      if (dres) unpack8(cr[i], res);
#pragma unroll
      for (int j = 0; j < 8; ++j) o[j] = r * g[i][j] * b[j] - a[j] * c + (dres ? res[j] : 0.f);
      dxr[tid + 128 * i] = pack8(o);
    }
    if (more) {
#pragma unroll
      for (int i = 0; i < NV; ++i) {
        cx[i] = nx[i];
        cd[i] = nd[i];
        cr[i] = nr[i];
      }
    }
  }
  if (grp == 1) {
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      float4* c4 = reinterpret_cast<float4*>(comb + (tid + 128 * i) * 8);
      c4[0] = make_float4(acc[i][0], acc[i][1], acc[i][2], acc[i][3]);
      c4[1] = make_float4(acc[i][4], acc[i][5], acc[i][6], acc[i][7]);
    }
  }
  __syncthreads();
  if (grp == 0) {
    float4* out = reinterpret_cast<float4*>(dw_partial + (int64_t)blockIdx.x * cols);
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const int c8 = tid + 128 * i;
      const float4* c4 = reinterpret_cast<const float4*>(comb + c8 * 8);
      const float4 p = c4[0], q = c4[1];
      out[c8 * 2] = make_float4(acc[i][0] + p.x, acc[i][1] + p.y, acc[i][2] + p.z, acc[i][3] + p.w);
      out[c8 * 2 + 1] = make_float4(acc[i][4] + q.x, acc[i][5] + q.y, acc[i][6] + q.z, acc[i][7] + q.w);
    }
  }
}

// rows per CTA (even: the two row groups stay in step) and CTA count of the fused backward
static inline void fused_norm_bwd_grid(int64_t rows, int& rows_per_cta, int& grid) {
  int sms = num_sms();
  if (sms <= 0) sms = 148;  // no device visible (host-only queries): B200's SM count
  // two CTAs per SM's worth of row blocks (run as two waves): when an SM-budgeted collective holds
  // some SMs, the blocks it displaces are half as long (in-step 42.5 -> 36.4 us with the comm
  // overlapped, unchanged alone; four waves cost 8 us alone)
  static const int per_sm = getenv("KPO_NORM_BWD_WAVES") ? atoi(getenv("KPO_NORM_BWD_WAVES")) : 2;
  const int64_t ctas = (int64_t)sms * (per_sm > 0 ? per_sm : 1);
  int64_t rpc = (rows + ctas - 1) / ctas;
  rpc += rpc & 1;
  if (rpc < 2) rpc = 2;
  rows_per_cta = (int)rpc;
  grid = (int)((rows + rpc - 1) / rpc);
}
static inline bool fused_norm_bwd_ok(int64_t cols) { return cols % 1024 == 0 && cols / 1024 <= 4; }

// one thread per 8-column chunk, a 64-row slab per blockIdx.y; coalesced 16-byte loads along rows
__global__ void __launch_bounds__(128)
    rmsnorm_bwd_dw(const __nv_bfloat16* __restrict__ dy, const __nv_bfloat16* __restrict__ x,
                   const float* __restrict__ rstd, float* __restrict__ dw_partial, int64_t rows, int cols) {
  KPO_PDL_ENTRY();
  const int chunk = blockIdx.x * blockDim.x + threadIdx.x;
  if (chunk * 8 >= cols) return;
  const int64_t r0 = (int64_t)blockIdx.y * kNormBwdSlab;
  const int64_t r1 = r0 + kNormBwdSlab < rows ? r0 + kNormBwdSlab : rows;
  float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll 4
  for (int64_t row = r0; row < r1; ++row) {
    float a[8], b[8];
    unpack8(*reinterpret_cast<const uint4*>(x + row * cols + chunk * 8), a);
    unpack8(*reinterpret_cast<const uint4*>(dy + row * cols + chunk * 8), b);
    const float rr = rstd[row];
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[j] += b[j] * a[j] * rr;
  }
  float4* out = reinterpret_cast<float4*>(dw_partial + (int64_t)blockIdx.y * cols + chunk * 8);
  out[0] = make_float4(acc[0], acc[1], acc[2], acc[3]);
  out[1] = make_float4(acc[4], acc[5], acc[6], acc[7]);
}

// out[c] = sum_r in[r, c] (fp32 partial rows -> bf16), e.g. the per-CTA dγ partials of both nanobatches.
// One launch, two levels: CTA (x, y) reduces rows [y*kColsumRows, +kColsumRows) of the 128-column block
// x (8 warps x 4 rows, lane = 4 consecutive columns, coalesced float4 loads) into one fp32 partial row of
// a library workspace; the last CTA of column block x (arrival counter, self-resetting, so a captured
// graph replays) adds the gridDim.y partial rows in a fixed order and writes bf16.  The first version
// (one thread per column looping over all rows) took 55 us for 592 x 3072; this is bandwidth-bound.
constexpr int kColsumRows = 32;
constexpr int kColsumMaxSplits = 64;
constexpr int kColsumMaxCols = 16384;
__device__ float g_colsum_ws[kColsumMaxSplits * kColsumMaxCols];
__device__ unsigned int g_colsum_cnt[kColsumMaxCols / 128];

__global__ void __launch_bounds__(256) colsum_kernel(const float* __restrict__ in, __nv_bfloat16* __restrict__ out,
                                                     int64_t rows, int64_t cols, int rows_per_split) {
  KPO_PDL_ENTRY();
  __shared__ float4 red[8][32];
  __shared__ bool last;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t c = (int64_t)blockIdx.x * 128 + lane * 4;
  const int64_t r0 = (int64_t)blockIdx.y * rows_per_split;
  const int64_t r1 = min(rows, r0 + rows_per_split);
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  if (c < cols) {
#pragma unroll 4
    for (int64_t r = r0 + warp; r < r1; r += 8) {
      const float4 v = *reinterpret_cast<const float4*>(in + r * cols + c);
      acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    }
  }
  red[warp][lane] = acc;
  __syncthreads();
  if (warp == 0) {
    float4 t = red[0][lane];
#pragma unroll
    for (int w = 1; w < 8; ++w) {
      const float4 v = red[w][lane];
      t.x += v.x; t.y += v.y; t.z += v.z; t.w += v.w;
    }
    if (c < cols) *reinterpret_cast<float4*>(g_colsum_ws + (int64_t)blockIdx.y * cols + c) = t;
    __threadfence();
  }
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(&g_colsum_cnt[blockIdx.x], 1u) == gridDim.y - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  if (warp == 0 && c < cols) {
    float4 t = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int y = 0; y < (int)gridDim.y; ++y) {
      const float4 v = __ldcg(reinterpret_cast<const float4*>(g_colsum_ws + (int64_t)y * cols + c));
      t.x += v.x; t.y += v.y; t.z += v.z; t.w += v.w;
    }
    uint2 o;
    o.x = pack_bf16x2(t.x, t.y);
    o.y = pack_bf16x2(t.z, t.w);
    *reinterpret_cast<uint2*>(out + c) = o;
  }
  if (threadIdx.x == 0) g_colsum_cnt[blockIdx.x] = 0;
}

// fallback for very wide rows: one thread per column, coalesced across the warp
__global__ void colsum_wide_kernel(const float* __restrict__ in, __nv_bfloat16* __restrict__ out, int64_t rows,
                                   int64_t cols) {
  KPO_PDL_ENTRY();
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= cols) return;
  float s = 0.f;
  for (int64_t r = 0; r < rows; ++r) s += in[r * cols + c];
  out[c] = f2bf(s);
}

// ===================================================================== RoPE
// One CTA per token; the token's cos/sin table (head_dim/2 entries) is built once in smem and
// reused by every head.  Each thread rotates 8 consecutive pairs of one head.
__global__ void rope_kernel(const __nv_bfloat16* __restrict__ in, int64_t in_stride,
                            __nv_bfloat16* __restrict__ out, int64_t out_stride, int heads,
                            int head_dim, float log2_theta, int64_t pos0, int inverse) {
  KPO_PDL_ENTRY();
  extern __shared__ float cs[];  // [half] cos, [half] sin
  const int half = head_dim / 2;
  const int64_t t = blockIdx.x;
  const float pos = (float)(pos0 + t);
  for (int i = threadIdx.x; i < half; i += blockDim.x) {
    const float inv_freq = exp2f(-(2.0f * (float)i / (float)head_dim) * log2_theta);
    float s, c;
    sincosf(pos * inv_freq, &s, &c);
    cs[i] = c;
    cs[half + i] = inverse ? -s : s;
  }
  __syncthreads();
  const int chunks = half / 8;  // 8-pair chunks per head
  const __nv_bfloat16* src = in + t * in_stride;
  __nv_bfloat16* dst = out + t * out_stride;
  for (int job = threadIdx.x; job < heads * chunks; job += blockDim.x) {
    const int h = job / chunks, ch = job % chunks;
    const int i0 = ch * 8;
    const __nv_bfloat16* hp = src + (int64_t)h * head_dim;
    float a[8], b[8], oa[8], ob[8];
    unpack8(*reinterpret_cast<const uint4*>(hp + i0), a);
    unpack8(*reinterpret_cast<const uint4*>(hp + half + i0), b);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const float c = cs[i0 + j], s = cs[half + i0 + j];
      oa[j] = a[j] * c - b[j] * s;
      ob[j] = b[j] * c + a[j] * s;
    }
    __nv_bfloat16* op = dst + (int64_t)h * head_dim;
    *reinterpret_cast<uint4*>(op + i0) = pack8(oa);
    *reinterpret_cast<uint4*>(op + half + i0) = pack8(ob);
  }
}

// ===================================================================== SwiGLU
__device__ __forceinline__ float sigmoidf_(float x) { return kpo_sigmoid(x); }

// gate / up column of act column j: halves layout (blk == 0): g at j, u at ffn + j; blocked layout
// (blk > 0, the fused gate|up GEMM's weight order): blocks of blk gate columns followed by the
// matching blk up columns.
__device__ __forceinline__ int64_t gate_col(int64_t j, int64_t ffn, int blk) {
  return blk ? (j / blk) * 2 * blk + j % blk : j;
}

__global__ void swiglu_fwd_kernel(const __nv_bfloat16* __restrict__ gu, __nv_bfloat16* __restrict__ act,
                                  int64_t rows, int64_t ffn, int blk) {
  KPO_PDL_ENTRY();
  const int64_t nvr = ffn / 8;
  const int64_t total = rows * nvr;
  const int64_t uoff = blk ? blk : ffn;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = idx / nvr, c = idx % nvr;
    const __nv_bfloat16* gp = gu + r * 2 * ffn + gate_col(c * 8, ffn, blk);
    float g[8], u[8], o[8];
    unpack8(ld_nc_v4(gp), g);
    unpack8(ld_nc_v4(gp + uoff), u);
#pragma unroll
    for (int j = 0; j < 8; ++j) o[j] = g[j] * sigmoidf_(g[j]) * u[j];
    *reinterpret_cast<uint4*>(act + r * ffn + c * 8) = pack8(o);
  }
}

__global__ void swiglu_bwd_kernel(const __nv_bfloat16* __restrict__ dact, const __nv_bfloat16* __restrict__ gu,
                                  __nv_bfloat16* __restrict__ dgu, int64_t rows, int64_t ffn, int blk) {
  KPO_PDL_ENTRY();
  const int64_t nvr = ffn / 8;
  const int64_t total = rows * nvr;
  const int64_t uoff = blk ? blk : ffn;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = idx / nvr, c = idx % nvr;
    const int64_t gc = r * 2 * ffn + gate_col(c * 8, ffn, blk);
    float g[8], u[8], d[8], dg[8], du[8];
    unpack8(ld_nc_v4(gu + gc), g);
    unpack8(ld_nc_v4(gu + gc + uoff), u);
    unpack8(ld_nc_v4(dact + r * ffn + c * 8), d);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const float s = sigmoidf_(g[j]);
      const float silu = g[j] * s;
      du[j] = d[j] * silu;
      dg[j] = d[j] * u[j] * s * (1.f + g[j] * (1.f - s));
    }
    *reinterpret_cast<uint4*>(dgu + gc) = pack8(dg);
    *reinterpret_cast<uint4*>(dgu + gc + uoff) = pack8(du);
  }
}

static int elem_grid(int64_t work, int threads) {
  const int64_t want = (work + threads - 1) / threads;
  const int64_t cap = (int64_t)num_sms() * 16;
  return (int)(want < cap ? (want > 0 ? want : 1) : cap);
}

}  // namespace kpo

using namespace kpo;

static inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

extern "C" int kpo_rmsnorm_fwd(const void* x, const void* w, void* y, float* rstd, int64_t rows,
                               int64_t cols, float eps, void* stream) {
  KPO_CHECK_ARG(x && w && y, "rmsnorm_fwd: null pointer");
  KPO_CHECK_ARG(rows >= 0 && cols > 0 && cols % 8 == 0, "rmsnorm_fwd: cols must be a positive multiple of 8");
  KPO_CHECK_ARG(aligned16(x) && aligned16(w) && aligned16(y), "rmsnorm_fwd: pointers must be 16B aligned");
  if (rows == 0) return KPO_OK;
  cudaStream_t s = (cudaStream_t)stream;
  const int warps = 8;
  const dim3 grid((unsigned)((rows + warps - 1) / warps)), block(warps * 32);
  auto X = (const __nv_bfloat16*)x;
  auto W = (const __nv_bfloat16*)w;
  auto Y = (__nv_bfloat16*)y;
  if (cols % 1024 == 0 && cols / 1024 <= 8 && cols / 1024 != 7) {
    switch (cols / 1024) {
#define KPO_NORM_ROW_CASE(n) \
  case n: KPO_CUDA(::kpo::pdl_launch(rmsnorm_fwd_row<n>, dim3((unsigned)rows), dim3(128), 0, s, X, W, Y, rstd, rows, (int)cols, eps)); break;
      KPO_NORM_ROW_CASE(1) KPO_NORM_ROW_CASE(2) KPO_NORM_ROW_CASE(3) KPO_NORM_ROW_CASE(4) KPO_NORM_ROW_CASE(5)
      KPO_NORM_ROW_CASE(6) KPO_NORM_ROW_CASE(8)
#undef KPO_NORM_ROW_CASE
    }
  } else if (cols % 256 == 0 && cols / 256 <= 16) {
    switch (cols / 256) {
#define KPO_NORM_CASE(n) \
  case n: KPO_CUDA(::kpo::pdl_launch(rmsnorm_fwd_cached<n>, grid, block, 0, s, X, W, Y, rstd, rows, (int)cols, eps)); break;
      KPO_NORM_CASE(1) KPO_NORM_CASE(2) KPO_NORM_CASE(3) KPO_NORM_CASE(4) KPO_NORM_CASE(5)
      KPO_NORM_CASE(6) KPO_NORM_CASE(8) KPO_NORM_CASE(10) KPO_NORM_CASE(12) KPO_NORM_CASE(16)
#undef KPO_NORM_CASE
      default: KPO_CUDA(::kpo::pdl_launch(rmsnorm_fwd_generic, grid, block, 0, s, X, W, Y, rstd, rows, (int)cols, eps));
    }
  } else {
    KPO_CUDA(::kpo::pdl_launch(rmsnorm_fwd_generic, grid, block, 0, s, X, W, Y, rstd, rows, (int)cols, eps));
  }
  KPO_LAUNCH_CHECK();
  return KPO_OK;
}

extern "C" int kpo_rmsnorm_bwd_partial_rows(int64_t rows, int64_t cols, int64_t* n_partials) {
  KPO_CHECK_ARG(n_partials, "null n_partials");
  if (fused_norm_bwd_ok(cols) && rows > 0) {
    int rpw, grid;
    fused_norm_bwd_grid(rows, rpw, grid);
    *n_partials = grid;
    return KPO_OK;
  }
  *n_partials = (rows + kNormBwdSlab - 1) / kNormBwdSlab;
  return KPO_OK;
}

extern "C" int kpo_rmsnorm_bwd(const void* dy, const void* x, const void* w, const float* rstd,
                               const void* dres, void* dx, float* dw_partial, int64_t rows, int64_t cols,
                               void* stream) {
  KPO_CHECK_ARG(dy && x && w && rstd && dx && dw_partial, "rmsnorm_bwd: null pointer");
  KPO_CHECK_ARG(cols > 0 && cols % 8 == 0, "rmsnorm_bwd: cols must be a positive multiple of 8");
  KPO_CHECK_ARG(aligned16(dy) && aligned16(x) && aligned16(w) && aligned16(dx) && (!dres || aligned16(dres)),
                "rmsnorm_bwd: pointers must be 16B aligned");
  if (rows == 0) return KPO_OK;
  cudaStream_t st = (cudaStream_t)stream;
  auto Dy = (const __nv_bfloat16*)dy;
  auto X = (const __nv_bfloat16*)x;
  auto W = (const __nv_bfloat16*)w;
  auto Dr = (const __nv_bfloat16*)dres;
  auto Dx = (__nv_bfloat16*)dx;
  if (fused_norm_bwd_ok(cols)) {
    int rpc, g;
    fused_norm_bwd_grid(rows, rpc, g);
    switch (cols / 1024) {
#define KPO_NBF_CASE(n) \
  case n: KPO_CUDA(::kpo::pdl_launch(rmsnorm_bwd_rows<n>, g, 256, 0, st, Dy, X, W, rstd, Dr, Dx, dw_partial, rows, rpc)); break;
      KPO_NBF_CASE(1) KPO_NBF_CASE(2) KPO_NBF_CASE(3) KPO_NBF_CASE(4)
#undef KPO_NBF_CASE
    }
    KPO_LAUNCH_CHECK();
    return KPO_OK;
  }
  const dim3 grid((unsigned)((rows + 7) / 8)), block(256);
  if (cols % 256 == 0 && cols / 256 <= 4) {  // small rows: cache in registers; large rows: two-pass re-read
    switch (cols / 256) {
#define KPO_NB_CASE(n) \
  case n: KPO_CUDA(::kpo::pdl_launch(rmsnorm_bwd_dx_cached<n>, grid, block, 0, st, Dy, X, W, rstd, Dr, Dx, rows, (int)cols)); break;
      KPO_NB_CASE(1) KPO_NB_CASE(2) KPO_NB_CASE(3) KPO_NB_CASE(4)
#undef KPO_NB_CASE
      default: KPO_CUDA(::kpo::pdl_launch(rmsnorm_bwd_dx_generic, grid, block, 0, st, Dy, X, W, rstd, Dr, Dx, rows, (int)cols));
    }
  } else {
    KPO_CUDA(::kpo::pdl_launch(rmsnorm_bwd_dx_generic, grid, block, 0, st, Dy, X, W, rstd, Dr, Dx, rows, (int)cols));
  }
  KPO_LAUNCH_CHECK();
  const dim3 g2((unsigned)((cols / 8 + 127) / 128), (unsigned)((rows + kNormBwdSlab - 1) / kNormBwdSlab));
  KPO_CUDA(::kpo::pdl_launch(rmsnorm_bwd_dw, g2, 128, 0, st, Dy, X, rstd, dw_partial, rows, (int)cols));
  KPO_LAUNCH_CHECK();
  return KPO_OK;
}

extern "C" int kpo_colsum_f32_to_bf16(const float* in, void* out, int64_t rows, int64_t cols, void* stream) {
  KPO_CHECK_ARG(in && out && rows >= 0 && cols > 0, "colsum: bad args");
  if (cols % 4 == 0 && cols <= kColsumMaxCols && aligned16(in) && ((uintptr_t)out % 8) == 0 && rows > 0) {
    int per = kColsumRows;
    int64_t splits = (rows + per - 1) / per;
    if (splits > kColsumMaxSplits) {
      per = (int)((rows + kColsumMaxSplits - 1) / kColsumMaxSplits);
      splits = (rows + per - 1) / per;
    }
    dim3 grid((unsigned)((cols + 127) / 128), (unsigned)splits);
    KPO_CUDA(::kpo::pdl_launch(colsum_kernel, grid, 256, 0, (cudaStream_t)stream, in, (__nv_bfloat16*)out, rows,
                               cols, per));
  } else {
    KPO_CUDA(::kpo::pdl_launch(colsum_wide_kernel, (unsigned)((cols + 255) / 256), 256, 0, (cudaStream_t)stream, in,
                               (__nv_bfloat16*)out, rows, cols));
  }
  KPO_LAUNCH_CHECK();
  return KPO_OK;
}

extern "C" int kpo_rope(const void* in, int64_t in_row_stride, void* out, int64_t out_row_stride,
                        int64_t tokens, int heads, int head_dim, float theta, int64_t pos0, int inverse,
                        void* stream) {
  KPO_CHECK_ARG(in && out, "rope: null pointer");
  KPO_CHECK_ARG(head_dim % 16 == 0 && head_dim <= 512, "rope: head_dim must be a multiple of 16");
  KPO_CHECK_ARG(in_row_stride % 8 == 0 && out_row_stride % 8 == 0 && aligned16(in) && aligned16(out),
                "rope: strides/pointers must be 16B aligned");
  KPO_CHECK_ARG(theta > 1.f, "rope: theta must be > 1");
  if (tokens == 0) return KPO_OK;
  const int threads = 256;
  KPO_CUDA(::kpo::pdl_launch(rope_kernel, (unsigned)tokens, threads, head_dim * sizeof(float), (cudaStream_t)stream, 
      (const __nv_bfloat16*)in, in_row_stride, (__nv_bfloat16*)out, out_row_stride, heads, head_dim,
      log2f(theta), pos0, inverse));
  KPO_LAUNCH_CHECK();
  return KPO_OK;
}

// (cos, sin) of position pos0 + t and frequency i, for t < tokens and i < head_dim / 2: the same
// arithmetic as rope_kernel, tabulated once for the fused rotary epilogue of the QKV GEMM.
__global__ void rope_table_kernel(float2* __restrict__ table, int64_t tokens, int half, float log2_theta,
                                  int64_t pos0) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= tokens * half) return;
  const int64_t t = e / half;
  const int i = (int)(e % half);
  const float inv_freq = exp2f(-(2.0f * (float)i / (float)(2 * half)) * log2_theta);
  float sn, cn;
  sincosf((float)(pos0 + t) * inv_freq, &sn, &cn);
  table[e] = make_float2(cn, sn);
}

extern "C" int kpo_rope_table(int64_t tokens, int head_dim, float theta, int64_t pos0, float* table, void* stream) {
  KPO_CHECK_ARG(table && tokens >= 0 && head_dim % 2 == 0 && head_dim > 0 && theta > 1.f, "rope_table: bad args");
  if (tokens == 0) return KPO_OK;
  const int64_t n = tokens * (head_dim / 2);
  rope_table_kernel<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
      reinterpret_cast<float2*>(table), tokens, head_dim / 2, log2f(theta), pos0);
  KPO_LAUNCH_CHECK();
  return KPO_OK;
}

extern "C" int kpo_swiglu_fwd_blocked(const void* gu, void* act, int64_t rows, int64_t ffn, int block,
                                      void* stream) {
  KPO_CHECK_ARG(gu && act && ffn % 8 == 0 && aligned16(gu) && aligned16(act), "swiglu_fwd: bad args");
  KPO_CHECK_ARG(block >= 0 && block % 8 == 0 && (block == 0 || ffn % block == 0),
                "swiglu_fwd: block must be 0 (gate | up halves) or a multiple of 8 dividing ffn");
  if (rows == 0) return KPO_OK;
  KPO_CUDA(::kpo::pdl_launch(swiglu_fwd_kernel, elem_grid(rows * ffn / 8, 256), 256, 0, (cudaStream_t)stream,
                             (const __nv_bfloat16*)gu, (__nv_bfloat16*)act, rows, ffn, block));
  KPO_LAUNCH_CHECK();
  return KPO_OK;
}

extern "C" int kpo_swiglu_fwd(const void* gu, void* act, int64_t rows, int64_t ffn, void* stream) {
  return kpo_swiglu_fwd_blocked(gu, act, rows, ffn, 0, stream);
}

extern "C" int kpo_swiglu_bwd_blocked(const void* dact, const void* gu, void* dgu, int64_t rows, int64_t ffn,
                                      int block, void* stream) {
  KPO_CHECK_ARG(dact && gu && dgu && ffn % 8 == 0 && aligned16(dact) && aligned16(gu) && aligned16(dgu),
                "swiglu_bwd: bad args");
  KPO_CHECK_ARG(block >= 0 && block % 8 == 0 && (block == 0 || ffn % block == 0),
                "swiglu_bwd: block must be 0 (gate | up halves) or a multiple of 8 dividing ffn");
  if (rows == 0) return KPO_OK;
  KPO_CUDA(::kpo::pdl_launch(swiglu_bwd_kernel, elem_grid(rows * ffn / 8, 256), 256, 0, (cudaStream_t)stream,
                             (const __nv_bfloat16*)dact, (const __nv_bfloat16*)gu, (__nv_bfloat16*)dgu, rows, ffn,
                             block));
  KPO_LAUNCH_CHECK();
  return KPO_OK;
}

extern "C" int kpo_swiglu_bwd(const void* dact, const void* gu, void* dgu, int64_t rows, int64_t ffn,
                              void* stream) {
  return kpo_swiglu_bwd_blocked(dact, gu, dgu, rows, ffn, 0, stream);
}
