// gemm_sm100.cu — warp-specialized tcgen05 GEMM for sm_100a (bf16 in, fp32 accumulate in TMEM).
//
// Replaces the reference's abstract compute-bound kernels ("linear_qkv", "linear_proj",
// "linear_up", "linear_down", "linear"; reference workloads.py:45,48,61-62,73) whose cost the
// simulator models as flops / (SMs * peak_flops_per_sm_mhz * f)  (simgpu.py:77-79,166).
//
// Design (B200-first):
//   * one CTA per SM (smem > half the SM), 6 warps: warp0 = tile scheduler + TMA producer,
//     warp1 = TMEM allocator + single-thread tcgen05.mma issuer, warps 2-5 = epilogue
//     (tcgen05.ld TMEM -> registers -> bf16 -> TMA stores; optional fused residual add, RoPE for
//     the QKV projection, SwiGLU for the gate|up projection, SwiGLU backward for the down dgrad);
//   * operands staged by TMA (cp.async.bulk.tensor, 128B swizzle) into a STAGES-deep
//     smem ring guarded by mbarriers; accumulators double-buffered in TMEM so the epilogue of
//     tile i overlaps the main loop of tile i+1;
//   * K-major or MN-major A/B (forward = TN, dgrad = NN, wgrad = TT) selected by template,
//     expressed only in the TMA boxes and the UMMA smem/instruction descriptors;
//   * dynamic persistent tile scheduler: grid = min(tiles, max_ctas) CTAs fetch tiles from a
//     global atomic counter.  CTAs that cannot become resident while the SM-budgeted collective
//     owns its SMs launch when those SMs free up and steal the remaining tiles — this is the
//     hardware analogue of the simulator handing all SMs back once communication ends
//     (simgpu.py:221).  The last CTA to finish resets the counter (graph-replay safe).
#include "sm100.cuh"
#include <stdlib.h>

namespace kpo {
namespace gemm {
using namespace kpo::sm100;

constexpr int BM = 128;
constexpr int BK = 64;
constexpr int kThreads = 192;
constexpr int GROUP_M = 16;

template <int BN>
struct Cfg {
  static constexpr int A_BYTES = BM * BK * 2;
  static constexpr int B_BYTES = BN * BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int STAGES = (BN == 256) ? 4 : (BN == 192 ? 5 : 6);
  static constexpr int TMEM_COLS = (2 * BN <= 256) ? 256 : 512;  // double-buffered accumulator (power of two)
  static constexpr int BAR_OFF = STAGES * STAGE_BYTES;
  // epilogue staging for the TMA stores: per epilogue warp EPI_BUFS x [32 rows x 64 cols] bf16 (SW128)
  static constexpr int EPI_OFF = BAR_OFF + 1024;
  static constexpr int EPI_BUFS = (EPI_OFF + 4 * 2 * 4096 + 1024 <= 232448) ? 2 : 1;
  static constexpr int SMEM = EPI_OFF + 4 * EPI_BUFS * 4096 + 1024;  // + alignment slack
};

__device__ __forceinline__ void tile_coords(int t, int num_m, int num_n, int& mb, int& nb) {
  const int per_group = GROUP_M * num_n;
  const int g = t / per_group;
  const int first_m = g * GROUP_M;
  const int gsize = min(num_m - first_m, GROUP_M);
  const int r = t % per_group;
  mb = first_m + r % gsize;
  nb = r / gsize;
}

// Epilogue of one accumulator tile for one thread's output row (TMEM lane == row): 32-column chunks
// tcgen05.ld -> fp32 (+ C) -> bf16 stores.  The optional C input (fused residual / gradient
// accumulation, which may alias D: every element is read before the same thread overwrites it) is
// row-strided per thread, so its loads are issued kCPre chunks ahead — the first ones before the
// accumulator is even ready — instead of serialising a full memory latency into every chunk
// (measured: +45% on a K=3072 residual GEMM without the prefetch, tools/gemm_epilogue_bench.py).
constexpr int kCPre = 4;
// D leaves through TMA: each epilogue warp converts 64 columns of its 32 rows to bf16, writes them
// to its shared-memory staging box (128 B rows, SWIZZLE_128B, conflict-free) and one lane issues a
// bulk tensor store [64 cols x 32 rows].  Full-line writes instead of 16-byte row-strided stores
// (measured: the row-strided stores cost ~1.5x the L2 throughput of cuBLAS's TMA-store epilogue for
// the same tile); rows / columns beyond M / N are clipped by the tensor map.
// Fused rotary embedding for the QKV projection: output columns [0, cols) are q / k heads of 128;
// each pair (i, i + 64) of a head is rotated by the row's angle table entry i (cos, sin), exactly the
// rotation of rope_kernel (elementwise.cu), but on the fp32 accumulator before the single bf16
// rounding.  cs = [rows][64] float2 (kpo_rope_table).
struct RopeArgs {
  const float2* cs;
  int cols;
};

template <int BUFS>
__device__ __forceinline__ void store_box(uint32_t stage, int lane, int& store_cnt, const uint4* packed,
                                          const CUtensorMap* tmD, int col0, int warp_row0) {
  const int b = store_cnt % BUFS;
  if (lane == 0) {
    if (BUFS == 2) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
    else asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
  }
  __syncwarp();
  const uint32_t box = stage + b * 4096;
#pragma unroll
  for (int k = 0; k < 8; ++k)
    asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(box + lane * 128 + ((k ^ (lane & 7)) << 4)),
                 "r"(packed[k].x), "r"(packed[k].y), "r"(packed[k].z), "r"(packed[k].w)
                 : "memory");
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncwarp();
  if (lane == 0) {
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                     reinterpret_cast<uint64_t>(tmD)),
                 "r"(box), "r"(col0), "r"(warp_row0)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
  }
  ++store_cnt;
}

// one 128-column head of a rope tile: chunks (0, 2) then (1, 3) are the rotation pairs
template <int BUFS>
__device__ __forceinline__ void epilogue_rope_head(uint32_t tmem_head, const float2* cs_row, bool row_ok, int col0,
                                                   int warp_row0, uint32_t stage, int lane, int& store_cnt,
                                                   const CUtensorMap* tmD) {
  uint4 lo[8], hi[8];  // output columns [0, 64) and [64, 128) of the head, packed bf16
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    uint32_t a[32], b[32];
    tmem_ld32(tmem_head + h * 32, a);
    tmem_ld32(tmem_head + 64 + h * 32, b);
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      float oa[8], ob[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int i = h * 32 + v * 8 + j;  // frequency index
        const float2 t = row_ok ? cs_row[i] : make_float2(1.f, 0.f);
        const float x = __uint_as_float(a[v * 8 + j]), y = __uint_as_float(b[v * 8 + j]);
        oa[j] = x * t.x - y * t.y;
        ob[j] = y * t.x + x * t.y;
      }
      lo[h * 4 + v] = pack8(oa);
      hi[h * 4 + v] = pack8(ob);
    }
  }
  store_box<BUFS>(stage, lane, store_cnt, lo, tmD, col0, warp_row0);
  store_box<BUFS>(stage, lane, store_cnt, hi, tmD, col0 + 64, warp_row0);
}

template <int BN, int BUFS, bool ROPE, typename WaitAcc>
__device__ __forceinline__ void epilogue_row(uint32_t tmem_row, const CUtensorMap* tmD, const __nv_bfloat16* C,
                                             int row, bool row_ok, int col_base, int N, int64_t ldd, int warp_row0,
                                             uint32_t stage, int lane, int& store_cnt, RopeArgs rope,
                                             WaitAcc wait_acc) {
  constexpr int NC = BN / 32;
  static_assert(NC % 2 == 0, "64-column store boxes");
  if (ROPE && BN % 128 == 0 && rope.cs != nullptr && col_base < rope.cols) {  // tile-uniform: q / k heads
    wait_acc();
    const float2* cs_row = rope.cs + (int64_t)(row_ok ? row : 0) * 64;
#pragma unroll 1
    for (int hh = 0; hh < BN / 128; ++hh) {
      const int col0 = col_base + hh * 128;
      if (col0 >= N) break;
      if (col0 < rope.cols)
        epilogue_rope_head<BUFS>(tmem_row + hh * 128, cs_row, row_ok, col0, warp_row0, stage, lane, store_cnt, tmD);
      else {  // a v head in the same tile: plain conversion
        uint4 lo[8], hi[8];
#pragma unroll
        for (int h = 0; h < 4; ++h) {
          uint32_t r[32];
          tmem_ld32(tmem_row + hh * 128 + h * 32, r);
#pragma unroll
          for (int v = 0; v < 4; ++v) {
            float f[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) f[j] = __uint_as_float(r[v * 8 + j]);
            (h < 2 ? lo : hi)[(h & 1) * 4 + v] = pack8(f);
          }
        }
        store_box<BUFS>(stage, lane, store_cnt, lo, tmD, col0, warp_row0);
        store_box<BUFS>(stage, lane, store_cnt, hi, tmD, col0 + 64, warp_row0);
      }
    }
    return;
  }
  const __nv_bfloat16* crow = (C != nullptr && row_ok) ? C + (int64_t)row * ldd : nullptr;
  uint4 cpf[kCPre][4];
  auto cload = [&](int c, uint4* dst) {
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      const int col = col_base + c * 32 + v * 8;
      dst[v] = col < N ? *reinterpret_cast<const uint4*>(crow + col) : make_uint4(0, 0, 0, 0);
    }
  };
  if (crow) {
#pragma unroll
    for (int p = 0; p < kCPre && p < NC; ++p) cload(p, cpf[p]);
  }
  wait_acc();
#pragma unroll
  for (int pc = 0; pc < NC / 2; ++pc) {
    const int col0 = col_base + pc * 64;
    uint4 packed[8];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int c = pc * 2 + h;
      uint32_t r[32];
      tmem_ld32(tmem_row + c * 32, r);
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        float f[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) f[j] = __uint_as_float(r[v * 8 + j]);
        if (crow) {
          float cf[8];
          unpack8(cpf[c % kCPre][v], cf);
#pragma unroll
          for (int j = 0; j < 8; ++j) f[j] += cf[j];
        }
        packed[h * 4 + v] = pack8(f);
      }
      if (crow && c + kCPre < NC) cload(c + kCPre, cpf[c % kCPre]);
    }
    if (col0 >= N) continue;  // warp-uniform: the whole box is past the last column
    store_box<BUFS>(stage, lane, store_cnt, packed, tmD, col0, warp_row0);
  }
  (void)row_ok;
}

// Fused SwiGLU for the gate|up projection (CTA-pair 256x256 tiles over weights stored in 128-row
// gate / up blocks, layer.py `interleave_gate_up`): accumulator columns [0, 128) of a tile are gate
// block nb and [128, 256) the matching up block, so act[:, nb*128 + i] = silu(g_i) * u_i is complete
// inside one tile.  g / u are rounded to bf16 first, exactly the values the separate swiglu kernel
// (elementwise.cu) would read back from gu, which is still written for the backward.
template <int BUFS>
__device__ __forceinline__ void epilogue_swiglu(uint32_t tmem_row, const CUtensorMap* tmGU, const CUtensorMap* tmAct,
                                                int gu_col0, int act_col0, int warp_row0, uint32_t stage, int lane,
                                                int& store_cnt) {
#pragma unroll 1
  for (int h2 = 0; h2 < 2; ++h2) {  // 64-column halves of the 128 act columns
    uint4 pa[8], pg[8], pu[8];
#pragma unroll
    for (int hh = 0; hh < 2; ++hh) {
      const int c = h2 * 2 + hh;
      uint32_t g[32], u[32];
      tmem_ld32(tmem_row + c * 32, g);
      tmem_ld32(tmem_row + 128 + c * 32, u);
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        float fg[8], fu[8], fa[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          fg[j] = __bfloat162float(__float2bfloat16_rn(__uint_as_float(g[v * 8 + j])));
          fu[j] = __bfloat162float(__float2bfloat16_rn(__uint_as_float(u[v * 8 + j])));
          fa[j] = fg[j] * kpo_sigmoid(fg[j]) * fu[j];  // = swiglu_fwd_kernel's expression
        }
        pg[hh * 4 + v] = pack8(fg);
        pu[hh * 4 + v] = pack8(fu);
        pa[hh * 4 + v] = pack8(fa);
      }
    }
    store_box<BUFS>(stage, lane, store_cnt, pg, tmGU, gu_col0 + h2 * 64, warp_row0);
    store_box<BUFS>(stage, lane, store_cnt, pu, tmGU, gu_col0 + 128 + h2 * 64, warp_row0);
    store_box<BUFS>(stage, lane, store_cnt, pa, tmAct, act_col0 + h2 * 64, warp_row0);
  }
}

// Fused SwiGLU backward for the down-projection dgrad (CTA-pair 256x256 tiles; gu / dgu in the 128-
// blocked gate|up order): the tile's accumulator is dact[:, nb*256 .. +256), i.e. gate/up blocks
// 2nb and 2nb+1, whose gate and up columns are the contiguous gu columns [512 nb, 512 nb + 512).
// Per 64 dact columns a warp TMA-loads its 32 rows of the matching gate box and up box into its
// staging buffers (the load for the first chunk is issued before the accumulator is ready), rounds
// dact to bf16 (the value the separate kernel would read), computes dgate / dup with
// swiglu_bwd_kernel's expressions in place, and TMA-stores both boxes to dgu.  dact itself is never
// written.
template <typename WaitAcc, typename Release>
__device__ __forceinline__ void epilogue_swiglu_bwd(uint32_t tmem_row, const CUtensorMap* tmDGU,
                                                    const CUtensorMap* tmGU, int act_col0, int warp_row0,
                                                    uint32_t stage, uint32_t bar, uint32_t& nchunk, int lane,
                                                    WaitAcc wait_acc, Release release_acc) {
  // two box-pair slots of 8 KB: chunk c+1's loads are issued before chunk c is computed
  auto gcol_of = [&](int c) { return (act_col0 / 128 + (c >> 1)) * 256 + (c & 1) * 64; };
  auto issue = [&](int c, uint32_t n) {
    const uint32_t buf = stage + (n & 1) * 8192;
    if (lane == 0) {
      // the slot's previous stores (chunk n-2) are the only bulk group still outstanding: once they have
      // read the buffers, the loads may overwrite them
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      const uint32_t b = bar + (n & 1) * 8;
      mbar_arrive_expect_tx(b, 8192);
      tma_load_2d(buf, tmGU, b, gcol_of(c), warp_row0);
      tma_load_2d(buf + 4096, tmGU, b, gcol_of(c) + 128, warp_row0);
    }
  };
  issue(0, nchunk);
  wait_acc();
#pragma unroll 1
  for (int c = 0; c < 4; ++c) {
    const uint32_t n = nchunk + c;
    uint32_t dv[64];
    tmem_ld32_nowait(tmem_row + c * 64, dv);
    tmem_ld32_nowait(tmem_row + c * 64 + 32, dv + 32);
    tmem_wait_ld();
    if (c == 3) release_acc();
    if (c < 3) issue(c + 1, n + 1);
    const uint32_t buf = stage + (n & 1) * 8192;
    mbar_wait(bar + (n & 1) * 8, (n >> 1) & 1);
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const uint32_t off = lane * 128 + ((k ^ (lane & 7)) << 4);
      uint4 gv, uv;
      asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
                   : "=r"(gv.x), "=r"(gv.y), "=r"(gv.z), "=r"(gv.w)
                   : "r"(buf + off));
      asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
                   : "=r"(uv.x), "=r"(uv.y), "=r"(uv.z), "=r"(uv.w)
                   : "r"(buf + 4096 + off));
      float g[8], u[8], dg[8], du[8];
      unpack8(gv, g);
      unpack8(uv, u);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const float dd = __bfloat162float(__float2bfloat16_rn(__uint_as_float(dv[k * 8 + j])));
        const float sg = kpo_sigmoid(g[j]);
        const float silu = g[j] * sg;
        du[j] = dd * silu;
        dg[j] = dd * u[j] * sg * (1.f + g[j] * (1.f - sg));
      }
      const uint4 pg = pack8(dg), pu = pack8(du);
      asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(buf + off), "r"(pg.x), "r"(pg.y), "r"(pg.z),
                   "r"(pg.w)
                   : "memory");
      asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(buf + 4096 + off), "r"(pu.x), "r"(pu.y),
                   "r"(pu.z), "r"(pu.w)
                   : "memory");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    if (lane == 0) {
      const int gcol = gcol_of(c);
      asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                       reinterpret_cast<uint64_t>(tmDGU)),
                   "r"(buf), "r"(gcol), "r"(warp_row0)
                   : "memory");
      asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                       reinterpret_cast<uint64_t>(tmDGU)),
                   "r"(buf + 4096), "r"(gcol + 128), "r"(warp_row0)
                   : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
  }
  nchunk += 4;
}

template <int BN, bool A_MN, bool B_MN>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                const __grid_constant__ CUtensorMap tmD,
                __nv_bfloat16* __restrict__ D, const __nv_bfloat16* C /* may alias D */, int M, int N, int K,
                int64_t ldd, int* __restrict__ sched, RopeArgs rope) {
  ::kpo::pdl_launch_dependents();  // the next kernel may start its prologue; it waits for us
  using CF = Cfg<BN>;
  constexpr int STAGES = CF::STAGES;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + CF::BAR_OFF);
  // barrier layout
  uint64_t* full = bars;                  // [STAGES]
  uint64_t* empty = bars + STAGES;        // [STAGES]
  uint64_t* tfull = bars + 2 * STAGES;    // [2]
  uint64_t* tempty = tfull + 2;           // [2]
  uint64_t* sfull = tempty + 2;           // [2]
  uint64_t* sempty = sfull + 2;           // [2]
  int* stile = reinterpret_cast<int*>(sempty + 2);        // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(stile + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int num_m = (M + BM - 1) / BM, num_n = (N + BN - 1) / BN;
  const int num_tiles = num_m * num_n;
  const int num_kb = (K + BK - 1) / BK;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(smem_u32(&full[s]), 1);
      mbar_init(smem_u32(&empty[s]), 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(smem_u32(&tfull[i]), 1);
      mbar_init(smem_u32(&tempty[i]), 4);
      mbar_init(smem_u32(&sfull[i]), 1);
      mbar_init(smem_u32(&sempty[i]), 5);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(CF::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  ::kpo::pdl_wait();  // inputs, scheduler words and outputs of the previous kernel are settled

  if (warp == 0) {
    if (lane == 0) {
      // ===================== tile scheduler + TMA producer
      int it = 0, stage = 0;
      uint32_t phase = 0;
      while (true) {
        const int tile = atomicAdd(&sched[0], 1);
        const int slot = it & 1;
        mbar_wait(smem_u32(&sempty[slot]), ((it >> 1) & 1) ^ 1);
        stile[slot] = tile;
        mbar_arrive(smem_u32(&sfull[slot]));
        ++it;
        if (tile >= num_tiles) break;
        int mb, nb;
        tile_coords(tile, num_m, num_n, mb, nb);
        const int m0 = mb * BM, n0 = nb * BN;
        for (int kb = 0; kb < num_kb; ++kb) {
          mbar_wait(smem_u32(&empty[stage]), phase ^ 1);
          const uint32_t fb = smem_u32(&full[stage]);
          mbar_arrive_expect_tx(fb, CF::STAGE_BYTES);
          const uint32_t sa = smem_u32(smem + stage * CF::STAGE_BYTES);
          const uint32_t sb = sa + CF::A_BYTES;
          const int k0 = kb * BK;
          if (!A_MN) {
            tma_load_2d(sa, &tmA, fb, k0, m0);
          } else {
#pragma unroll
            for (int c = 0; c < BM / 64; ++c) tma_load_2d(sa + c * (BK * 128), &tmA, fb, m0 + c * 64, k0);
          }
          if (!B_MN) {
            tma_load_2d(sb, &tmB, fb, k0, n0);
          } else {
#pragma unroll
            for (int c = 0; c < BN / 64; ++c) tma_load_2d(sb + c * (BK * 128), &tmB, fb, n0 + c * 64, k0);
          }
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
      // the last CTA out resets the scheduler word for the next launch (graph-replay safe)
      __threadfence();
      const int done = atomicAdd(&sched[1], 1);
      if (done == (int)gridDim.x - 1) {
        sched[0] = 0;
        sched[1] = 0;
        __threadfence();
      }
    }
  } else if (warp == 1) {
    {
      // ===================== MMA issuer: the whole warp runs the loop (warp-uniform operands in
      // uniform registers), elect.sync issues each tcgen05.mma / commit
      constexpr uint32_t IDESC = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)A_MN << 15) |
                                 ((uint32_t)B_MN << 16) | ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
      // K-major SW128: SBO = 8 rows * 128B; MN-major SW128: LBO = MN-chunk stride, SBO = 8 K-rows.
      constexpr uint32_t A_LBO = A_MN ? BK * 128 : 16, A_SBO = 1024;
      constexpr uint32_t B_LBO = B_MN ? BK * 128 : 16, B_SBO = 1024;
      constexpr uint32_t A_KSTEP = A_MN ? 16 * 128 : 32;  // bytes per UMMA_K=16 step
      constexpr uint32_t B_KSTEP = B_MN ? 16 * 128 : 32;
      int it = 0, stage = 0, acc_it = 0;
      uint32_t phase = 0;
      while (true) {
        const int slot = it & 1;
        mbar_wait(smem_u32(&sfull[slot]), (it >> 1) & 1);
        const int tile = stile[slot];
        __syncwarp();
        if (lane == 0) mbar_arrive(smem_u32(&sempty[slot]));
        ++it;
        if (tile >= num_tiles) break;
        const int acc = acc_it & 1;
        mbar_wait(smem_u32(&tempty[acc]), ((acc_it >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = 0; kb < num_kb; ++kb) {
          mbar_wait(smem_u32(&full[stage]), phase);
          tc_fence_after();
          const uint32_t sa = smem_u32(smem + stage * CF::STAGE_BYTES);
          const uint32_t sb = sa + CF::A_BYTES;
          static_assert(A_SBO == 1024 && B_SBO == 1024, "split descriptors assume SBO 1024 / SWIZZLE_128B");
          const uint32_t a_lo = desc_lo(sa, A_LBO), b_lo = desc_lo(sb, B_LBO);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k)
            tc_mma_lo_w(d_tmem, a_lo + k * (A_KSTEP >> 4), b_lo + k * (B_KSTEP >> 4), IDESC, (kb | k) != 0);
          tc_commit_w(smem_u32(&empty[stage]));
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        tc_commit_w(smem_u32(&tfull[acc]));
        ++acc_it;
      }
    }
  } else {
    // ===================== epilogue warps 2..5: TMEM lanes 32*(warp%4) .. +31
    const int q = warp & 3;
    int it = 0, acc_it = 0, store_cnt = 0;
    while (true) {
      const int slot = it & 1;
      mbar_wait(smem_u32(&sfull[slot]), (it >> 1) & 1);
      const int tile = stile[slot];
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_u32(&sempty[slot]));
      ++it;
      if (tile >= num_tiles) break;
      int mb, nb;
      tile_coords(tile, num_m, num_n, mb, nb);
      const int acc = acc_it & 1;
      const int row = mb * BM + q * 32 + lane;
      epilogue_row<BN, CF::EPI_BUFS, !A_MN && !B_MN>(tmem_base + ((uint32_t)(q * 32) << 16) + acc * BN, &tmD, C, row, row < M,
                                     nb * BN, N, ldd, mb * BM + q * 32,
                                     smem_u32(smem + CF::EPI_OFF) + q * CF::EPI_BUFS * 4096, lane, store_cnt, rope,
                       [&] {
                         mbar_wait(smem_u32(&tfull[acc]), (acc_it >> 1) & 1);
                         tc_fence_after();
                       });
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_u32(&tempty[acc]));
      ++acc_it;
    }
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");  // D stores complete
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(CF::TMEM_COLS));
  }
}

// ------------------------------------------------------------------ host side
template <int BN, bool A_MN, bool B_MN>
static int launch(const CUtensorMap& ta, const CUtensorMap& tb, void* D, const void* C, int64_t M, int64_t N,
                  int64_t K, int64_t ldd, int grid, int* sched, cudaStream_t s, RopeArgs rope) {
  auto kern = gemm_kernel<BN, A_MN, B_MN>;
  CUtensorMap td;
  if (int e = make_map_2d(&td, D, N, M, ldd, 64, 32)) return e;
  static bool attr_set = false;
  if (!attr_set) {
    KPO_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg<BN>::SMEM));
    attr_set = true;
  }
  KPO_CUDA(::kpo::pdl_launch(kern, grid, kThreads, Cfg<BN>::SMEM, s, ta, tb, td, (__nv_bfloat16*)D, (const __nv_bfloat16*)C, (int)M, (int)N,
                                              (int)K, ldd, sched, rope));
  KPO_LAUNCH_CHECK();
  return KPO_OK;
}


// =====================================================================================
// CTA-pair variant (tcgen05.mma.cta_group::2): one 256 x BN tile per cluster of 2 CTAs on the
// same TPC.  A is split by M (each CTA stages its 128 rows), B is split by N (each CTA stages BN/2
// columns); the leader (rank 0) issues the M=256 MMAs, which read both CTAs' shared memory, and
// each CTA's TMEM receives its 128 accumulator rows.  Per CTA this halves B's shared-memory traffic
// per FLOP versus the 1-CTA kernel (64 B/clk instead of 96 B/clk at BN=256).
//   * both CTAs' TMA loads complete on the leader's full[] barrier (peer bit cleared);
//   * MMA completion is multicast (tcgen05.commit ... multicast::cluster, mask 0b11) to the
//     empty[] / tfull[] barriers of both CTAs;
//   * the leader fetches tile ids from the global scheduler word and broadcasts them to the peer
//     through distributed shared memory; consumers in the peer arrive remotely on the leader's
//     sempty[] / tempty[] barriers.
template <int BN, int EPI = 0>
struct Cfg2 {
  static constexpr int A_BYTES = 128 * BK * 2;
  static constexpr int B_BYTES = (BN / 2) * BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  // the fused SwiGLU backward's epilogue double-buffers its gate / up boxes: 4 buffers per warp, one
  // operand stage fewer
  static constexpr int STAGES = (BN == 256) ? (EPI == 2 ? 5 : 6) : 7;
  static constexpr int TMEM_COLS = (2 * BN <= 256) ? 256 : 512;
  static constexpr int BAR_OFF = STAGES * STAGE_BYTES;
  static constexpr int EPI_OFF = BAR_OFF + 1024;
  static constexpr int EPI_BUFS = EPI == 2 ? 4 : ((EPI_OFF + 4 * 2 * 4096 + 1024 <= 232448) ? 2 : 1);
  static constexpr int SMEM = EPI_OFF + 4 * EPI_BUFS * 4096 + 1024;
};

// EPI: 0 = plain / residual / rope epilogue, 1 = fused SwiGLU (gate|up forward), 2 = fused SwiGLU
// backward (down-projection dgrad)
template <int BN, bool A_MN, bool B_MN, int EPI = 0>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    gemm2_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                 const __grid_constant__ CUtensorMap tmD, const __grid_constant__ CUtensorMap tmAct,
                 __nv_bfloat16* __restrict__ D, const __nv_bfloat16* C /* may alias D */, int M, int N, int K,
                 int64_t ldd, int* __restrict__ sched, RopeArgs rope) {
  ::kpo::pdl_launch_dependents();  // the next kernel may start its prologue; it waits for us
  using CF = Cfg2<BN, EPI>;
  constexpr int STAGES = CF::STAGES;
  constexpr int HB = BN / 2;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + CF::BAR_OFF);
  uint64_t* full = bars;
  uint64_t* empty = bars + STAGES;
  uint64_t* tfull = bars + 2 * STAGES;
  uint64_t* tempty = tfull + 2;
  uint64_t* sfull = tempty + 2;
  uint64_t* sempty = sfull + 2;
  int* stile = reinterpret_cast<int*>(sempty + 2);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(stile + 2);
  uint64_t* ebar = sempty + 4;  // [warp][slot]: TMA loads of the fused SwiGLU backward's gu boxes

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  const int num_m = (M + 255) / 256, num_n = (N + BN - 1) / BN;
  const int num_tiles = num_m * num_n;
  const int num_kb = (K + BK - 1) / BK;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(smem_u32(&full[s]), 1);
      mbar_init(smem_u32(&empty[s]), 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(smem_u32(&tfull[i]), 1);
      mbar_init(smem_u32(&tempty[i]), 8);
      mbar_init(smem_u32(&sfull[i]), 1);
      mbar_init(smem_u32(&sempty[i]), 10);
    }
    if (EPI == 2)
      for (int i = 0; i < 8; ++i) mbar_init(smem_u32(&ebar[i]), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
  }
  if (warp == 1) tmem_alloc_pair(smem_u32(tmem_slot), CF::TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  ::kpo::pdl_wait();  // inputs, scheduler words and outputs of the previous kernel are settled
  const uint32_t leader_sempty0 = mapa(smem_u32(&sempty[0]), 0);
  const uint32_t leader_tempty0 = mapa(smem_u32(&tempty[0]), 0);

  if (warp == 0) {
    if (lane == 0) {
      // ===================== tile scheduler (leader) + TMA producer (both CTAs)
      int it = 0, stage = 0;
      uint32_t phase = 0;
      while (true) {
        const int slot = it & 1;
        int tile;
        if (leader) {
          tile = atomicAdd(&sched[0], 1);
          mbar_wait_cluster(smem_u32(&sempty[slot]), ((it >> 1) & 1) ^ 1);
          stile[slot] = tile;
          st_cluster_u32(mapa(smem_u32(&stile[slot]), 1), (uint32_t)tile);
          mbar_arrive(smem_u32(&sfull[slot]));
          mbar_arrive_remote(mapa(smem_u32(&sfull[slot]), 1));
        } else {
          mbar_wait_cluster(smem_u32(&sfull[slot]), (it >> 1) & 1);
          tile = stile[slot];
          mbar_arrive_remote(leader_sempty0 + slot * 8);
        }
        ++it;
        if (tile >= num_tiles) break;
        int mb, nb;
        tile_coords(tile, num_m, num_n, mb, nb);
        const int m0 = mb * 256 + (int)rank * 128, n0 = nb * BN + (int)rank * HB;
        for (int kb = 0; kb < num_kb; ++kb) {
          mbar_wait(smem_u32(&empty[stage]), phase ^ 1);
          const uint32_t fb = smem_u32(&full[stage]);
          if (leader) mbar_arrive_expect_tx(fb, 2 * CF::STAGE_BYTES);
          const uint32_t sa = smem_u32(smem + stage * CF::STAGE_BYTES);
          const uint32_t sb = sa + CF::A_BYTES;
          const int k0 = kb * BK;
          if (!A_MN) {
            tma_load_2d_pair(sa, &tmA, fb, k0, m0);
          } else {
#pragma unroll
            for (int c = 0; c < 2; ++c) tma_load_2d_pair(sa + c * (BK * 128), &tmA, fb, m0 + c * 64, k0);
          }
          if (!B_MN) {
            tma_load_2d_pair(sb, &tmB, fb, k0, n0);
          } else {
#pragma unroll
            for (int c = 0; c < HB / 64; ++c) tma_load_2d_pair(sb + c * (BK * 128), &tmB, fb, n0 + c * 64, k0);
          }
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
      if (leader) {
        __threadfence();
        const int done = atomicAdd(&sched[1], 1);
        if (done == (int)(gridDim.x / 2) - 1) {
          sched[0] = 0;
          sched[1] = 0;
          __threadfence();
        }
      }
    }
  } else if (warp == 1) {
    if (leader) {
      // ===================== MMA issuer (leader CTA's warp 1, M = 256 across the pair; elect.sync issues)
      constexpr uint32_t IDESC = idesc_bf16(256, BN, A_MN, B_MN);
      constexpr uint32_t A_LBO = A_MN ? BK * 128 : 16, A_SBO = 1024;
      constexpr uint32_t B_LBO = B_MN ? BK * 128 : 16, B_SBO = 1024;
      constexpr uint32_t A_KSTEP = A_MN ? 16 * 128 : 32;
      constexpr uint32_t B_KSTEP = B_MN ? 16 * 128 : 32;
      int it = 0, stage = 0, acc_it = 0;
      uint32_t phase = 0;
      while (true) {
        const int slot = it & 1;
        mbar_wait(smem_u32(&sfull[slot]), (it >> 1) & 1);
        const int tile = stile[slot];
        __syncwarp();
        if (lane == 0) mbar_arrive(smem_u32(&sempty[slot]));
        ++it;
        if (tile >= num_tiles) break;
        const int acc = acc_it & 1;
        mbar_wait_cluster(smem_u32(&tempty[acc]), ((acc_it >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = 0; kb < num_kb; ++kb) {
          mbar_wait(smem_u32(&full[stage]), phase);
          tc_fence_after();
          const uint32_t sa = smem_u32(smem + stage * CF::STAGE_BYTES);
          const uint32_t sb = sa + CF::A_BYTES;
          static_assert(A_SBO == 1024 && B_SBO == 1024, "split descriptors assume SBO 1024 / SWIZZLE_128B");
          const uint32_t a_lo = desc_lo(sa, A_LBO), b_lo = desc_lo(sb, B_LBO);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k)
            tc_mma_pair_lo_w(d_tmem, a_lo + k * (A_KSTEP >> 4), b_lo + k * (B_KSTEP >> 4), IDESC, (kb | k) != 0);
          tc_commit_pair_w(smem_u32(&empty[stage]));
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        tc_commit_pair_w(smem_u32(&tfull[acc]));
        ++acc_it;
      }
    }
  } else {
    // ===================== epilogue warps 2..5 (both CTAs): this CTA's 128 rows, all BN columns
    const int q = warp & 3;
    int it = 0, acc_it = 0, store_cnt = 0;
    uint32_t echunks = 0;  // fused SwiGLU backward: gate / up box pairs this warp has consumed
    while (true) {
      const int slot = it & 1;
      if (leader) mbar_wait(smem_u32(&sfull[slot]), (it >> 1) & 1);
      else mbar_wait_cluster(smem_u32(&sfull[slot]), (it >> 1) & 1);
      const int tile = stile[slot];
      __syncwarp();
      if (lane == 0) {
        if (leader) mbar_arrive(smem_u32(&sempty[slot]));
        else mbar_arrive_remote(leader_sempty0 + slot * 8);
      }
      ++it;
      if (tile >= num_tiles) break;
      int mb, nb;
      tile_coords(tile, num_m, num_n, mb, nb);
      const int acc = acc_it & 1;
      const int row = mb * 256 + (int)rank * 128 + q * 32 + lane;
      if constexpr (EPI == 2) {
        static_assert(BN == 256, "fused SwiGLU backward: 256x256 pair tiles");
        epilogue_swiglu_bwd(tmem_base + ((uint32_t)(q * 32) << 16) + acc * BN, &tmD, &tmAct, nb * BN,
                            mb * 256 + (int)rank * 128 + q * 32,
                            smem_u32(smem + CF::EPI_OFF) + q * CF::EPI_BUFS * 4096, smem_u32(&ebar[q * 2]), echunks,
                            lane,
                            [&] {
                              mbar_wait(smem_u32(&tfull[acc]), (acc_it >> 1) & 1);
                              tc_fence_after();
                            },
                            [&] {  // the accumulator is in registers: release it to the MMA warp
                              tc_fence_before();
                              __syncwarp();
                              if (lane == 0) mbar_arrive_remote(leader_tempty0 + acc * 8);
                            });
      } else if constexpr (EPI == 1) {
        static_assert(BN == 256 && !A_MN && !B_MN, "fused SwiGLU: TN 256x256 pair tiles");
        mbar_wait(smem_u32(&tfull[acc]), (acc_it >> 1) & 1);
        tc_fence_after();
        epilogue_swiglu<CF::EPI_BUFS>(tmem_base + ((uint32_t)(q * 32) << 16) + acc * BN, &tmD, &tmAct, nb * BN,
                                      nb * (BN / 2), mb * 256 + (int)rank * 128 + q * 32,
                                      smem_u32(smem + CF::EPI_OFF) + q * CF::EPI_BUFS * 4096, lane, store_cnt);
      } else {
        epilogue_row<BN, CF::EPI_BUFS, !A_MN && !B_MN>(tmem_base + ((uint32_t)(q * 32) << 16) + acc * BN, &tmD, C, row,
                                                       row < M, nb * BN, N, ldd, mb * 256 + (int)rank * 128 + q * 32,
                                                       smem_u32(smem + CF::EPI_OFF) + q * CF::EPI_BUFS * 4096, lane,
                                                       store_cnt, rope, [&] {
                                                         mbar_wait(smem_u32(&tfull[acc]), (acc_it >> 1) & 1);
                                                         tc_fence_after();
                                                       });
      }
      if constexpr (EPI != 2) {
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_remote(leader_tempty0 + acc * 8);
      }
      ++acc_it;
    }
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");  // D stores complete
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  if (warp == 1) tmem_dealloc_pair(tmem_base, CF::TMEM_COLS);
}

template <int BN, bool A_MN, bool B_MN, int EPI = 0>
static int launch2(const CUtensorMap& ta, const CUtensorMap& tb, void* D, const void* C, int64_t M, int64_t N,
                   int64_t K, int64_t ldd, int grid, int* sched, cudaStream_t s, RopeArgs rope,
                   void* act = nullptr, int64_t ldact = 0) {
  auto kern = gemm2_kernel<BN, A_MN, B_MN, EPI>;
  CUtensorMap td, tact;
  // EPI 2: D = dgu [M, 2N] (output), act = gu [M, 2N] (loaded); EPI 1: D = gu [M, N], act [M, N/2]
  if (int e = make_map_2d(&td, D, EPI == 2 ? 2 * N : N, M, ldd, 64, 32)) return e;
  if (EPI == 1) {
    if (int e = make_map_2d(&tact, act, N / 2, M, ldact, 64, 32)) return e;
  } else if (EPI == 2) {
    if (int e = make_map_2d(&tact, act, 2 * N, M, ldact, 64, 32)) return e;
  } else {
    tact = td;
  }
  static bool attr_set = false;
  if (!attr_set) {
    KPO_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg2<BN, EPI>::SMEM));
    attr_set = true;
  }
  KPO_CUDA(::kpo::pdl_launch(kern, grid, kThreads, Cfg2<BN, EPI>::SMEM, s, ta, tb, td, tact, (__nv_bfloat16*)D, (const __nv_bfloat16*)C, (int)M, (int)N,
                                               (int)K, ldd, sched, rope));
  KPO_LAUNCH_CHECK();
  return KPO_OK;
}
}  // namespace gemm

namespace sm100 {
PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// 2-D bf16 tensor map: inner (contiguous) extent, outer extent, outer stride (elements), box, SW128.
int make_map_2d(CUtensorMap* m, const void* ptr, uint64_t inner, uint64_t outer, uint64_t stride_elems,
                uint32_t box_inner, uint32_t box_outer) {
  auto enc = get_encode();
  if (!enc) {
    set_error("cuTensorMapEncodeTiled unavailable");
    return KPO_ERR_UNSUPPORTED;
  }
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {stride_elems * 2};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled failed (%d) inner=%llu outer=%llu stride=%llu", (int)r,
              (unsigned long long)inner, (unsigned long long)outer, (unsigned long long)stride_elems);
    return KPO_ERR_INVALID;
  }
  return KPO_OK;
}
int make_map_2d_f32(CUtensorMap* m, const void* ptr, uint64_t inner, uint64_t outer, uint64_t stride_elems,
                    uint32_t box_inner, uint32_t box_outer, bool swizzle128) {
  auto enc = get_encode();
  if (!enc) {
    set_error("cuTensorMapEncodeTiled unavailable");
    return KPO_ERR_UNSUPPORTED;
  }
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {stride_elems * 4};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(ptr), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, swizzle128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled(f32) failed (%d)", (int)r);
    return KPO_ERR_INVALID;
  }
  return KPO_OK;
}
}  // namespace sm100
}  // namespace kpo

using namespace kpo;
using namespace kpo::sm100;

static int gemm_impl(const void* A, const void* B, void* D, const void* C, int64_t M, int64_t N, int64_t K,
                     int a_mn_major, int b_mn_major, int64_t lda, int64_t ldb, int64_t ldd, int max_ctas, int* sched,
                     void* stream, kpo::gemm::RopeArgs rope) {
  using namespace kpo::gemm;
  KPO_CHECK_ARG(A && B && D && sched, "gemm: null pointer");
  KPO_CHECK_ARG(M > 0 && N > 0 && K > 0, "gemm: M, N, K must be positive");
  KPO_CHECK_ARG(M < (1ll << 31) && N < (1ll << 31) && K < (1ll << 31), "gemm: dims too large");
  KPO_CHECK_ARG(N % 8 == 0 && K % 8 == 0 && ldd % 8 == 0 && lda % 8 == 0 && ldb % 8 == 0,
                "gemm: N, K and leading dimensions must be multiples of 8");
  KPO_CHECK_ARG(((uintptr_t)A & 15) == 0 && ((uintptr_t)B & 15) == 0 && ((uintptr_t)D & 15) == 0 &&
                    ((uintptr_t)C & 15) == 0,
                "gemm: pointers must be 16B aligned");
  KPO_CHECK_ARG(ldd >= N, "gemm: ldd < N");
  KPO_CHECK_ARG(a_mn_major ? lda >= M : lda >= K, "gemm: lda too small");
  KPO_CHECK_ARG(b_mn_major ? ldb >= N : ldb >= K, "gemm: ldb too small");
  const int sms = num_sms();
  // Tile choice: maximise (useful fraction of padded N) x (SM-wave fill) x (per-tile efficiency measured on
  // B200 for the layer shapes, tools/gemm_bench.py): CTA-pair 256xBN tiles halve B's shared-memory
  // traffic per FLOP; single-CTA BN=128 tiles are shared-memory-bandwidth bound.
  struct Choice { bool pair; int bn; double base; };
  const Choice choices[] = {{true, 256, 1.00}, {true, 128, 0.74}, {false, 256, 0.90}, {false, 192, 0.86},
                            {false, 128, 0.64}};
  auto eff = [&](const Choice& c) {
    const int units = c.pair ? sms / 2 : sms;
    const int bm = c.pair ? 256 : BM;
    const int64_t nt = (N + c.bn - 1) / c.bn;
    const int64_t tiles = ((M + bm - 1) / bm) * nt;
    const int64_t waves = (tiles + units - 1) / units;
    const double mfill = (double)M / (double)(((M + bm - 1) / bm) * bm);
    return (double)N / (double)(nt * c.bn) * mfill * (double)tiles / (double)(waves * units) * c.base;
  };
  static const bool no_pair = getenv("KPO_GEMM_NO_PAIR") != nullptr;
  Choice best = {false, 256, 0.0};
  double best_eff = -1.0;
  for (const Choice& c : choices) {
    if (c.pair && (no_pair || M < 256)) continue;
    if (rope.cs && c.bn % 128 != 0) continue;  // rope tiles hold whole 128-column heads
    const double e = eff(c);
    if (e > best_eff * 1.01) {
      best = c;
      best_eff = e;
    }
  }
  const int bn = best.bn;
  const int64_t tiles = ((M + BM - 1) / BM) * ((N + bn - 1) / bn);
  int cap = max_ctas > 0 ? max_ctas : sms;
  if (cap > sms) cap = sms;
  const int grid = (int)(tiles < cap ? tiles : cap);

  // CTA-pair (cta_group::2) path: 256 x BN tiles, BN in {256, 128} chosen by the same wave model
  if (best.pair) {
    const int clusters = sms / 2;
    const int bn2 = best.bn;
    const int64_t tiles2 = ((M + 255) / 256) * ((N + bn2 - 1) / bn2);
    int cap2 = max_ctas > 0 ? max_ctas / 2 : clusters;
    if (cap2 < 1) cap2 = 1;
    if (cap2 > clusters) cap2 = clusters;
    const int grid2 = 2 * (int)(tiles2 < cap2 ? tiles2 : cap2);
    CUtensorMap ta2, tb2;
    int st2;
    if (!a_mn_major) st2 = make_map_2d(&ta2, A, K, M, lda, BK, 128);
    else st2 = make_map_2d(&ta2, A, M, K, lda, 64, BK);
    if (st2) return st2;
    if (!b_mn_major) st2 = make_map_2d(&tb2, B, K, N, ldb, BK, bn2 / 2);
    else st2 = make_map_2d(&tb2, B, N, K, ldb, 64, BK);
    if (st2) return st2;
    cudaStream_t s2 = (cudaStream_t)stream;
#define KPO_GEMM2_DISPATCH(BNv)                                                                                    \
  if (!a_mn_major && !b_mn_major) return launch2<BNv, false, false>(ta2, tb2, D, C, M, N, K, ldd, grid2, sched, s2, rope); \
  if (!a_mn_major && b_mn_major) return launch2<BNv, false, true>(ta2, tb2, D, C, M, N, K, ldd, grid2, sched, s2, rope);   \
  if (a_mn_major && !b_mn_major) return launch2<BNv, true, false>(ta2, tb2, D, C, M, N, K, ldd, grid2, sched, s2, rope);   \
  return launch2<BNv, true, true>(ta2, tb2, D, C, M, N, K, ldd, grid2, sched, s2, rope);
    if (bn2 == 256) {
      KPO_GEMM2_DISPATCH(256)
    } else {
      KPO_GEMM2_DISPATCH(128)
    }
#undef KPO_GEMM2_DISPATCH
  }
  CUtensorMap ta, tb;
  int st;
  if (!a_mn_major) st = make_map_2d(&ta, A, K, M, lda, BK, BM);
  else st = make_map_2d(&ta, A, M, K, lda, 64, BK);
  if (st) return st;
  if (!b_mn_major) st = make_map_2d(&tb, B, K, N, ldb, BK, bn);
  else st = make_map_2d(&tb, B, N, K, ldb, 64, BK);
  if (st) return st;
  cudaStream_t s = (cudaStream_t)stream;
#define KPO_GEMM_DISPATCH(BNv)                                                                      \
  if (!a_mn_major && !b_mn_major) return launch<BNv, false, false>(ta, tb, D, C, M, N, K, ldd, grid, sched, s, rope); \
  if (!a_mn_major && b_mn_major) return launch<BNv, false, true>(ta, tb, D, C, M, N, K, ldd, grid, sched, s, rope);   \
  if (a_mn_major && !b_mn_major) return launch<BNv, true, false>(ta, tb, D, C, M, N, K, ldd, grid, sched, s, rope);   \
  return launch<BNv, true, true>(ta, tb, D, C, M, N, K, ldd, grid, sched, s, rope);
  if (bn == 256) {
    KPO_GEMM_DISPATCH(256)
  } else if (bn == 192) {
    KPO_GEMM_DISPATCH(192)
  } else {
    KPO_GEMM_DISPATCH(128)
  }
#undef KPO_GEMM_DISPATCH
}

extern "C" int kpo_gemm(const void* A, const void* B, void* D, const void* C, int64_t M, int64_t N, int64_t K,
                        int a_mn_major, int b_mn_major, int64_t lda, int64_t ldb, int64_t ldd, int max_ctas,
                        int* sched, void* stream) {
  return gemm_impl(A, B, D, C, M, N, K, a_mn_major, b_mn_major, lda, ldb, ldd, max_ctas, sched, stream,
                   kpo::gemm::RopeArgs{nullptr, 0});
}

extern "C" int kpo_gemm_rope(const void* A, const void* B, void* D, int64_t M, int64_t N, int64_t K, int64_t lda,
                             int64_t ldb, int64_t ldd, int max_ctas, int* sched, const float* rope_table,
                             int64_t rope_cols, int head_dim, void* stream) {
  KPO_CHECK_ARG(rope_table, "gemm_rope: null rope table");
  KPO_CHECK_ARG(head_dim == 128, "gemm_rope: the fused rotary epilogue handles head_dim 128");
  KPO_CHECK_ARG(rope_cols > 0 && rope_cols % head_dim == 0 && rope_cols <= N,
                "gemm_rope: rope_cols must be a positive multiple of head_dim within N");
  return gemm_impl(A, B, D, nullptr, M, N, K, 0, 0, lda, ldb, ldd, max_ctas, sched, stream,
                   kpo::gemm::RopeArgs{reinterpret_cast<const float2*>(rope_table), (int)rope_cols});
}

extern "C" int kpo_gemm_swiglu(const void* A, const void* B, void* gu, void* act, int64_t M, int64_t N, int64_t K,
                               int64_t lda, int64_t ldb, int64_t ldgu, int64_t ldact, int max_ctas, int* sched,
                               void* stream) {
  using namespace kpo::gemm;
  KPO_CHECK_ARG(A && B && gu && act && sched, "gemm_swiglu: null pointer");
  KPO_CHECK_ARG(M >= 256 && M < (1ll << 31) && K > 0 && K % 8 == 0 && K < (1ll << 31),
                "gemm_swiglu: M must be >= 256 (CTA-pair tiles) and K a positive multiple of 8");
  KPO_CHECK_ARG(N > 0 && N % 256 == 0 && N < (1ll << 31),
                "gemm_swiglu: N (= 2 * ffn) must be a multiple of 256 (128-row gate / up blocks)");
  KPO_CHECK_ARG(lda >= K && ldb >= K && ldgu >= N && ldact >= N / 2 && lda % 8 == 0 && ldb % 8 == 0 &&
                    ldgu % 8 == 0 && ldact % 8 == 0,
                "gemm_swiglu: bad leading dimensions");
  KPO_CHECK_ARG(((uintptr_t)A & 15) == 0 && ((uintptr_t)B & 15) == 0 && ((uintptr_t)gu & 15) == 0 &&
                    ((uintptr_t)act & 15) == 0,
                "gemm_swiglu: pointers must be 16B aligned");
  const int clusters = num_sms() / 2;
  const int64_t tiles = ((M + 255) / 256) * (N / 256);
  int cap = max_ctas > 0 ? max_ctas / 2 : clusters;
  if (cap < 1) cap = 1;
  if (cap > clusters) cap = clusters;
  const int grid = 2 * (int)(tiles < cap ? tiles : cap);
  CUtensorMap ta, tb;
  if (int e = make_map_2d(&ta, A, K, M, lda, BK, 128)) return e;
  if (int e = make_map_2d(&tb, B, K, N, ldb, BK, 128)) return e;
  return launch2<256, false, false, 1>(ta, tb, gu, nullptr, M, N, K, ldgu, grid, sched, (cudaStream_t)stream,
                                          RopeArgs{nullptr, 0}, act, ldact);
}

extern "C" int kpo_gemm_swiglu_bwd(const void* dy, const void* w, const void* gu, void* dgu, int64_t M, int64_t N,
                                   int64_t K, int64_t lddy, int64_t ldw, int64_t ldgu, int64_t lddgu, int max_ctas,
                                   int* sched, void* stream) {
  using namespace kpo::gemm;
  KPO_CHECK_ARG(dy && w && gu && dgu && sched, "gemm_swiglu_bwd: null pointer");
  KPO_CHECK_ARG(M >= 256 && M < (1ll << 31) && K > 0 && K % 8 == 0 && K < (1ll << 31),
                "gemm_swiglu_bwd: M must be >= 256 (CTA-pair tiles) and K a positive multiple of 8");
  KPO_CHECK_ARG(N > 0 && N % 256 == 0 && N < (1ll << 30),
                "gemm_swiglu_bwd: N (= ffn) must be a multiple of 256 (two 128-column gate / up blocks per tile)");
  KPO_CHECK_ARG(lddy >= K && ldw >= N && ldgu >= 2 * N && lddgu >= 2 * N && lddy % 8 == 0 && ldw % 8 == 0 &&
                    ldgu % 8 == 0 && lddgu % 8 == 0,
                "gemm_swiglu_bwd: bad leading dimensions");
  KPO_CHECK_ARG(((uintptr_t)dy & 15) == 0 && ((uintptr_t)w & 15) == 0 && ((uintptr_t)gu & 15) == 0 &&
                    ((uintptr_t)dgu & 15) == 0,
                "gemm_swiglu_bwd: pointers must be 16B aligned");
  const int clusters = num_sms() / 2;
  const int64_t tiles = ((M + 255) / 256) * (N / 256);
  int cap = max_ctas > 0 ? max_ctas / 2 : clusters;
  if (cap < 1) cap = 1;
  if (cap > clusters) cap = clusters;
  const int grid = 2 * (int)(tiles < cap ? tiles : cap);
  CUtensorMap ta, tb;
  if (int e = make_map_2d(&ta, dy, K, M, lddy, BK, 128)) return e;
  if (int e = make_map_2d(&tb, w, N, K, ldw, 64, BK)) return e;
  return launch2<256, false, true, 2>(ta, tb, dgu, nullptr, M, N, K, lddgu, grid, sched, (cudaStream_t)stream,
                                      RopeArgs{nullptr, 0}, const_cast<void*>(gu), ldgu);
}
