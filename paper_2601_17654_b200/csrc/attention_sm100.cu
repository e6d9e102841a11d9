// attention_sm100.cu — causal GQA flash attention on the 5th-gen tensor cores (tcgen05 + TMEM + TMA).
//
// Replaces the reference's abstract "attention_core" kernel (workloads.py:47).  Forward, one CTA =
// 128 query rows of one q head, 128-key tiles:
//   warp 0     TMA producer: Q once, then K_j / V_j into a 2-stage smem ring (128B swizzle)
//   warp 1     TMEM allocator + single-thread tcgen05.mma issuer:
//                S_j = Q K_j^T  -> TMEM (double-buffered, 2 x 128 columns)
//                O  += P_j V_j  -> TMEM (D columns), P_j from smem, V_j MN-major from smem
//   warps 2-5  softmax: one thread owns one query row (its TMEM lane), so row max / row sum need
//              no shuffles; P_j is written to smem in the UMMA K-major SW128 layout; O is rescaled
//              in TMEM only when the running max grows by more than 2^8 (lazy rescaling), then
//              normalised, converted and stored at the end together with the log-sum-exp.
// The issue order S_0, S_1, PV_0, S_2, PV_1, ... lets the softmax of tile j overlap the tensor
// core's work on tiles j+1 / j-1.
#include "sm100.cuh"

namespace kpo {
namespace attn_tc {
using namespace kpo::sm100;

constexpr float kLog2e = 1.4426950408889634f;
constexpr int kThreads = 320;  // TMA warp, MMA warp, 8 softmax warps (two per TMEM lane quarter)

template <int D>
struct Fwd {
  // K and V have separate rings (3 and 2 stages): K_j is released as soon as S_j is done, V_j after
  // P_j V_j, so the next tiles' loads start early enough to hide the L2 latency (measured: with one
  // 2-stage K+V ring the S MMAs waited on the loads ~1/4 of the time)
  static constexpr int BM = 128, BN = 128, STAGES = 3, VSTAGES = 2;
  static constexpr int Q_BYTES = BM * D * 2;  // D/64 sub-tiles of [128 rows x 64] (16 KB each)
  static constexpr int KV_BYTES = BN * D * 2;
  static constexpr int OFF_Q = 0;
  static constexpr int OFF_K = OFF_Q + Q_BYTES;
  static constexpr int OFF_V = OFF_K + STAGES * KV_BYTES;
  static constexpr int OFF_BAR = OFF_V + VSTAGES * KV_BYTES;
  static constexpr int OFF_XCH = OFF_BAR + 256;  // [2 parities][2 halves][128 rows] fp32 row-max exchange
  static constexpr int SMEM_RAW = OFF_XCH + 2 * 2 * 128 * 4 + 1024;
  // keep one CTA per SM (the kernel allocates all 512 TMEM columns)
  static constexpr int SMEM = SMEM_RAW > 120 * 1024 ? SMEM_RAW : 120 * 1024;
  static constexpr int TMEM_COLS = 512;
  // S_j in buffer j & 1; the softmax overwrites the first 64 columns of S_j with P_j (bf16 pairs),
  // the TMEM A operand of the P V MMA
  static constexpr int COL_S0 = 0, COL_S1 = 128, COL_O = 256;
};

__device__ __forceinline__ void named_bar(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n)); }

// byte offset of the 16-byte chunk `chunk` (0..7) of row `r` in a [rows x 64] bf16 SW128 sub-tile
__device__ __forceinline__ uint32_t sw128(int r, int chunk) {
  return (uint32_t)(r * 128 + ((chunk ^ (r & 7)) << 4));
}

template <int D, int POLY_MASK>
__global__ void __launch_bounds__(kThreads, 1)
    attn_fwd_tc_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                       const __grid_constant__ CUtensorMap tmV, __nv_bfloat16* __restrict__ o, float* __restrict__ lse,
                       int T, int hq, int hkv, int64_t os, float scale_log2, int causal) {
  ::kpo::pdl_launch_dependents();  // the next kernel may start its prologue; it waits for us
  using C = Fwd<D>;
  constexpr int BM = C::BM, BN = C::BN, KSUB = D / 64;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + C::OFF_BAR);
  uint64_t* q_full = bar + 0;
  uint64_t* k_full = bar + 1;    // [3]
  uint64_t* k_empty = bar + 4;   // [3]
  uint64_t* v_full = bar + 7;    // [3]
  uint64_t* v_empty = bar + 10;  // [3]
  uint64_t* s_full = bar + 13;   // [2]
  uint64_t* p_full = bar + 15;   // [2]
  uint64_t* pv_done = bar + 17;  // [2]  PV(i) commits to pv_done[i & 1]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 19);
  constexpr int KS = C::STAGES, VS = C::VSTAGES;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int mblk = gridDim.y - 1 - blockIdx.y;  // heavy (late) causal rows first, all heads of a row-tile together
  const int h = blockIdx.x;
  const int kvh = h / (hq / hkv);
  const int m0 = mblk * BM;
  int n_tiles = (T + BN - 1) / BN;
  if (causal) n_tiles = min(n_tiles, (m0 + BM + BN - 1) / BN);

  if (threadIdx.x == 0) {
    mbar_init(smem_u32(q_full), 1);
    for (int i = 0; i < KS; ++i) {
      mbar_init(smem_u32(&k_full[i]), 1);
      mbar_init(smem_u32(&k_empty[i]), 1);
    }
    for (int i = 0; i < VS; ++i) {
      mbar_init(smem_u32(&v_full[i]), 1);
      mbar_init(smem_u32(&v_empty[i]), 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(smem_u32(&s_full[i]), 1);
      mbar_init(smem_u32(&p_full[i]), 8);
      mbar_init(smem_u32(&pv_done[i]), 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) tmem_alloc(smem_u32(tmem_slot), C::TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  // one CTA per SM owns all 512 columns, so the allocation starts at lane 0 / column 0; a constant base
  // keeps every TMEM address of the MMA issue loops in uniform registers (no per-MMA R2UR)
  if (*tmem_slot != 0) __trap();
  ::kpo::pdl_wait();  // the previous kernel's outputs (our inputs) are complete and visible
  constexpr uint32_t tmem = 0;
  const uint32_t sQ = smem_u32(smem + C::OFF_Q), sK = smem_u32(smem + C::OFF_K);
  const uint32_t sV = smem_u32(smem + C::OFF_V);

  if (warp == 0) {
    if (lane == 0) {
      // ---------------------------------------------------------------- TMA producer
      mbar_arrive_expect_tx(smem_u32(q_full), C::Q_BYTES);
#pragma unroll
      for (int kb = 0; kb < KSUB; ++kb) tma_load_2d(sQ + kb * BM * 128, &tmQ, smem_u32(q_full), h * D + kb * 64, m0);
      for (int j = 0, s = 0, ph = 0, v = 0, vph = 0; j < n_tiles; ++j) {
        mbar_wait(smem_u32(&k_empty[s]), ph ^ 1);
        uint32_t fb = smem_u32(&k_full[s]);
        mbar_arrive_expect_tx(fb, C::KV_BYTES);
#pragma unroll
        for (int kb = 0; kb < KSUB; ++kb)
          tma_load_2d(sK + s * C::KV_BYTES + kb * BN * 128, &tmK, fb, kvh * D + kb * 64, j * BN);
        mbar_wait(smem_u32(&v_empty[v]), vph ^ 1);
        fb = smem_u32(&v_full[v]);
        mbar_arrive_expect_tx(fb, C::KV_BYTES);
#pragma unroll
        for (int kb = 0; kb < KSUB; ++kb)
          tma_load_2d(sV + v * C::KV_BYTES + kb * BN * 128, &tmV, fb, kvh * D + kb * 64, j * BN);
        if (++s == KS) s = 0, ph ^= 1;
        if (++v == VS) v = 0, vph ^= 1;
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---------------------------------------------------------------- MMA issuer
      constexpr uint32_t ID_S = idesc_bf16(BM, BN, false, false);
      constexpr uint32_t ID_O = idesc_bf16(BM, D, false, true);
      mbar_wait(smem_u32(q_full), 0);
      const uint32_t q_k = desc_lo(sQ, 16);
      auto issue_pv = [&](int i) {
        const int vs = i % VS;
        mbar_wait(smem_u32(&v_full[vs]), (i / VS) & 1);
        mbar_wait(smem_u32(&p_full[i & 1]), (i >> 1) & 1);
        tc_fence_after();
        const uint32_t v_mn = desc_lo(sV + vs * C::KV_BYTES, BN * 128);
        const uint32_t p_t = tmem + ((i & 1) ? C::COL_S1 : C::COL_S0);
#pragma unroll
        for (int kk = 0; kk < BN / 16; ++kk)  // 16 keys per UMMA, P from TMEM (8 columns of bf16 pairs)
          tc_mma_ts_lo(tmem + C::COL_O, p_t + kk * 8, v_mn + kk * 128, ID_O, (i > 0 || kk > 0) ? 1u : 0u);
        tc_commit(smem_u32(&pv_done[i & 1]));
        tc_commit(smem_u32(&v_empty[vs]));
      };
      for (int j = 0; j < n_tiles; ++j) {
        const int s = j & 1, ks = j % KS;
        mbar_wait(smem_u32(&k_full[ks]), (j / KS) & 1);
        // buffer s holds P_{j-2}: PV_{j-2} was issued before this S_j and tcgen05.mma executes in
        // issue order, so no wait is needed
        tc_fence_after();
        const uint32_t k_k = desc_lo(sK + ks * C::KV_BYTES, 16);
        const uint32_t d_s = tmem + (s ? C::COL_S1 : C::COL_S0);
#pragma unroll
        for (int kb = 0; kb < KSUB; ++kb) {
#pragma unroll
          for (int k = 0; k < 4; ++k)
            tc_mma_lo(d_s, q_k + kb * (BM * 8) + k * 2, k_k + kb * (BN * 8) + k * 2, ID_S, (kb | k) ? 1u : 0u);
        }
        tc_commit(smem_u32(&s_full[s]));
        tc_commit(smem_u32(&k_empty[ks]));
        if (j > 0) issue_pv(j - 1);
      }
      issue_pv(n_tiles - 1);
    }
  } else {
    // ---------------------------------------------------------------- softmax warps 2..9
    // Two warps per TMEM lane quarter (warp % 4): the row's 128 keys are split in two halves of 64, so
    // every SM sub-partition runs two softmax warps and one's MUFU / FMA latency hides under the
    // other's.  The halves exchange their row max through shared memory once per tile (named barrier
    // per quarter); the row sums stay per half and are combined in the epilogue.
    const int quarter = warp & 3;
    const int half = (warp - 2) >> 2;
    const int r = quarter * 32 + lane;  // query row within the tile == TMEM lane
    const int q = m0 + r;
    const uint32_t lane_addr = tmem + ((uint32_t)(quarter * 32) << 16);
    float* xch = reinterpret_cast<float*>(smem + C::OFF_XCH);  // [parity][half][row]
    const int bar_id = 1 + quarter;
    float m_run = -INFINITY, l_run = 0.f;
    for (int j = 0; j < n_tiles; ++j) {
      const int s = j & 1;
      mbar_wait(smem_u32(&s_full[s]), (j >> 1) & 1);
      tc_fence_after();
      constexpr int HN = BN / 2;
      float sv[HN];
      const uint32_t s_addr = lane_addr + (s ? C::COL_S1 : C::COL_S0);
#pragma unroll
      for (int c = 0; c < HN / 32; ++c)
        tmem_ld32_nowait(s_addr + half * HN + c * 32, reinterpret_cast<uint32_t*>(sv + c * 32));
      tmem_wait_ld();
      const int k0 = j * BN + half * HN;
      const bool mask = (causal && j * BN + BN - 1 > m0) || (j * BN + BN > T);  // CTA-uniform
      if (mask) {
#pragma unroll
        for (int i = 0; i < HN; ++i) {
          const int key = k0 + i;
          sv[i] = (key >= T || (causal && key > q)) ? -INFINITY : sv[i];
        }
      }
      // row max over raw scores with 8 independent chains (scale > 0 commutes with max)
      float pm[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) pm[e] = sv[e];
#pragma unroll
      for (int i = 8; i < HN; ++i) pm[i & 7] = fmaxf(pm[i & 7], sv[i]);
      float mx = fmaxf(fmaxf(fmaxf(pm[0], pm[1]), fmaxf(pm[2], pm[3])), fmaxf(fmaxf(pm[4], pm[5]), fmaxf(pm[6], pm[7])));
      xch[(s * 2 + half) * BM + r] = mx;
      named_bar(bar_id, 64);
      mx = fmaxf(mx, xch[(s * 2 + (half ^ 1)) * BM + r]) * scale_log2;
      float corr = 1.f;
      bool rescale = false;
      if (mx > m_run + 8.f) {  // lazy rescaling: only when the max grows by more than 2^8
        corr = (m_run == -INFINITY) ? 0.f : ex2(m_run - mx);
        rescale = (j > 0);
        m_run = mx;
      }
      // tcgen05.ld/st are warp-collective (.sync.aligned): the rescale decision must be warp-uniform;
      // lanes that do not need it multiply by corr == 1.  Each half rescales its 64 output columns.
      if (__any_sync(0xffffffffu, rescale)) {
        mbar_wait(smem_u32(&pv_done[s ^ 1]), ((j - 1) >> 1) & 1);  // O stable (PV(j-1) done)
        tc_fence_after();
#pragma unroll 1
        for (int c = 0; c < D / 64; ++c) {
          uint32_t ov[32];
          const uint32_t oa = lane_addr + C::COL_O + half * (D / 2) + c * 32;
          tmem_ld32_nowait(oa, ov);
          tmem_wait_ld();
#pragma unroll
          for (int i = 0; i < 32; ++i) ov[i] = __float_as_uint(__uint_as_float(ov[i]) * corr);
          tmem_st32(oa, ov);
        }
      }
      const float neg_m = -m_run;
      float ps[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
      uint32_t pk[32];  // this half's 64 keys -> 32 columns of bf16 pairs over S_j
#pragma unroll
      for (int c = 0; c < 32; ++c) {
        float p[2];
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int i = c * 2 + e;
          const float xe = fmaf(sv[i], scale_log2, neg_m);
          p[e] = ((POLY_MASK >> (i & 7)) & 1) ? ex2_poly(xe) : ex2(xe);
          ps[i & 7] += p[e];
        }
        pk[c] = pack_bf16x2(p[0], p[1]);
      }
      tmem_st32(s_addr + half * 32, pk);
      const float lsum = ((ps[0] + ps[1]) + (ps[2] + ps[3])) + ((ps[4] + ps[5]) + (ps[6] + ps[7]));
      l_run = l_run * corr + lsum;
      tmem_wait_st();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_u32(&p_full[s]));
    }
    // ---------------------------------------------------------------- epilogue
    // combine the two halves' row sums (the exchange buffer is free: both warps are past their last
    // max exchange once they meet at this barrier)
    named_bar(bar_id, 64);
    xch[half * BM + r] = l_run;
    named_bar(bar_id, 64);
    const float l_tot = l_run + xch[(half ^ 1) * BM + r];
    mbar_wait(smem_u32(&pv_done[(n_tiles - 1) & 1]), ((n_tiles - 1) >> 1) & 1);
    tc_fence_after();
    const float inv = 1.f / l_tot;
    const bool row_ok = q < T;
    __nv_bfloat16* orow = o + (int64_t)q * os + (int64_t)h * D + half * (D / 2);
#pragma unroll 1
    for (int c = 0; c < D / 64; ++c) {
      uint32_t ov[32];
      tmem_ld32_nowait(lane_addr + C::COL_O + half * (D / 2) + c * 32, ov);
      tmem_wait_ld();
      if (row_ok) {
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          uint4 u;
          u.x = pack_bf16x2(__uint_as_float(ov[v * 8 + 0]) * inv, __uint_as_float(ov[v * 8 + 1]) * inv);
          u.y = pack_bf16x2(__uint_as_float(ov[v * 8 + 2]) * inv, __uint_as_float(ov[v * 8 + 3]) * inv);
          u.z = pack_bf16x2(__uint_as_float(ov[v * 8 + 4]) * inv, __uint_as_float(ov[v * 8 + 5]) * inv);
          u.w = pack_bf16x2(__uint_as_float(ov[v * 8 + 6]) * inv, __uint_as_float(ov[v * 8 + 7]) * inv);
          *reinterpret_cast<uint4*>(orow + c * 32 + v * 8) = u;
        }
      }
    }
    if (row_ok && half == 0) lse[(int64_t)h * T + q] = (m_run + __log2f(l_tot)) / kLog2e;
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) tmem_dealloc(tmem, C::TMEM_COLS);
}

// -------------------------------------------------------------------------------------------------
// Forward, two Q tiles per CTA (256 query rows).  Each softmax warpgroup owns one 128-row Q tile and
// one O accumulator; the two groups are fed by different S MMAs at different times, so on every SM
// sub-partition one warp's exponentials (MUFU) overlap the other warp's TMEM loads / row max / P
// stores, and every K / V tile feeds four MMAs (2 S + 2 PV) instead of two.
//   warps 0-3  softmax Q tile 0 (TMEM lanes = rows), warps 4-7 softmax Q tile 1   (setmaxnreg 232)
//   warp 8     TMA producer (Q0, Q1 once; K / V 2-stage rings)                    (setmaxnreg 40)
//   warp 9     TMEM allocator + MMA issuer; warps 10-11 idle
//   TMEM: S0 0..127, S1 128..255 (P_g written over the first 64 columns of S_g), O0 256..383, O1 384..511
//   MMA order: S0_0, S1_0, then per KV tile j and per group g, in the order the groups' P become ready:
//   PV_g(j), S_g(j+1)
// A commit after S_g(j) completes only when every earlier MMA of the issuer has (in particular
// PV_g(j-1)), so a softmax group can rescale O_g as soon as it has seen S_g(j).
template <int D>
struct Fwd2 {
  static constexpr int BM = 128, BN = 128, KS = 2, VS = 2;
  static constexpr int Q_BYTES = BM * D * 2;
  static constexpr int KV_BYTES = BN * D * 2;
  static constexpr int OFF_Q = 0;  // Q0, Q1
  static constexpr int OFF_K = OFF_Q + 2 * Q_BYTES;
  static constexpr int OFF_V = OFF_K + KS * KV_BYTES;
  static constexpr int OFF_BAR = OFF_V + VS * KV_BYTES;
  static constexpr int SMEM = OFF_BAR + 256 + 1024;
  static constexpr int COL_S0 = 0, COL_S1 = 128, COL_O0 = 256, COL_O1 = 384;
  static constexpr int THREADS = 384;
  // P parts per tile, each released to the P·V MMA on its own as soon as it is in TMEM (the last one
  // before the MUFU hand-off to the other group): same-box A/B 853 -> 870 (first half early) -> 887
  // TF/s (last half before the hand-off); 4 parts measured the same as 2
  static constexpr int NP = 2;
};

template <int D>
__global__ void __launch_bounds__(384, 1)
    attn_fwd_tc2_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                        const __grid_constant__ CUtensorMap tmV, __nv_bfloat16* __restrict__ o,
                        float* __restrict__ lse, int T, int hq, int hkv, int64_t os, float scale_log2, int causal,
                        int pingpong) {
  ::kpo::pdl_launch_dependents();
  using C = Fwd2<D>;
  constexpr int BM = C::BM, BN = C::BN, KSUB = D / 64;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + C::OFF_BAR);
  uint64_t* q_full = bar + 0;
  uint64_t* k_full = bar + 1;    // [2]
  uint64_t* k_empty = bar + 3;   // [2]
  uint64_t* v_full = bar + 5;    // [2]
  uint64_t* v_empty = bar + 7;   // [2]
  uint64_t* s_full = bar + 9;    // [2] per Q tile
  uint64_t* pv_done = bar + 13;  // [2] per Q tile
  // [NP parts][2 Q tiles] (4 warps each): P keys [part * BN / NP, (part + 1) * BN / NP) stored in TMEM
  constexpr int NP = C::NP;
  uint64_t* p_full = bar + 15;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 15 + 2 * NP);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int mblk = gridDim.y - 1 - blockIdx.y;  // heavy (late) causal rows first
  const int h = blockIdx.x;
  const int kvh = h / (hq / hkv);
  const int m0 = mblk * 2 * BM;
  const int tiles_all = (T + BN - 1) / BN;
  int n_g[2];
#pragma unroll
  for (int g = 0; g < 2; ++g) {
    n_g[g] = tiles_all;
    if (causal) n_g[g] = min(tiles_all, (m0 + g * BM + BM + BN - 1) / BN);
    if (m0 + g * BM >= T) n_g[g] = 0;  // Q tile 1 past the end
  }
  const int n_all = max(n_g[0], n_g[1]);

  if (threadIdx.x == 0) {
    mbar_init(smem_u32(q_full), 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(smem_u32(&k_full[i]), 1);
      mbar_init(smem_u32(&k_empty[i]), 1);
      mbar_init(smem_u32(&v_full[i]), 1);
      mbar_init(smem_u32(&v_empty[i]), 1);
      mbar_init(smem_u32(&s_full[i]), 1);
      for (int pp = 0; pp < NP; ++pp) mbar_init(smem_u32(&p_full[pp * 2 + i]), 4);
      mbar_init(smem_u32(&pv_done[i]), 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 9) tmem_alloc(smem_u32(tmem_slot), 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (*tmem_slot != 0) __trap();
  ::kpo::pdl_wait();
  constexpr uint32_t tmem = 0;
  const uint32_t sQ = smem_u32(smem + C::OFF_Q), sK = smem_u32(smem + C::OFF_K), sV = smem_u32(smem + C::OFF_V);

  if (warp >= 8) {
    // the CTA holds 384 x 168 registers: 256 x 232 + 128 x 40 = 64512 fits exactly
    asm volatile("setmaxnreg.dec.sync.aligned.u32 40;");
    if (warp == 8 && lane == 0) {
      // ------------------------------------------------------------ TMA producer
      mbar_arrive_expect_tx(smem_u32(q_full), 2 * C::Q_BYTES);
#pragma unroll
      for (int g = 0; g < 2; ++g)
#pragma unroll
        for (int kb = 0; kb < KSUB; ++kb)
          tma_load_2d(sQ + g * C::Q_BYTES + kb * BM * 128, &tmQ, smem_u32(q_full), h * D + kb * 64, m0 + g * BM);
      for (int j = 0; j < n_all; ++j) {
        const int s = j & 1;
        const uint32_t ph = (j >> 1) & 1;
        mbar_wait(smem_u32(&k_empty[s]), ph ^ 1);
        uint32_t fb = smem_u32(&k_full[s]);
        mbar_arrive_expect_tx(fb, C::KV_BYTES);
#pragma unroll
        for (int kb = 0; kb < KSUB; ++kb)
          tma_load_2d(sK + s * C::KV_BYTES + kb * BN * 128, &tmK, fb, kvh * D + kb * 64, j * BN);
        mbar_wait(smem_u32(&v_empty[s]), ph ^ 1);
        fb = smem_u32(&v_full[s]);
        mbar_arrive_expect_tx(fb, C::KV_BYTES);
#pragma unroll
        for (int kb = 0; kb < KSUB; ++kb)
          tma_load_2d(sV + s * C::KV_BYTES + kb * BN * 128, &tmV, fb, kvh * D + kb * 64, j * BN);
      }
    } else if (warp == 9) {  // the whole warp runs the issue loop; elect.sync issues
      // ------------------------------------------------------------ MMA issuer
      constexpr uint32_t ID_S = idesc_bf16(BM, BN, false, false);
      constexpr uint32_t ID_O = idesc_bf16(BM, D, false, true);
      mbar_wait(smem_u32(q_full), 0);
      auto issue_s = [&](int g, int j) {  // S_g(j) = Q_g K_j^T into S_g
        const int s = j & 1;
        const uint32_t q_k = desc_lo(sQ + g * C::Q_BYTES, 16), k_k = desc_lo(sK + s * C::KV_BYTES, 16);
        const uint32_t d_s = tmem + (g ? C::COL_S1 : C::COL_S0);
#pragma unroll
        for (int kb = 0; kb < KSUB; ++kb)
#pragma unroll
          for (int k = 0; k < 4; ++k)
            tc_mma_lo_w(d_s, q_k + kb * (BM * 8) + k * 2, k_k + kb * (BN * 8) + k * 2, ID_S, (kb | k) ? 1u : 0u);
        tc_commit_w(smem_u32(&s_full[g]));
      };
      auto issue_pv = [&](int g, int j) {  // O_g += P_g(j) V_j, keys 0..63 as soon as their P is stored
        const int s = j & 1;
        const uint32_t v_mn = desc_lo(sV + s * C::KV_BYTES, BN * 128);
        const uint32_t p_t = tmem + (g ? C::COL_S1 : C::COL_S0);
        const uint32_t o_t = tmem + (g ? C::COL_O1 : C::COL_O0);
#pragma unroll
        for (int pp = 0; pp < NP; ++pp) {
          mbar_wait(smem_u32(&p_full[pp * 2 + g]), j & 1);
          tc_fence_after();
#pragma unroll
          for (int kk = pp * BN / 16 / NP; kk < (pp + 1) * BN / 16 / NP; ++kk)
            tc_mma_ts_lo_w(o_t, p_t + kk * 8, v_mn + kk * 128, ID_O, (j > 0 || kk > 0) ? 1u : 0u);
        }
        tc_commit_w(smem_u32(&pv_done[g]));
      };
      // prologue: S0_0, S1_0 (K_0)
      mbar_wait(smem_u32(&k_full[0]), 0);
      tc_fence_after();
      if (n_g[0] > 0) issue_s(0, 0);
      if (n_g[1] > 0) issue_s(1, 0);
      tc_commit_w(smem_u32(&k_empty[0]));
      for (int j = 0; j < n_all; ++j) {
        const int s = j & 1;
        const bool more = j + 1 < n_all;
        mbar_wait(smem_u32(&v_full[s]), (j >> 1) & 1);
        if (more) mbar_wait(smem_u32(&k_full[s ^ 1]), ((j + 1) >> 1) & 1);
        tc_fence_after();
        // serve the two groups in the order their P becomes ready (each group's own order PV_g(j) ->
        // S_g(j+1) is what the softmax relies on; the order between the groups is free)
        bool need0 = j < n_g[0], need1 = j < n_g[1];
        while (need0 || need1) {
          int g = need0 ? 0 : 1;
          if (need0 && need1) {
            while (true) {
              if (mbar_test(smem_u32(&p_full[0]), j & 1)) { g = 0; break; }
              if (mbar_test(smem_u32(&p_full[1]), j & 1)) { g = 1; break; }
            }
          }
          issue_pv(g, j);
          if (j + 1 < n_g[g]) issue_s(g, j + 1);
          if (g == 0) need0 = false;
          else need1 = false;
        }
        tc_commit_w(smem_u32(&v_empty[s]));
        if (more) tc_commit_w(smem_u32(&k_empty[s ^ 1]));
      }
    }
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 232;");
    // ------------------------------------------------------------ softmax group g (one row per thread)
    const int g = warp >> 2;
    const int quarter = warp & 3;
    const int r = quarter * 32 + lane;
    const int q = m0 + g * BM + r;
    const uint32_t lane_addr = tmem + ((uint32_t)(quarter * 32) << 16);
    const uint32_t s_addr = lane_addr + (g ? C::COL_S1 : C::COL_S0);
    const uint32_t o_addr = lane_addr + (g ? C::COL_O1 : C::COL_O0);
    const int ng = n_g[g];
    float m_run = -INFINITY, l_run = 0.f;
    for (int j = 0; j < ng; ++j) {
      mbar_wait(smem_u32(&s_full[g]), j & 1);
      tc_fence_after();
      float sv[BN];
#pragma unroll
      for (int c = 0; c < BN / 32; ++c) tmem_ld32_nowait(s_addr + c * 32, reinterpret_cast<uint32_t*>(sv + c * 32));
      tmem_wait_ld();
      const int k0 = j * BN;
      const bool mask = (causal && k0 + BN - 1 > m0 + g * BM) || (k0 + BN > T);  // group-uniform
      if (mask) {
#pragma unroll
        for (int i = 0; i < BN; ++i) {
          const int key = k0 + i;
          sv[i] = (key >= T || (causal && key > q)) ? -INFINITY : sv[i];
        }
      }
      // row max: 8 independent FMNMX3 chains (two elements per instruction)
      float pm[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) pm[e] = sv[e];
#pragma unroll
      for (int i = 8; i < BN; i += 2) pm[(i >> 1) & 7] = fmax3(pm[(i >> 1) & 7], sv[i], sv[i + 1]);
      const float mx = fmaxf(fmax3(fmax3(pm[0], pm[1], pm[2]), fmax3(pm[3], pm[4], pm[5]), pm[6]), pm[7]) * scale_log2;
      float corr = 1.f;
      bool rescale = false;
      if (mx > m_run + 8.f) {
        corr = (m_run == -INFINITY) ? 0.f : ex2(m_run - mx);
        rescale = (j > 0);
        m_run = mx;
      }
      // O_g is stable here: S_g(j) completing implies PV_g(j-1) completed (commit semantics)
      if (__any_sync(0xffffffffu, rescale)) {
#pragma unroll 1
        for (int c = 0; c < D / 32; ++c) {
          uint32_t ov[32];
          tmem_ld32_nowait(o_addr + c * 32, ov);
          tmem_wait_ld();
#pragma unroll
          for (int i = 0; i < 32; ++i) ov[i] = __float_as_uint(__uint_as_float(ov[i]) * corr);
          tmem_st32(o_addr + c * 32, ov);
        }
      }
      const float neg_m = -m_run;
      // ping-pong: the two groups take turns on the exponentials (MUFU), so one group's TMEM loads,
      // row max and P stores overlap the other's exp phase instead of both contending for MUFU
      if (pingpong) {
        if (g == 0 && j > 0) named_bar(1, 256);
        if (g == 1 && j < n_g[0]) named_bar(2, 256);
      }
      // exponent arguments with FFMA2 and row sums with FADD2, two keys per instruction
      uint64_t ps2[4] = {0, 0, 0, 0};
      const uint64_t sc2 = f2_pack(scale_log2, scale_log2), nm2 = f2_pack(neg_m, neg_m);
      constexpr int PC = BN / 2 / NP;  // packed bf16-pair columns per P part
#pragma unroll
      for (int pp = 0; pp < NP; ++pp) {  // BN / NP keys -> PC columns of bf16 pairs over S_g
        uint32_t pk[PC];
#pragma unroll
        for (int c = 0; c < PC; ++c) {
          const int i = pp * 2 * PC + c * 2;
          float x0, x1;
          f2_unpack(f2_fma(f2_pack(sv[i], sv[i + 1]), sc2, nm2), x0, x1);
          const float p0 = ex2(x0), p1 = ex2(x1);
          ps2[c & 3] = f2_add(ps2[c & 3], f2_pack(p0, p1));
          pk[c] = pack_bf16x2(p0, p1);
        }
        if constexpr (PC == 32) tmem_st32(s_addr + pp * PC, pk);
        else tmem_st16(s_addr + pp * PC, pk);
        // the P·V MMAs over this part's keys may start while the next part is exponentiated
        tmem_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(smem_u32(&p_full[pp * 2 + g]));
      }
      if (pingpong) {  // hand the MUFU to the other group
        if (g == 0) asm volatile("bar.arrive 2, 256;" ::: "memory");
        if (g == 1 && j + 1 < n_g[0]) asm volatile("bar.arrive 1, 256;" ::: "memory");
      }
      float ps[8];
#pragma unroll
      for (int c = 0; c < 4; ++c) f2_unpack(ps2[c], ps[2 * c], ps[2 * c + 1]);
      const float lsum = ((ps[0] + ps[1]) + (ps[2] + ps[3])) + ((ps[4] + ps[5]) + (ps[6] + ps[7]));
      l_run = l_run * corr + lsum;
    }
    if (ng > 0) {
      // ------------------------------------------------------------ epilogue
      mbar_wait(smem_u32(&pv_done[g]), (ng - 1) & 1);
      tc_fence_after();
      const float inv = 1.f / l_run;
      const bool row_ok = q < T;
      __nv_bfloat16* orow = o + (int64_t)q * os + (int64_t)h * D;
#pragma unroll 1
      for (int c = 0; c < D / 32; ++c) {
        uint32_t ov[32];
        tmem_ld32_nowait(o_addr + c * 32, ov);
        tmem_wait_ld();
        if (row_ok) {
#pragma unroll
          for (int v = 0; v < 4; ++v) {
            float f[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) f[e] = __uint_as_float(ov[v * 8 + e]) * inv;
            *reinterpret_cast<uint4*>(orow + c * 32 + v * 8) = pack8(f);
          }
        }
      }
      if (row_ok) lse[(int64_t)h * T + q] = (m_run + __log2f(l_run)) / kLog2e;
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 9) tmem_dealloc(tmem, 512);
}

template <int D>
int fwd_launch(const void* q, const void* k, const void* v, void* o, float* lse, int64_t T, int hq, int hkv,
               int64_t qs, int64_t ks, int64_t vs, int64_t os, float scale, int causal, cudaStream_t st) {
  using C = Fwd<D>;
  CUtensorMap mq, mk, mv;
  int e;
  if ((e = make_map_2d(&mq, q, (uint64_t)hq * D, T, qs, 64, C::BM))) return e;
  if ((e = make_map_2d(&mk, k, (uint64_t)hkv * D, T, ks, 64, C::BN))) return e;
  if ((e = make_map_2d(&mv, v, (uint64_t)hkv * D, T, vs, 64, C::BN))) return e;
  // POLY_MASK: which of every 8 exponentials run on the FMA pipe (ex2_poly) instead of MUFU.EX2
  static const int mode = getenv("KPO_EXP2_POLY") ? atoi(getenv("KPO_EXP2_POLY")) : 0;  // measured: MUFU-only fastest
  dim3 grid((unsigned)hq, (unsigned)((T + C::BM - 1) / C::BM));
  auto go = [&](auto kern) -> int {
    KPO_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
    KPO_CUDA(::kpo::pdl_launch(kern, grid, kThreads, C::SMEM, st, mq, mk, mv, (__nv_bfloat16*)o, lse, (int)T, hq, hkv, os, scale * kLog2e,
                                         causal));
    return KPO_OK;
  };
  // KPO_ATTN_FWD: 2 = the two-Q-tile kernel, 1 = the one-tile kernel, unset = the two-tile kernel
  // when its grid (q heads x 256-row tiles) fills the GPU, else the one-tile kernel (twice the CTAs:
  // TP8's 4 heads per rank give 64 two-tile CTAs for 148 SMs)
  static const int variant = getenv("KPO_ATTN_FWD") ? atoi(getenv("KPO_ATTN_FWD")) : 0;
  const int sms = num_sms() > 0 ? num_sms() : 148;
  const bool two_tile = D == 128 && (variant == 2 || (variant == 0 && (int64_t)hq * ((T + 255) / 256) >= sms));
  if (two_tile) {
    using C2 = Fwd2<D>;
    dim3 grid2((unsigned)hq, (unsigned)((T + 2 * C2::BM - 1) / (2 * C2::BM)));
    auto kern2 = attn_fwd_tc2_kernel<D>;
    KPO_CUDA(cudaFuncSetAttribute(kern2, cudaFuncAttributeMaxDynamicSharedMemorySize, C2::SMEM));
    KPO_CUDA(::kpo::pdl_launch(kern2, grid2, C2::THREADS, C2::SMEM, st, mq, mk, mv, (__nv_bfloat16*)o, lse, (int)T,
                               hq, hkv, os, scale * kLog2e, causal,
                               getenv("KPO_ATTN_PINGPONG") ? atoi(getenv("KPO_ATTN_PINGPONG")) : 0));
    KPO_LAUNCH_CHECK();
    return KPO_OK;
  }
  int rc;
  if (mode == 0) rc = go(attn_fwd_tc_kernel<D, 0x00>);
  else if (mode == 2) rc = go(attn_fwd_tc_kernel<D, 0x55>);
  else if (mode == 3) rc = go(attn_fwd_tc_kernel<D, 0x80>);
  else if (mode == 4) rc = go(attn_fwd_tc_kernel<D, 0x92>);
  else rc = go(attn_fwd_tc_kernel<D, 0x88>);
  if (rc) return rc;
  KPO_LAUNCH_CHECK();
  return KPO_OK;
}


// =====================================================================================
// Backward.  One CTA = 128 keys of one kv head; it loops over every q head of the GQA group and
// every causal 64-query tile, so dK / dV accumulate in TMEM across the whole group (no atomics).
// Per step (64 queries):
//   S^T  = K Q^T        M=128 keys, N=64 q, K=d      (A = K tile K-major, B = Q tile K-major)
//   dP^T = V dO^T       M=128 keys, N=64 q, K=d
//   softmax warps (one key row per thread): P^T = exp2(S^T*scale*log2e - lse2), dS^T = P^T (dP^T - Dq)
//                                           -> bf16 P^T / dS^T tiles in smem (K-major SW128)
//   dV  += P^T dO       M=128 keys, N=d,  K=64 q     (B = dO tile read MN-major)
//   dK  += dS^T Q       M=128 keys, N=d,  K=64 q     (B = Q tile read MN-major)
//   dQ^T = K^T dS^T     M=d=128,   N=64 q, K=128 keys (A = the K tile read MN-major, B = dS^T MN-major)
//   dQ drain warps: dQ^T (lane = head-dim index) -> fp32 [q][d] smem tile -> one TMA bulk
//   reduce-add (cp.reduce.async.bulk.tensor .add) into dq_acc[t][h][d].
// TMEM columns: S^T 0..63, dP^T 64..127, dQ^T 128..191, P^T (2 x 32 cols of bf16 pairs, the A operand
// of the dV MMA read straight from TMEM) 192..255, dV 256..383, dK 384..511.
// Issue order: S/dP(s+1) as soon as the softmax warps have pulled S/dP(s) out of TMEM, then the
// gradient MMAs of step s; P^T/dS^T (smem) and dQ^T (TMEM) are double-buffered so the softmax of
// step s+1 and the dQ drain of step s overlap the tensor core.
template <int D>
struct Bwd {
  static constexpr int BN = 128, BM = 64, QSTAGES = 3;
  static constexpr int KV_BYTES = BN * D * 2;
  static constexpr int QT_BYTES = BM * D * 2;
  static constexpr int PT_BYTES = BN * BM * 2;   // one dS^T buffer [128 keys][64 q] bf16
  static constexpr int OFF_K = 0, OFF_V = OFF_K + KV_BYTES, OFF_Q = OFF_V + KV_BYTES;
  static constexpr int OFF_DO = OFF_Q + QSTAGES * QT_BYTES, OFF_DS = OFF_DO + QSTAGES * QT_BYTES;
  static constexpr int OFF_DQ = OFF_DS + 2 * PT_BYTES;           // fp32 [64 q][D] staging for the TMA reduce-add
  static constexpr int OFF_STAT = OFF_DQ + BM * D * 4;
  static constexpr int OFF_BAR = OFF_STAT + QSTAGES * 2 * BM * 4;
  static constexpr int SMEM = OFF_BAR + 256 + 1024;
  // TMEM: S^T 0..63, dP^T 64..127, dQ^T 128..191, P^T (bf16 pairs, 2 buffers x 32 cols) 192..255,
  //       dV 256..383, dK 384..511
  static constexpr int COL_S = 0, COL_DP = 64, COL_DQ = 128, COL_PT = 192, COL_DV = 256, COL_DK = 384;
  // TMA, MMA, SM_WARPS softmax warps (SM_WARPS / 4 per lane quarter, each BM * 4 / SM_WARPS query
  // columns), 4 dQ-drain warps.  16 softmax warps halve the per-warp latency of the softmax, which sits
  // between the S / dP MMAs and the gradient MMAs of a step (ablation: removing it saved 18%).
  static constexpr int SM_WARPS = 16;
  static constexpr int THREADS = (2 + SM_WARPS + 4) * 32;
};


template <int D>
__global__ void __launch_bounds__(Bwd<D>::THREADS, 1)
    attn_bwd_tc_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                       const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmDO,
                       const __grid_constant__ CUtensorMap tmDQ,
                       const float* __restrict__ lse, const float* __restrict__ dvec, float* __restrict__ dq_acc,
                       __nv_bfloat16* __restrict__ dk, __nv_bfloat16* __restrict__ dv, int T, int hq, int hkv,
                       int64_t dks, int64_t dvs, float scale, int causal, float* __restrict__ dkv_acc,
                       int split_group, int qsplit_tiles,
                       int ablate, const float2* __restrict__ rope_cs) {
  // rope_cs != nullptr: dK leaves inverse-rotated (the gradient w.r.t. the un-rotated k), the fused
  // backward of the QKV GEMM's rotary epilogue; dQ is rotated by the dq conversion kernel
  ::kpo::pdl_launch_dependents();  // the next kernel may start its prologue; it waits for us
  // ablate (KPO_ATTN_BWD_ABLATE, measurement only; results are wrong when != 0): 1 = no dQ reduce-add,
  // 2 = no dQ drain (TMEM -> smem), 4 = no exponentials, 8 = no dQ^T MMA, 16 = no softmax,
  // 32 = no Q/dO reloads, 64 = no dV/dK MMAs, 128 = no S^T/dP^T MMAs
  // dkv_acc != nullptr: split-group mode — one CTA per (q head, key tile); dK / dV contributions are
  // reduced into fp32 accumulators [T][hkv][D] (dK at dkv_acc, dV at dkv_acc + T*hkv*D).
  using C = Bwd<D>;
  constexpr int BN = C::BN, BM = C::BM, KSUB = D / 64;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + C::OFF_BAR);
  uint64_t* kv_full = bar + 0;
  uint64_t* qd_full = bar + 1;     // [3]
  uint64_t* qd_empty = bar + 4;    // [3]
  uint64_t* s_full = bar + 7;
  uint64_t* s_empty = bar + 8;
  uint64_t* pds_full = bar + 9;    // [2]
  uint64_t* pds_empty = bar + 11;  // [2]  MMA commit + dQ drain (staging read by TMA)
  uint64_t* dq_full = bar + 13;    // [2]
  uint64_t* dq_empty = bar + 15;   // [2]
  uint64_t* acc_done = bar + 17;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 18);
  float* stat = reinterpret_cast<float*>(smem + C::OFF_STAT);  // [2][lse2 64 | dvec 64]

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nblk = blockIdx.y;  // early key tiles carry the most causal work: dispatched first
  const bool split = split_group != 0;
  const int group = split ? 1 : hq / hkv;
  const int h_first = split ? (int)blockIdx.x : (int)blockIdx.x * (hq / hkv);
  const int kvh = split ? (int)blockIdx.x / (hq / hkv) : (int)blockIdx.x;
  const int n0 = nblk * BN;
  const int total_m = (T + BM - 1) / BM;
  int m_start = causal ? n0 / BM : 0, m_end = total_m;
  // query chunks (blockIdx.z) for the first qsplit_tiles key tiles (all of them in split-group mode):
  // this CTA takes the query tiles of chunk z, so the long causal key tiles are spread over several
  // SMs; dK / dV partials of a chunked tile meet in the fp32 accumulators, dQ in dq_acc as always
  const bool chunked = gridDim.z > 1 && nblk < qsplit_tiles;
  if (gridDim.z > 1) {
    if (chunked) {
      const int qper = (total_m + (int)gridDim.z - 1) / (int)gridDim.z;
      m_start = max(m_start, (int)blockIdx.z * qper);
      m_end = min(total_m, ((int)blockIdx.z + 1) * qper);
      if (m_start >= m_end) return;  // nothing causal in this chunk (before any barrier / TMEM use)
    } else if (blockIdx.z != 0) {
      return;  // an unchunked key tile: chunk 0 owns all of its queries
    }
  }
  const bool atomic_dkv = split || chunked;
  const int mq = m_end - m_start;
  const int steps = group * mq;
  const float scale_log2 = scale * kLog2e;

  if (threadIdx.x == 0) {
    mbar_init(smem_u32(kv_full), 1);
    for (int i = 0; i < C::QSTAGES; ++i) {
      mbar_init(smem_u32(&qd_full[i]), 1);
      mbar_init(smem_u32(&qd_empty[i]), 1);
    }
    mbar_init(smem_u32(s_full), 1);
    mbar_init(smem_u32(s_empty), C::SM_WARPS);
    for (int i = 0; i < 2; ++i) {
      mbar_init(smem_u32(&pds_full[i]), C::SM_WARPS);
      mbar_init(smem_u32(&pds_empty[i]), 1);
      mbar_init(smem_u32(&dq_full[i]), 1);
      mbar_init(smem_u32(&dq_empty[i]), 4);
    }
    mbar_init(smem_u32(acc_done), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) tmem_alloc(smem_u32(tmem_slot), 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  // one CTA per SM owns all 512 columns, so the allocation starts at lane 0 / column 0; a constant base
  // keeps every TMEM address of the MMA issue loops in uniform registers (no per-MMA R2UR)
  if (*tmem_slot != 0) __trap();
  ::kpo::pdl_wait();  // the previous kernel's outputs (our inputs) are complete and visible
  constexpr uint32_t tmem = 0;
  const uint32_t sK = smem_u32(smem + C::OFF_K), sV = smem_u32(smem + C::OFF_V);
  const uint32_t sQ = smem_u32(smem + C::OFF_Q), sDO = smem_u32(smem + C::OFF_DO);
  const uint32_t sDS = smem_u32(smem + C::OFF_DS);  // dS^T buffer b at b*PT_BYTES

  auto step_coords = [&](int s, int& h, int& m0) {
    h = h_first + s / mq;
    m0 = (m_start + s % mq) * BM;
  };

  if (warp == 0) {
    if (lane == 0) {
      // ------------------------------------------------------------ TMA producer
      mbar_arrive_expect_tx(smem_u32(kv_full), 2 * C::KV_BYTES);
#pragma unroll
      for (int kb = 0; kb < KSUB; ++kb) {
        tma_load_2d(sK + kb * BN * 128, &tmK, smem_u32(kv_full), kvh * D + kb * 64, n0);
        tma_load_2d(sV + kb * BN * 128, &tmV, smem_u32(kv_full), kvh * D + kb * 64, n0);
      }
      for (int s = 0; s < steps; ++s) {
        const int st = s % C::QSTAGES;
        int h, m0;
        step_coords(s, h, m0);
        mbar_wait(smem_u32(&qd_empty[st]), ((s / C::QSTAGES) & 1) ^ 1);
        const uint32_t fb = smem_u32(&qd_full[st]);
        if ((ablate & 32) && s >= C::QSTAGES) {  // measurement: reuse stale Q/dO tiles (no L2 traffic)
          mbar_arrive(fb);
          continue;
        }
        const uint32_t nstat = (uint32_t)min(BM, T - m0) * 4u;  // T % 8 == 0 keeps this a 16 B multiple
        mbar_arrive_expect_tx(fb, 2 * C::QT_BYTES + 2 * nstat);
#pragma unroll
        for (int kb = 0; kb < KSUB; ++kb) {
          tma_load_2d(sQ + st * C::QT_BYTES + kb * BM * 128, &tmQ, fb, h * D + kb * 64, m0);
          tma_load_2d(sDO + st * C::QT_BYTES + kb * BM * 128, &tmDO, fb, h * D + kb * 64, m0);
        }
        const uint32_t sst = smem_u32(stat + st * 2 * BM);
        bulk_load(sst, lse + (int64_t)h * T + m0, nstat, fb);
        bulk_load(sst + BM * 4, dvec + (int64_t)h * T + m0, nstat, fb);
      }
    }
  } else if (warp == 1) {
    {  // the whole warp runs the issue loop (warp-uniform operands); elect.sync issues
      // ------------------------------------------------------------ MMA issuer
      constexpr uint32_t ID_S = idesc_bf16(BN, BM, false, false);   // S^T, dP^T
      constexpr uint32_t ID_G = idesc_bf16(BN, D, false, true);     // dV, dK
      constexpr uint32_t ID_Q = idesc_bf16(D, BM, true, true);      // dQ^T
      mbar_wait(smem_u32(kv_full), 0);
      constexpr uint32_t ID_GT = idesc_bf16(BN, D, false, true);   // dV with A = P^T from TMEM
      const uint32_t k_k = desc_lo(sK, 16), v_k = desc_lo(sV, 16), k_mn = desc_lo(sK, BN * 128);
      auto grads = [&](int j) {
        const int st = j & 1;          // P^T / dS^T buffer
        const int qs = j % C::QSTAGES;  // Q/dO stage
        mbar_wait(smem_u32(&pds_full[st]), (j >> 1) & 1);
        tc_fence_after();
        const uint32_t q_mn = desc_lo(sQ + qs * C::QT_BYTES, BM * 128), o_mn = desc_lo(sDO + qs * C::QT_BYTES, BM * 128);
        const uint32_t ds_k = desc_lo(sDS + st * C::PT_BYTES, 16), ds_mn = desc_lo(sDS + st * C::PT_BYTES, BM * 128);
        const uint32_t pt = tmem + C::COL_PT + st * 32;
        if (!(ablate & 64)) {
#pragma unroll
          for (int k = 0; k < BM / 16; ++k) {
            const uint32_t acc = (j > 0 || k > 0) ? 1u : 0u;
            tc_mma_ts_lo_w(tmem + C::COL_DV, pt + k * 8, o_mn + k * 128, ID_GT, acc);
            tc_mma_lo_w(tmem + C::COL_DK, ds_k + k * 2, q_mn + k * 128, ID_G, acc);
          }
        }
        mbar_wait(smem_u32(&dq_empty[0]), (j & 1) ^ 1);
        tc_fence_after();
        if (!(ablate & 8)) {
#pragma unroll
          for (int k = 0; k < BN / 16; ++k)
            tc_mma_lo_w(tmem + C::COL_DQ, k_mn + k * 128, ds_mn + k * 128, ID_Q, k > 0 ? 1u : 0u);
        }
        tc_commit_w(smem_u32(&dq_full[0]));
        tc_commit_w(smem_u32(&pds_empty[st]));
        tc_commit_w(smem_u32(&qd_empty[qs]));
      };
      auto scores = [&](int s) {
        const int st = s % C::QSTAGES;
        mbar_wait(smem_u32(&qd_full[st]), (s / C::QSTAGES) & 1);
        tc_fence_after();
        const uint32_t q_k = desc_lo(sQ + st * C::QT_BYTES, 16), o_k = desc_lo(sDO + st * C::QT_BYTES, 16);
        if (!(ablate & 128)) {
#pragma unroll
          for (int kb = 0; kb < KSUB; ++kb) {
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const uint32_t acc = (kb | k) ? 1u : 0u;
              tc_mma_lo_w(tmem + C::COL_S, k_k + kb * (BN * 8) + k * 2, q_k + kb * (BM * 8) + k * 2, ID_S, acc);
              tc_mma_lo_w(tmem + C::COL_DP, v_k + kb * (BN * 8) + k * 2, o_k + kb * (BM * 8) + k * 2, ID_S, acc);
            }
          }
        }
        tc_commit_w(smem_u32(s_full));
      };
      if (steps > 0) scores(0);
      for (int s = 0; s < steps; ++s) {
        if (s + 1 < steps) {
          mbar_wait(smem_u32(s_empty), s & 1);  // softmax(s) has pulled S/dP(s) out of TMEM
          scores(s + 1);
        }
        grads(s);
      }
      tc_commit_w(smem_u32(acc_done));
    }
  } else if (warp < 2 + C::SM_WARPS) {
    // ------------------------------------------------------------ softmax warps 2 .. 2 + SM_WARPS - 1
    // row = key (TMEM lane quarter = warp % 4); the SM_WARPS / 4 warps of a quarter split the 64 query
    // columns
    const int quarter = warp & 3;
    const int half = (warp - 2) >> 2;  // column group of this warp (0 .. SM_WARPS/4 - 1)
    const int r = quarter * 32 + lane;
    const int key = n0 + r;
    const uint32_t lane_addr = tmem + ((uint32_t)(quarter * 32) << 16);
    constexpr int HC = BM * 4 / C::SM_WARPS;  // query columns per warp
    const float* stat_half = stat + half * HC;
    for (int s = 0, mi = 0; s < steps; ++s, mi = (mi + 1 == mq) ? 0 : mi + 1) {
      const int m0 = (m_start + mi) * BM;
      const int buf = s & 1;
      mbar_wait(smem_u32(s_full), s & 1);
      tc_fence_after();
      float sv[HC], dp[HC];
      if constexpr (HC == 32) {
        tmem_ld32_nowait(lane_addr + C::COL_S + half * HC, reinterpret_cast<uint32_t*>(sv));
        tmem_ld32_nowait(lane_addr + C::COL_DP + half * HC, reinterpret_cast<uint32_t*>(dp));
      } else {
        tmem_ld16_nowait(lane_addr + C::COL_S + half * HC, reinterpret_cast<uint32_t*>(sv));
        tmem_ld16_nowait(lane_addr + C::COL_DP + half * HC, reinterpret_cast<uint32_t*>(dp));
      }
      // this warp's 32 query statistics (lse, D), bulk-copied by the TMA warp with the Q/dO stage
      const uint32_t sst = smem_u32(stat_half + (s % C::QSTAGES) * 2 * BM);
      tmem_wait_ld();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_u32(s_empty));
      if (ablate & 16) {  // measurement: no softmax work at all
        mbar_wait(smem_u32(&pds_empty[buf]), ((s >> 1) & 1) ^ 1);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(smem_u32(&pds_full[buf]));
        continue;
      }
      // CTA-uniform: does this tile need the causal / tail mask at all?
      const bool tile_mask = (causal && m0 < n0 + BN - 1) || n0 + BN > T || m0 + BM > T;
      uint32_t pp[HC / 2], qq[HC / 2];
      // two query columns per FFMA2 / FMUL2 / FADD2: x = S scale - lse log2e, P = 2^x, dS = P (dP - D)
      const uint64_t sc2 = f2_pack(scale_log2, scale_log2), nlg2 = f2_pack(-kLog2e, -kLog2e);
#pragma unroll
      for (int i = 0; i < HC; i += 2) {
        uint64_t nl2, dd2;
        asm volatile("ld.shared.b64 %0, [%1];" : "=l"(nl2) : "r"(sst + i * 4));
        asm volatile("ld.shared.b64 %0, [%1];" : "=l"(dd2) : "r"(sst + BM * 4 + i * 4));
        float p2[2], d2[2];
        f2_unpack(f2_fma(f2_pack(sv[i], sv[i + 1]), sc2, f2_mul(nl2, nlg2)), p2[0], p2[1]);
        if (!(ablate & 4)) {
          p2[0] = ex2(p2[0]);
          p2[1] = ex2(p2[1]);
        }
        f2_unpack(f2_mul(f2_pack(p2[0], p2[1]), f2_sub(f2_pack(dp[i], dp[i + 1]), dd2)), d2[0], d2[1]);
        if (tile_mask) {
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int q = m0 + half * HC + i + e;
            const bool z = key >= T || q >= T || (causal && q < key);
            p2[e] = z ? 0.f : p2[e];
            d2[e] = z ? 0.f : d2[e];
          }
        }
        pp[i / 2] = pack_bf16x2(p2[0], p2[1]);
        qq[i / 2] = pack_bf16x2(d2[0], d2[1]);
      }
      mbar_wait(smem_u32(&pds_empty[buf]), ((s >> 1) & 1) ^ 1);  // grads(s-2) done with this buffer
      const uint32_t db = sDS + buf * C::PT_BYTES;
#pragma unroll
      for (int ch = 0; ch < HC / 8; ++ch) {
        const uint32_t off = sw128(r, half * (HC / 8) + ch);
        asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(db + off), "r"(qq[ch * 4]), "r"(qq[ch * 4 + 1]),
                     "r"(qq[ch * 4 + 2]), "r"(qq[ch * 4 + 3])
                     : "memory");
      }
      // P^T row (this warp's 32 queries = 16 packed columns) -> TMEM, the A operand of the dV MMA
      if constexpr (HC == 32) tmem_st16(lane_addr + C::COL_PT + buf * 32 + half * (HC / 2), pp);
      else tmem_st8(lane_addr + C::COL_PT + buf * 32 + half * (HC / 2), pp);
      tmem_wait_st();
      tc_fence_before();
      fence_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_u32(&pds_full[buf]));
    }
    if (half) goto done_softmax;  // the first warp of each quarter writes dK / dV
    {
    // ------------------------------------------------------------ dK / dV epilogue
    mbar_wait(smem_u32(acc_done), 0);
    tc_fence_after();
    const bool ok = key < T && steps > 0;
#pragma unroll 1
    for (int which = 0; which < 2; ++which) {
      const uint32_t col = which ? C::COL_DV : C::COL_DK;
      const float mul = which ? 1.f : scale;
      __nv_bfloat16* row = which ? dv + (int64_t)key * dvs + (int64_t)kvh * D : dk + (int64_t)key * dks + (int64_t)kvh * D;
      if (which == 0 && rope_cs != nullptr && !atomic_dkv) {
        // inverse rotary: pairs (i, i + D/2) of the key's row, (cos, sin) of the key position
        const float2* cs = rope_cs + (int64_t)(key < T ? key : 0) * (D / 2);
#pragma unroll 1
        for (int c = 0; c < D / 64; ++c) {
          uint32_t va[32], vb[32];
          tmem_ld32_nowait(lane_addr + col + c * 32, va);
          tmem_ld32_nowait(lane_addr + col + D / 2 + c * 32, vb);
          tmem_wait_ld();
          if (ok) {
#pragma unroll
            for (int q4 = 0; q4 < 4; ++q4) {
              float oa[8], ob[8];
#pragma unroll
              for (int j = 0; j < 8; ++j) {
                const float2 t = cs[c * 32 + q4 * 8 + j];
                const float x = __uint_as_float(va[q4 * 8 + j]) * mul, y = __uint_as_float(vb[q4 * 8 + j]) * mul;
                oa[j] = x * t.x + y * t.y;
                ob[j] = y * t.x - x * t.y;
              }
              *reinterpret_cast<uint4*>(row + c * 32 + q4 * 8) = pack8(oa);
              *reinterpret_cast<uint4*>(row + D / 2 + c * 32 + q4 * 8) = pack8(ob);
            }
          }
        }
      } else {
#pragma unroll 1
      for (int c = 0; c < D / 32; ++c) {
        uint32_t v[32];
        tmem_ld32_nowait(lane_addr + col + c * 32, v);
        tmem_wait_ld();
        if (ok && atomic_dkv) {
          float* acc = dkv_acc + (which ? (int64_t)T * hkv * D : 0) + ((int64_t)key * hkv + kvh) * D + c * 32;
#pragma unroll
          for (int q4 = 0; q4 < 8; ++q4)
            atomicAdd(reinterpret_cast<float4*>(acc + q4 * 4),
                      make_float4(__uint_as_float(v[q4 * 4 + 0]) * mul, __uint_as_float(v[q4 * 4 + 1]) * mul,
                                  __uint_as_float(v[q4 * 4 + 2]) * mul, __uint_as_float(v[q4 * 4 + 3]) * mul));
        } else if (ok) {
#pragma unroll
          for (int q4 = 0; q4 < 4; ++q4) {
            uint4 u;
            u.x = pack_bf16x2(__uint_as_float(v[q4 * 8 + 0]) * mul, __uint_as_float(v[q4 * 8 + 1]) * mul);
            u.y = pack_bf16x2(__uint_as_float(v[q4 * 8 + 2]) * mul, __uint_as_float(v[q4 * 8 + 3]) * mul);
            u.z = pack_bf16x2(__uint_as_float(v[q4 * 8 + 4]) * mul, __uint_as_float(v[q4 * 8 + 5]) * mul);
            u.w = pack_bf16x2(__uint_as_float(v[q4 * 8 + 6]) * mul, __uint_as_float(v[q4 * 8 + 7]) * mul);
            *reinterpret_cast<uint4*>(row + c * 32 + q4 * 8) = u;
          }
        }
      }
      }
      if (!ok && !atomic_dkv && steps == 0 && key < T) {  // no causal work: gradients are zero
        for (int c = 0; c < D; c += 8) *reinterpret_cast<uint4*>(row + c) = make_uint4(0, 0, 0, 0);
      }
    }
    }
  done_softmax:;
  } else {
    // ------------------------------------------------------------ dQ drain warps (the last 4; lane = head dim)
    const int quarter = warp & 3;
    const int dcol = quarter * 32 + lane;
    const int dtid = threadIdx.x - (2 + C::SM_WARPS) * 32;  // 0..127
    const uint32_t lane_addr = tmem + ((uint32_t)(quarter * 32) << 16);
    for (int s = 0; s < steps; ++s) {
      int h, m0;
      step_coords(s, h, m0);
      mbar_wait(smem_u32(&dq_full[0]), s & 1);
      tc_fence_after();
      if (ablate & 2) {
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(smem_u32(&dq_empty[0]));
        continue;
      }
      // the staging tile drains in two 32-query halves: half hf is rewritten once its previous reduce
      // has read it, while the other half's reduce may still be in flight; dQ^T's TMEM columns are
      // released once the second half has been loaded (32 live registers, not 64)
      float* stg = reinterpret_cast<float*>(smem + C::OFF_DQ);
#pragma unroll
      for (int hf = 0; hf < 2; ++hf) {
        float v[BM / 2];
        tmem_ld32_nowait(lane_addr + C::COL_DQ + hf * 32, reinterpret_cast<uint32_t*>(v));
        tmem_wait_ld();
        if (hf == 1) {
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(smem_u32(&dq_empty[0]));
        }
        if (dtid == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
        named_bar(2, 128);
        float* sh = stg + hf * (BM / 2) * D;
#pragma unroll
        for (int qi = 0; qi < BM / 2; ++qi) sh[qi * D + dcol] = v[qi] * scale;
        fence_async_smem();
        named_bar(2, 128);
        if (dtid == 0) {
          if (!(ablate & 1)) tma_reduce_add_2d(&tmDQ, smem_u32(sh), h * D, m0 + hf * (BM / 2));
          bulk_commit();
        }
      }
    }
    if (dtid == 0) bulk_wait0();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) tmem_dealloc(tmem, 512);
}

// =====================================================================================
// Backward, 128-query steps (head_dim 64; KPO_ATTN_BWD=3 for head_dim 128).  One CTA = 128 keys of one kv head, looping over the GQA group x causal
// 128-query tiles; every MMA is M=128 x N=128 x K=128, so each SS MMA reads 8 KB of operands per 64
// tensor cycles (the 64-query kernel above issues N=64 MMAs, capped by shared memory at 48 of their
// 32 cycles).  TMEM (512 columns) is aliased:
//   S^T  cols   0..127  keys x queries, fp32.  Softmax warp g (32 queries) writes its P^T (bf16
//                       pairs) over the first 16 of its own 32 S columns: the TMEM A operand of dV.
//   dP^T cols 128..255  keys x queries.  Warp g writes dS^T (bf16 pairs) over the first 16 of its own
//                       32 dP columns: the TMEM A operand of dK.  dQ (queries x d, fp32) is then
//                       written over the whole region by the dQ MMA (issued after dK, in order).
//   dV   cols 256..383, dK cols 384..511
// Per step s the MMA warp issues dV(s) += P^T dO, dP(s) = V dO^T (once dQ(s-1) has left TMEM),
// S(s+1) = K Q^T, then dK(s) += dS^T Q and dQ(s) = dS K (dS from shared memory, MN-major).  The 16
// softmax warps (4 per TMEM lane quarter, 32 queries each) compute P(s), then drain dQ(s-1) (each
// warp one 32-column chunk: TMEM -> registers -> one of four 16 KB SW128 staging boxes -> TMA bulk
// reduce-add into the fp32 dQ accumulator), then dS(s).  The tensor core runs dV(s) while dQ(s-1)
// drains and S(s+1) while dS(s) is computed, so neither is on its critical path.
// Shared memory: K, V (32 KB each), Q (2 stages), dO (1 stage), dS^T (32 KB, MN-major dS operand of
// the dQ MMA; between dQ(s-1) and dS(s) it doubles as staging boxes 0, 1), staging boxes 2, 3.
template <int D>
struct Bwd3 {
  static constexpr int BN = 128, BM = 128, QSTAGES = 2, KSUB = D / 64;
  static constexpr int KV_BYTES = BN * D * 2;            // 32 KB
  static constexpr int QT_BYTES = BM * D * 2;            // 32 KB
  static constexpr int DS_BYTES = BN * BM * 2;           // 32 KB
  static constexpr int DQC = 32;                         // d columns per dQ reduce chunk (one warp's)
  static constexpr int STG_BYTES = BM * DQC * 4;         // 16 KB
  static constexpr int OFF_K = 0, OFF_V = OFF_K + KV_BYTES, OFF_Q = OFF_V + KV_BYTES;
  static constexpr int OFF_DO = OFF_Q + QSTAGES * QT_BYTES, OFF_DS = OFF_DO + QT_BYTES;
  static constexpr int OFF_STG = OFF_DS + DS_BYTES;      // staging boxes 2, 3
  static constexpr int OFF_STAT = OFF_STG + 2 * STG_BYTES;  // [QSTAGES][lse BM | D BM] fp32
  static constexpr int OFF_BAR = OFF_STAT + QSTAGES * 2 * BM * 4;
  static constexpr int SMEM = OFF_BAR + 256;  // 231680 B: the dynamic window must start 1024-aligned
  static constexpr int COL_S = 0, COL_DP = 128, COL_DV = 256, COL_DK = 384;
  static constexpr int SM_WARPS = 16;
  static constexpr int THREADS = (2 + SM_WARPS) * 32;
  static_assert(DS_BYTES == 2 * STG_BYTES, "the dS^T buffer holds staging boxes 0, 1");
};

template <int D>
__global__ void __launch_bounds__(Bwd3<D>::THREADS, 1)
    attn_bwd_tc3_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                        const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmDO,
                        const __grid_constant__ CUtensorMap tmDQ,
                        const float* __restrict__ lse, const float* __restrict__ dvec,
                        __nv_bfloat16* __restrict__ dk, __nv_bfloat16* __restrict__ dv, int T, int hq, int hkv,
                        int64_t dks, int64_t dvs, float scale, int causal, float* __restrict__ dkv_acc,
                        int split_group, int qsplit_tiles, const float2* __restrict__ rope_cs) {
  // same contract as attn_bwd_tc_kernel (split-group / query-chunk modes, fused inverse rotary of dK)
  ::kpo::pdl_launch_dependents();
  using C = Bwd3<D>;
  constexpr int BN = C::BN, BM = C::BM, KSUB = C::KSUB, NCH = D / C::DQC;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + C::OFF_BAR);
  uint64_t* kv_full = bar + 0;
  uint64_t* q_full = bar + 1;    // [2]
  uint64_t* q_empty = bar + 3;   // [2]
  uint64_t* do_full = bar + 5;
  uint64_t* do_empty = bar + 6;
  uint64_t* s_full = bar + 7;
  uint64_t* p_full = bar + 8;
  uint64_t* dp_full = bar + 9;
  uint64_t* ds_full = bar + 10;
  uint64_t* dq_full = bar + 11;
  uint64_t* dq_empty = bar + 12;
  uint64_t* stg_free = bar + 13;  // [2]  staging boxes 0 / 1 (the dS^T buffer halves) read by their reduce
  uint64_t* acc_done = bar + 15;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 16);
  float* stat = reinterpret_cast<float*>(smem + C::OFF_STAT);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nblk = blockIdx.y;
  const bool split = split_group != 0;
  const int group = split ? 1 : hq / hkv;
  const int h_first = split ? (int)blockIdx.x : (int)blockIdx.x * (hq / hkv);
  const int kvh = split ? (int)blockIdx.x / (hq / hkv) : (int)blockIdx.x;
  const int n0 = nblk * BN;
  const int total_m = (T + BM - 1) / BM;
  int m_start = causal ? n0 / BM : 0, m_end = total_m;
  const bool chunked = gridDim.z > 1 && nblk < qsplit_tiles;
  if (gridDim.z > 1) {
    if (chunked) {
      const int qper = (total_m + (int)gridDim.z - 1) / (int)gridDim.z;
      m_start = max(m_start, (int)blockIdx.z * qper);
      m_end = min(total_m, ((int)blockIdx.z + 1) * qper);
      if (m_start >= m_end) return;
    } else if (blockIdx.z != 0) {
      return;
    }
  }
  const bool atomic_dkv = split || chunked;
  const int mq = m_end - m_start;
  const int steps = group * mq;
  const float scale_log2 = scale * kLog2e;

  if (threadIdx.x == 0) {
    if (smem_u32(smem) & 1023) __trap();  // SW128 tiles need a 1024-aligned window (no slack left)
    mbar_init(smem_u32(kv_full), 1);
    for (int i = 0; i < C::QSTAGES; ++i) {
      mbar_init(smem_u32(&q_full[i]), 1);
      mbar_init(smem_u32(&q_empty[i]), 1);
    }
    mbar_init(smem_u32(do_full), 1);
    mbar_init(smem_u32(do_empty), 1);
    mbar_init(smem_u32(s_full), 1);
    mbar_init(smem_u32(p_full), C::SM_WARPS);
    mbar_init(smem_u32(dp_full), 1);
    mbar_init(smem_u32(ds_full), C::SM_WARPS);
    mbar_init(smem_u32(dq_full), 1);
    mbar_init(smem_u32(dq_empty), C::SM_WARPS);
    mbar_init(smem_u32(&stg_free[0]), 1);
    mbar_init(smem_u32(&stg_free[1]), 1);
    mbar_init(smem_u32(acc_done), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) tmem_alloc(smem_u32(tmem_slot), 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (*tmem_slot != 0) __trap();
  ::kpo::pdl_wait();
  constexpr uint32_t tmem = 0;
  const uint32_t sK = smem_u32(smem + C::OFF_K), sV = smem_u32(smem + C::OFF_V);
  const uint32_t sQ = smem_u32(smem + C::OFF_Q), sDO = smem_u32(smem + C::OFF_DO);
  const uint32_t sDS = smem_u32(smem + C::OFF_DS), sSTG = smem_u32(smem + C::OFF_STG);

  auto step_coords = [&](int s, int& h, int& m0) {
    h = h_first + s / mq;
    m0 = (m_start + s % mq) * BM;
  };

  if (warp == 0) {
    if (lane == 0) {
      // ------------------------------------------------------------ TMA producer
      mbar_arrive_expect_tx(smem_u32(kv_full), 2 * C::KV_BYTES);
#pragma unroll
      for (int kb = 0; kb < KSUB; ++kb) {
        tma_load_2d(sK + kb * BN * 128, &tmK, smem_u32(kv_full), kvh * D + kb * 64, n0);
        tma_load_2d(sV + kb * BN * 128, &tmV, smem_u32(kv_full), kvh * D + kb * 64, n0);
      }
      // order Q(0), dO(0), Q(1), dO(1), ... = the MMA warp's release order (dP(s) frees dO(s) before
      // dK(s) / dQ(s) free Q stage s)
      for (int s = 0; s < steps; ++s) {
        const int st = s % C::QSTAGES;
        int h, m0;
        step_coords(s, h, m0);
        mbar_wait(smem_u32(&q_empty[st]), ((s / C::QSTAGES) & 1) ^ 1);
        const uint32_t fb = smem_u32(&q_full[st]);
        const uint32_t nstat = (uint32_t)min(BM, T - m0) * 4u;
        mbar_arrive_expect_tx(fb, C::QT_BYTES + 2 * nstat);
#pragma unroll
        for (int kb = 0; kb < KSUB; ++kb) tma_load_2d(sQ + st * C::QT_BYTES + kb * BM * 128, &tmQ, fb, h * D + kb * 64, m0);
        const uint32_t sst = smem_u32(stat + st * 2 * BM);
        bulk_load(sst, lse + (int64_t)h * T + m0, nstat, fb);
        bulk_load(sst + BM * 4, dvec + (int64_t)h * T + m0, nstat, fb);
        mbar_wait(smem_u32(do_empty), (s & 1) ^ 1);
        mbar_arrive_expect_tx(smem_u32(do_full), C::QT_BYTES);
#pragma unroll
        for (int kb = 0; kb < KSUB; ++kb) tma_load_2d(sDO + kb * BM * 128, &tmDO, smem_u32(do_full), h * D + kb * 64, m0);
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer (whole warp, elect.sync)
    constexpr uint32_t ID_SS = idesc_bf16(BN, BM, false, false);  // S^T, dP^T
    constexpr uint32_t ID_G = idesc_bf16(BN, D, false, true);     // dV, dK (A from TMEM, B MN-major)
    constexpr uint32_t ID_Q = idesc_bf16(BM, D, true, true);      // dQ = dS K (A, B MN-major)
    const uint32_t k_k = desc_lo(sK, 16), v_k = desc_lo(sV, 16), k_mn = desc_lo(sK, BN * 128);
    const uint32_t o_k = desc_lo(sDO, 16), o_mn = desc_lo(sDO, BM * 128);
    const uint32_t ds_mn = desc_lo(sDS, BN * 128);
    auto mma_s = [&](int s) {
      const int st = s % C::QSTAGES;
      mbar_wait(smem_u32(&q_full[st]), (s / C::QSTAGES) & 1);
      tc_fence_after();
      const uint32_t q_k = desc_lo(sQ + st * C::QT_BYTES, 16);
#pragma unroll
      for (int kb = 0; kb < KSUB; ++kb)
#pragma unroll
        for (int k = 0; k < 4; ++k)
          tc_mma_lo_w(tmem + C::COL_S, k_k + kb * (BN * 8) + k * 2, q_k + kb * (BM * 8) + k * 2, ID_SS, (kb | k) ? 1u : 0u);
      tc_commit_w(smem_u32(s_full));
    };
    if (steps > 0) {
      mbar_wait(smem_u32(kv_full), 0);
      mma_s(0);
    }
    for (int s = 0; s < steps; ++s) {
      const int st = s % C::QSTAGES;
      // dV(s) += P^T(s) dO(s): P^T of queries 16k.. sits in warp (k / 2)'s columns, 8 per 16 queries
      mbar_wait(smem_u32(do_full), s & 1);
      mbar_wait(smem_u32(p_full), s & 1);
      tc_fence_after();
#pragma unroll
      for (int k = 0; k < BM / 16; ++k)
        tc_mma_ts_lo_w(tmem + C::COL_DV, tmem + C::COL_S + 32 * (k >> 1) + 8 * (k & 1), o_mn + k * 128, ID_G,
                       (s > 0 || k > 0) ? 1u : 0u);
      // dP^T(s) = V dO^T, once dQ(s-1) has been drained out of these columns
      if (s > 0) mbar_wait(smem_u32(dq_empty), (s - 1) & 1);
      tc_fence_after();
#pragma unroll
      for (int kb = 0; kb < KSUB; ++kb)
#pragma unroll
        for (int k = 0; k < 4; ++k)
          tc_mma_lo_w(tmem + C::COL_DP, v_k + kb * (BN * 8) + k * 2, o_k + kb * (BM * 8) + k * 2, ID_SS, (kb | k) ? 1u : 0u);
      tc_commit_w(smem_u32(dp_full));
      tc_commit_w(smem_u32(do_empty));
      // S(s+1) over S(s) / P(s): dV(s) (issued above) is the last reader of P(s)
      if (s + 1 < steps) mma_s(s + 1);
      // dK(s) += dS^T(s) Q(s) (A = dS^T from TMEM), dQ(s) = dS(s) K (over the dP / dS^T columns)
      mbar_wait(smem_u32(ds_full), s & 1);
      tc_fence_after();
      const uint32_t q_mn = desc_lo(sQ + st * C::QT_BYTES, BM * 128);
#pragma unroll
      for (int k = 0; k < BM / 16; ++k)
        tc_mma_ts_lo_w(tmem + C::COL_DK, tmem + C::COL_DP + 32 * (k >> 1) + 8 * (k & 1), q_mn + k * 128, ID_G,
                       (s > 0 || k > 0) ? 1u : 0u);
#pragma unroll
      for (int k = 0; k < BN / 16; ++k)
        tc_mma_lo_w(tmem + C::COL_DP, ds_mn + k * 128, k_mn + k * 128, ID_Q, k > 0 ? 1u : 0u);
      tc_commit_w(smem_u32(dq_full));
      tc_commit_w(smem_u32(&q_empty[st]));
    }
    tc_commit_w(smem_u32(acc_done));
  } else {
    // ------------------------------------------------------------ softmax warps: row = key, 32 queries each
    const int quarter = warp & 3;
    const int g = (warp - 2) >> 2;  // query column group 0..3 (= the dQ chunk this warp drains)
    const int r = quarter * 32 + lane;
    const int key = n0 + r;
    const uint32_t lane_addr = tmem + ((uint32_t)(quarter * 32) << 16);
    const bool issuer = (warp & 3) == 2 && lane == 0;  // one thread per column group issues its reduces
    // dQ(s-1) drain: this warp's 32 d columns of its 32 query rows (TMEM lane = query)
    auto drain = [&](int s_prev) {
      int h, m0;
      step_coords(s_prev, h, m0);
      mbar_wait(smem_u32(dq_full), s_prev & 1);
      tc_fence_after();
      if (C::DQC * g >= D) {  // head_dim 64: no chunk for this column group
        __syncwarp();
        if (lane == 0) mbar_arrive(smem_u32(dq_empty));
        return;
      }
      float v[32];
      tmem_ld32_nowait(lane_addr + C::COL_DP + C::DQC * g, reinterpret_cast<uint32_t*>(v));
      tmem_wait_ld();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_u32(dq_empty));
      // boxes 0, 1 live in the dS^T buffer (free until this step's dS store, which waits for their
      // reduces to have read them: stg_free); boxes 2, 3 are reused a step later (the issuer waits)
      const uint32_t sb = g < 2 ? sDS + g * C::STG_BYTES : sSTG + (g - 2) * C::STG_BYTES;
      if (g >= 2) {
        if (issuer) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        named_bar(1 + g, 128);
      }
#pragma unroll
      for (int cc = 0; cc < 8; ++cc)
        asm volatile("st.shared.v4.f32 [%0], {%1,%2,%3,%4};" ::"r"(sb + sw128(r, cc)), "f"(v[cc * 4] * scale),
                     "f"(v[cc * 4 + 1] * scale), "f"(v[cc * 4 + 2] * scale), "f"(v[cc * 4 + 3] * scale)
                     : "memory");
      fence_async_smem();
      named_bar(1 + g, 128);
      if (issuer) {
        tma_reduce_add_2d(&tmDQ, sb, h * D + C::DQC * g, m0);
        bulk_commit();
        if (g < 2) {
          asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
          mbar_arrive(smem_u32(&stg_free[g]));
        }
      }
    };
    for (int s = 0, mi = 0; s < steps; ++s, mi = (mi + 1 == mq) ? 0 : mi + 1) {
      const int m0 = (m_start + mi) * BM;
      const int st = s % C::QSTAGES;
      const bool tile_mask = (causal && m0 < n0 + BN - 1) || n0 + BN > T || m0 + BM > T;
      mbar_wait(smem_u32(&q_full[st]), (s / C::QSTAGES) & 1);  // lse / D rows of this step
      mbar_wait(smem_u32(s_full), s & 1);
      tc_fence_after();
      float p[32];
      tmem_ld32_nowait(lane_addr + C::COL_S + 32 * g, reinterpret_cast<uint32_t*>(p));
      tmem_wait_ld();
      const float* sl = stat + st * 2 * BM + 32 * g;
      {
        uint32_t pp[16];
#pragma unroll
        for (int i = 0; i < 32; i += 4) {
          const float4 nl = *reinterpret_cast<const float4*>(sl + i);
          const float l4[4] = {nl.x, nl.y, nl.z, nl.w};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            float pe = ex2(fmaf(p[i + e], scale_log2, -l4[e] * kLog2e));
            if (tile_mask) {
              const int q = m0 + 32 * g + i + e;
              pe = (key >= T || q >= T || (causal && q < key)) ? 0.f : pe;
            }
            p[i + e] = pe;
          }
          pp[i / 2] = pack_bf16x2(p[i], p[i + 1]);
          pp[i / 2 + 1] = pack_bf16x2(p[i + 2], p[i + 3]);
        }
        tmem_st16(lane_addr + C::COL_S + 32 * g, pp);  // over this warp's own (already read) S columns
        tmem_wait_st();
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_u32(p_full));
      if (s > 0) drain(s - 1);  // runs while the tensor core does dV(s)
      mbar_wait(smem_u32(dp_full), s & 1);
      tc_fence_after();
      uint32_t qq[16];
#pragma unroll
      for (int hf = 0; hf < 2; ++hf) {
        float dp[16];
        tmem_ld16_nowait(lane_addr + C::COL_DP + 32 * g + 16 * hf, reinterpret_cast<uint32_t*>(dp));
        tmem_wait_ld();
#pragma unroll
        for (int i = 0; i < 16; i += 4) {
          const float4 dd = *reinterpret_cast<const float4*>(sl + BM + 16 * hf + i);
          const int b = 16 * hf + i;
          qq[b / 2] = pack_bf16x2(p[b] * (dp[i] - dd.x), p[b + 1] * (dp[i + 1] - dd.y));
          qq[b / 2 + 1] = pack_bf16x2(p[b + 2] * (dp[i + 2] - dd.z), p[b + 3] * (dp[i + 3] - dd.w));
        }
      }
      // dS^T row r -> TMEM over this warp's own (already read) dP columns: the A operand of dK
      tmem_st16(lane_addr + C::COL_DP + 32 * g, qq);
      // and -> shared memory (queries 32g .. 32g+31: box g / 2, 16-byte chunks 4 (g & 1) .. + 3), the
      // dS operand of the dQ MMA, once box g / 2's staging reduce of dQ(s-1) has read that half
      if (s > 0) mbar_wait(smem_u32(&stg_free[g >> 1]), (s - 1) & 1);
      const uint32_t db = sDS + (g >> 1) * (BN * 128);
#pragma unroll
      for (int ch = 0; ch < 4; ++ch)
        asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(db + sw128(r, (g & 1) * 4 + ch)), "r"(qq[ch * 4]),
                     "r"(qq[ch * 4 + 1]), "r"(qq[ch * 4 + 2]), "r"(qq[ch * 4 + 3])
                     : "memory");
      tmem_wait_st();
      fence_async_smem();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_u32(ds_full));
    }
    if (steps > 0) drain(steps - 1);
    if (issuer) bulk_wait0();
    // ------------------------------------------------------------ dK / dV epilogue (all 16 warps)
    mbar_wait(smem_u32(acc_done), 0);
    tc_fence_after();
    const bool ok = key < T && steps > 0;
#pragma unroll 1
    for (int which = 0; which < 2; ++which) {
      const uint32_t col = which ? C::COL_DV : C::COL_DK;
      const float mul = which ? 1.f : scale;
      __nv_bfloat16* row = which ? dv + (int64_t)key * dvs + (int64_t)kvh * D : dk + (int64_t)key * dks + (int64_t)kvh * D;
      if (32 * g >= D) break;  // head_dim 64: warps g = 0, 1 hold the columns
      if (which == 0 && rope_cs != nullptr && !atomic_dkv) {
        // inverse rotary (head_dim 128 only, checked on the host), pairs (i, i + D/2): i in [16g, 16g + 16)
        const float2* cs = rope_cs + (int64_t)(key < T ? key : 0) * (D / 2);
        uint32_t va[16], vb[16];
        tmem_ld16_nowait(lane_addr + col + 16 * g, va);
        tmem_ld16_nowait(lane_addr + col + D / 2 + 16 * g, vb);
        tmem_wait_ld();
        if (ok) {
#pragma unroll
          for (int q8 = 0; q8 < 2; ++q8) {
            float oa[8], ob[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              const float2 t = cs[16 * g + q8 * 8 + j];
              const float x = __uint_as_float(va[q8 * 8 + j]) * mul, y = __uint_as_float(vb[q8 * 8 + j]) * mul;
              oa[j] = x * t.x + y * t.y;
              ob[j] = y * t.x - x * t.y;
            }
            *reinterpret_cast<uint4*>(row + 16 * g + q8 * 8) = pack8(oa);
            *reinterpret_cast<uint4*>(row + D / 2 + 16 * g + q8 * 8) = pack8(ob);
          }
        }
      } else {
        uint32_t v[32];
        tmem_ld32_nowait(lane_addr + col + 32 * g, v);
        tmem_wait_ld();
        if (ok && atomic_dkv) {
          float* acc = dkv_acc + (which ? (int64_t)T * hkv * D : 0) + ((int64_t)key * hkv + kvh) * D + 32 * g;
#pragma unroll
          for (int q4 = 0; q4 < 8; ++q4)
            atomicAdd(reinterpret_cast<float4*>(acc + q4 * 4),
                      make_float4(__uint_as_float(v[q4 * 4 + 0]) * mul, __uint_as_float(v[q4 * 4 + 1]) * mul,
                                  __uint_as_float(v[q4 * 4 + 2]) * mul, __uint_as_float(v[q4 * 4 + 3]) * mul));
        } else if (ok) {
#pragma unroll
          for (int q4 = 0; q4 < 4; ++q4) {
            float f[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) f[j] = __uint_as_float(v[q4 * 8 + j]) * mul;
            *reinterpret_cast<uint4*>(row + 32 * g + q4 * 8) = pack8(f);
          }
        }
      }
      if (!atomic_dkv && steps == 0 && key < T) {  // no causal work: gradients are zero
        for (int c = 32 * g; c < 32 * g + 32; c += 8) *reinterpret_cast<uint4*>(row + c) = make_uint4(0, 0, 0, 0);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) tmem_dealloc(tmem, 512);
}

// =====================================================================================
// Backward as two kernels (KPO_ATTN_BWD=4; deterministic dQ, measured slower than the 64-query kernel:
// with P / dS aliased over S / dP in TMEM, each step's softmax sits between the dV and S MMAs, and
// the dQ kernel's short CTAs pay their prologue / epilogue serially):
//   attn_bwd_dq_kernel    one CTA per (q head, 128 queries), loops over the causal key tiles:
//                           S = Q K^T, dP = dO V^T, dS = P (dP - D), dQ += dS K
//                         Q and dO stay in TMEM (the A operands of S and dP), dS is written over dP
//                         (the TMEM A operand of the dQ MMA), dQ accumulates in TMEM and leaves once,
//                         in bf16 (inverse-rotated for the fused RoPE path).  It also computes
//                         D = rowsum(dO * O) for its rows and writes it for the second kernel.
//   attn_bwd_dkdv_kernel  one CTA per (kv head, 128 keys), loops over the GQA group x causal query
//                         tiles: S^T = K Q^T, dP^T = V dO^T, dV += P^T dO, dK += dS^T Q, with P^T / dS^T
//                         written over S^T / dP^T (the TMEM A operands of dV / dK).
// The single-kernel backward reduces dQ across key tiles through fp32 atomics in L2 and stages it
// through shared memory; here every MMA is M=128 x N=128 x K=128, the K / V (dQ kernel) and Q / dO
// (dK/dV kernel) A operands come from TMEM or are read once per 128x128 block, nothing is reduced
// across CTAs (deterministic), and the pre / post kernels (D vector, dQ accumulator zeroing and
// conversion) disappear, at the price of recomputing S and dP (7 GEMMs per block instead of 5).
template <int D>
struct BwdDq {
  static constexpr int BM = 128, BN = 128, STAGES = 2, KSUB = D / 64;
  static constexpr int KV_BYTES = BN * D * 2;
  static constexpr int OFF_K = 0, OFF_V = STAGES * KV_BYTES, OFF_RED = 2 * STAGES * KV_BYTES;
  static constexpr int OFF_BAR = OFF_RED + 4 * BM * 4;
  static constexpr int SMEM = OFF_BAR + 256 + 1024;
  static constexpr int COL_S = 0, COL_DP = 128, COL_DQ = 256, COL_Q = 384, COL_DO = 384 + D / 2;
  static constexpr int SM_WARPS = 16;
  static constexpr int THREADS = (2 + SM_WARPS) * 32;
};

template <int D>
__global__ void __launch_bounds__(BwdDq<D>::THREADS, 1)
    attn_bwd_dq_kernel(const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmV,
                       const __nv_bfloat16* __restrict__ q, const __nv_bfloat16* __restrict__ dout,
                       const __nv_bfloat16* __restrict__ o, const float* __restrict__ lse,
                       float* __restrict__ dvec, __nv_bfloat16* __restrict__ dq, int T, int hq, int hkv,
                       int64_t qs, int64_t os, int64_t dqs, float scale, int causal,
                       const float2* __restrict__ rope_cs) {
  ::kpo::pdl_launch_dependents();
  using C = BwdDq<D>;
  constexpr int BM = C::BM, BN = C::BN, KSUB = C::KSUB;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + C::OFF_BAR);
  uint64_t* kv_full = bar + 0;   // [2]
  uint64_t* kv_empty = bar + 2;  // [2]
  uint64_t* s_full = bar + 4;
  uint64_t* s_empty = bar + 5;
  uint64_t* dp_full = bar + 6;
  uint64_t* ds_full = bar + 7;
  uint64_t* qo_ready = bar + 8;
  uint64_t* acc_done = bar + 9;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 10);
  float* red = reinterpret_cast<float*>(smem + C::OFF_RED);  // [4 column groups][BM] partial D

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int h = blockIdx.x;
  const int ntiles = (T + BM - 1) / BM;
  const int mt = ntiles - 1 - (int)blockIdx.y;  // the longest causal rows first
  const int m0 = mt * BM;
  const int kvh = h / (hq / hkv);
  const int steps = causal ? min(mt + 1, (T + BN - 1) / BN) : (T + BN - 1) / BN;
  const float scale_log2 = scale * kLog2e;

  if (threadIdx.x == 0) {
    for (int i = 0; i < C::STAGES; ++i) {
      mbar_init(smem_u32(&kv_full[i]), 1);
      mbar_init(smem_u32(&kv_empty[i]), 1);
    }
    mbar_init(smem_u32(s_full), 1);
    mbar_init(smem_u32(s_empty), C::SM_WARPS);
    mbar_init(smem_u32(dp_full), 1);
    mbar_init(smem_u32(ds_full), C::SM_WARPS);
    mbar_init(smem_u32(qo_ready), C::SM_WARPS);
    mbar_init(smem_u32(acc_done), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) tmem_alloc(smem_u32(tmem_slot), 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (*tmem_slot != 0) __trap();
  ::kpo::pdl_wait();
  constexpr uint32_t tmem = 0;
  const uint32_t sK = smem_u32(smem + C::OFF_K), sV = smem_u32(smem + C::OFF_V);

  if (warp == 0) {
    if (lane == 0) {
      // ------------------------------------------------------------ TMA producer: K_n, V_n ring
      for (int n = 0; n < steps; ++n) {
        const int st = n % C::STAGES;
        mbar_wait(smem_u32(&kv_empty[st]), ((n / C::STAGES) & 1) ^ 1);
        const uint32_t fb = smem_u32(&kv_full[st]);
        mbar_arrive_expect_tx(fb, 2 * C::KV_BYTES);
#pragma unroll
        for (int kb = 0; kb < KSUB; ++kb) {
          tma_load_2d(sK + st * C::KV_BYTES + kb * BN * 128, &tmK, fb, kvh * D + kb * 64, n * BN);
          tma_load_2d(sV + st * C::KV_BYTES + kb * BN * 128, &tmV, fb, kvh * D + kb * 64, n * BN);
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer (whole warp, elect.sync)
    constexpr uint32_t ID_S = idesc_bf16(BM, BN, false, false);   // S, dP: A (Q / dO) from TMEM
    constexpr uint32_t ID_Q = idesc_bf16(BM, D, false, true);     // dQ += dS K: A = dS from TMEM, B MN-major
    mbar_wait(smem_u32(qo_ready), 0);
    tc_fence_after();
    auto mma_qk = [&](int n, uint32_t col_a, uint32_t b_base, uint32_t col_d, uint64_t* done) {
      // col_d = A (from TMEM, D / 2 packed columns) x B^T (tile [BN keys][D], K-major)
      const uint32_t b_k = desc_lo(b_base, 16);
#pragma unroll
      for (int kk = 0; kk < D / 16; ++kk)
        tc_mma_ts_lo_w(tmem + col_d, tmem + col_a + 8 * kk, b_k + (kk >> 2) * (BN * 8) + (kk & 3) * 2, ID_S,
                       kk > 0 ? 1u : 0u);
      tc_commit_w(smem_u32(done));
    };
    auto mma_s = [&](int n) {
      const int st = n % C::STAGES;
      mbar_wait(smem_u32(&kv_full[st]), (n / C::STAGES) & 1);
      tc_fence_after();
      mma_qk(n, C::COL_Q, sK + st * C::KV_BYTES, C::COL_S, s_full);
    };
    auto mma_dp = [&](int n) {
      const int st = n % C::STAGES;  // kv_full[st] was waited for by mma_s(n)
      mma_qk(n, C::COL_DO, sV + st * C::KV_BYTES, C::COL_DP, dp_full);
    };
    if (steps > 0) {
      mma_s(0);
      mma_dp(0);
    }
    for (int n = 0; n < steps; ++n) {
      const int st = n % C::STAGES;
      if (n + 1 < steps) {
        mbar_wait(smem_u32(s_empty), n & 1);  // the softmax has read S(n)
        mma_s(n + 1);
      }
      // dQ += dS(n) K_n: dS of keys 16k.. sits in softmax warp (k / 2)'s dP columns, 8 per 16 keys
      mbar_wait(smem_u32(ds_full), n & 1);
      tc_fence_after();
      const uint32_t k_mn = desc_lo(sK + st * C::KV_BYTES, BN * 128);
#pragma unroll
      for (int k = 0; k < BN / 16; ++k)
        tc_mma_ts_lo_w(tmem + C::COL_DQ, tmem + C::COL_DP + 32 * (k >> 1) + 8 * (k & 1), k_mn + k * 128, ID_Q,
                       (n > 0 || k > 0) ? 1u : 0u);
      tc_commit_w(smem_u32(&kv_empty[st]));
      if (n + 1 < steps) mma_dp(n + 1);  // over dS(n): the dQ MMA above is its last reader
    }
    tc_commit_w(smem_u32(acc_done));
  } else {
    // ------------------------------------------------------------ softmax warps: row = query, 32 keys each
    const int quarter = warp & 3;
    const int g = (warp - 2) >> 2;
    const int qr = quarter * 32 + lane;
    const int t = m0 + qr;
    const bool row_ok = t < T;
    const uint32_t lane_addr = tmem + ((uint32_t)(quarter * 32) << 16);
    // Q / dO rows -> TMEM (this warp's 32 head-dim columns = 16 packed TMEM columns); D partials
    float dpart = 0.f;
    if (32 * g < D) {
      uint32_t qa[16], da[16];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        uint4 uq = make_uint4(0, 0, 0, 0), ud = uq, uo = uq;
        if (row_ok) {
          uq = *reinterpret_cast<const uint4*>(q + (int64_t)t * qs + (int64_t)h * D + 32 * g + 8 * c);
          ud = *reinterpret_cast<const uint4*>(dout + (int64_t)t * os + (int64_t)h * D + 32 * g + 8 * c);
          uo = *reinterpret_cast<const uint4*>(o + (int64_t)t * os + (int64_t)h * D + 32 * g + 8 * c);
        }
        qa[4 * c] = uq.x, qa[4 * c + 1] = uq.y, qa[4 * c + 2] = uq.z, qa[4 * c + 3] = uq.w;
        da[4 * c] = ud.x, da[4 * c + 1] = ud.y, da[4 * c + 2] = ud.z, da[4 * c + 3] = ud.w;
        float fd[8], fo[8];
        unpack8(ud, fd);
        unpack8(uo, fo);
#pragma unroll
        for (int j = 0; j < 8; ++j) dpart = fmaf(fd[j], fo[j], dpart);
      }
      tmem_st16(lane_addr + C::COL_Q + 16 * g, qa);
      tmem_st16(lane_addr + C::COL_DO + 16 * g, da);
      tmem_wait_st();
    }
    red[g * BM + qr] = dpart;
    tc_fence_before();
    named_bar(1, C::SM_WARPS * 32);
    const float dsum = red[qr] + red[BM + qr] + red[2 * BM + qr] + red[3 * BM + qr];
    if (g == 0 && row_ok) dvec[(int64_t)h * T + t] = dsum;
    const float nl = row_ok ? lse[(int64_t)h * T + t] * kLog2e : 0.f;
    __syncwarp();
    if (lane == 0) mbar_arrive(smem_u32(qo_ready));
    for (int n = 0; n < steps; ++n) {
      const int k0 = n * BN + 32 * g;
      const bool tile_mask = (causal && n * BN + BN - 1 > m0) || n * BN + BN > T || m0 + BM > T;
      mbar_wait(smem_u32(s_full), n & 1);
      tc_fence_after();
      float p[32];
      tmem_ld32_nowait(lane_addr + C::COL_S + 32 * g, reinterpret_cast<uint32_t*>(p));
      tmem_wait_ld();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_u32(s_empty));
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        float pe = ex2(fmaf(p[i], scale_log2, -nl));
        if (tile_mask) {
          const int key = k0 + i;
          pe = (!row_ok || key >= T || (causal && key > t)) ? 0.f : pe;
        }
        p[i] = pe;
      }
      mbar_wait(smem_u32(dp_full), n & 1);
      tc_fence_after();
      uint32_t qq[16];
#pragma unroll
      for (int hf = 0; hf < 2; ++hf) {
        float dp[16];
        tmem_ld16_nowait(lane_addr + C::COL_DP + 32 * g + 16 * hf, reinterpret_cast<uint32_t*>(dp));
        tmem_wait_ld();
#pragma unroll
        for (int i = 0; i < 16; i += 2)
          qq[(16 * hf + i) / 2] = pack_bf16x2(p[16 * hf + i] * (dp[i] - dsum), p[16 * hf + i + 1] * (dp[i + 1] - dsum));
      }
      tmem_st16(lane_addr + C::COL_DP + 32 * g, qq);  // over this warp's own (already read) dP columns
      tmem_wait_st();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_u32(ds_full));
    }
    // ------------------------------------------------------------ dQ epilogue: row t, bf16 (+ inverse rotary)
    mbar_wait(smem_u32(acc_done), 0);
    tc_fence_after();
    if (32 * g < D) {
      __nv_bfloat16* row = dq + (int64_t)t * dqs + (int64_t)h * D;
      if (rope_cs != nullptr) {  // head_dim 128 (host-checked): pairs (i, i + 64), i in [16g, 16g + 16)
        uint32_t va[16], vb[16];
        tmem_ld16_nowait(lane_addr + C::COL_DQ + 16 * g, va);
        tmem_ld16_nowait(lane_addr + C::COL_DQ + D / 2 + 16 * g, vb);
        tmem_wait_ld();
        if (row_ok) {
          const float2* cs = rope_cs + (int64_t)t * (D / 2);
#pragma unroll
          for (int q8 = 0; q8 < 2; ++q8) {
            float oa[8], ob[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              const float2 r = cs[16 * g + q8 * 8 + j];
              const float x = __uint_as_float(va[q8 * 8 + j]) * scale, y = __uint_as_float(vb[q8 * 8 + j]) * scale;
              oa[j] = x * r.x + y * r.y;
              ob[j] = y * r.x - x * r.y;
            }
            *reinterpret_cast<uint4*>(row + 16 * g + q8 * 8) = pack8(oa);
            *reinterpret_cast<uint4*>(row + D / 2 + 16 * g + q8 * 8) = pack8(ob);
          }
        }
      } else {
        uint32_t v[32];
        tmem_ld32_nowait(lane_addr + C::COL_DQ + 32 * g, v);
        tmem_wait_ld();
        if (row_ok) {
#pragma unroll
          for (int q4 = 0; q4 < 4; ++q4) {
            float f[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) f[j] = __uint_as_float(v[q4 * 8 + j]) * scale;
            *reinterpret_cast<uint4*>(row + 32 * g + q4 * 8) = pack8(f);
          }
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) tmem_dealloc(tmem, 512);
}

template <int D>
struct BwdKV {
  static constexpr int BN = 128, BM = 128, STAGES = 2, KSUB = D / 64;
  static constexpr int KV_BYTES = BN * D * 2, QT_BYTES = BM * D * 2;
  static constexpr int OFF_K = 0, OFF_V = KV_BYTES, OFF_Q = 2 * KV_BYTES;
  static constexpr int OFF_DO = OFF_Q + STAGES * QT_BYTES;
  static constexpr int OFF_STAT = OFF_DO + STAGES * QT_BYTES;  // [STAGES][lse BM | D BM]
  static constexpr int OFF_BAR = OFF_STAT + STAGES * 2 * BM * 4;
  static constexpr int SMEM = OFF_BAR + 256 + 1024;
  static constexpr int COL_S = 0, COL_DP = 128, COL_DV = 256, COL_DK = 384;
  static constexpr int SM_WARPS = 16;
  static constexpr int THREADS = (2 + SM_WARPS) * 32;
};

template <int D>
__global__ void __launch_bounds__(BwdKV<D>::THREADS, 1)
    attn_bwd_dkdv_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                         const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmDO,
                         const float* __restrict__ lse, const float* __restrict__ dvec,
                         __nv_bfloat16* __restrict__ dk, __nv_bfloat16* __restrict__ dv, int T, int hq, int hkv,
                         int64_t dks, int64_t dvs, float scale, int causal, float* __restrict__ dkv_acc,
                         int split_group, int qsplit_tiles, const float2* __restrict__ rope_cs) {
  // grid / modes as attn_bwd_tc_kernel (split-group, query chunks, fused inverse rotary of dK)
  ::kpo::pdl_launch_dependents();
  using C = BwdKV<D>;
  constexpr int BN = C::BN, BM = C::BM, KSUB = C::KSUB;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + C::OFF_BAR);
  uint64_t* kv_full = bar + 0;
  uint64_t* q_full = bar + 1;    // [2]
  uint64_t* q_empty = bar + 3;   // [2]
  uint64_t* do_full = bar + 5;   // [2]
  uint64_t* do_empty = bar + 7;  // [2]
  uint64_t* s_full = bar + 9;
  uint64_t* p_full = bar + 10;
  uint64_t* dp_full = bar + 11;
  uint64_t* ds_full = bar + 12;
  uint64_t* acc_done = bar + 13;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 14);
  float* stat = reinterpret_cast<float*>(smem + C::OFF_STAT);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nblk = blockIdx.y;
  const bool split = split_group != 0;
  const int group = split ? 1 : hq / hkv;
  const int h_first = split ? (int)blockIdx.x : (int)blockIdx.x * (hq / hkv);
  const int kvh = split ? (int)blockIdx.x / (hq / hkv) : (int)blockIdx.x;
  const int n0 = nblk * BN;
  const int total_m = (T + BM - 1) / BM;
  int m_start = causal ? n0 / BM : 0, m_end = total_m;
  const bool chunked = gridDim.z > 1 && nblk < qsplit_tiles;
  if (gridDim.z > 1) {
    if (chunked) {
      const int qper = (total_m + (int)gridDim.z - 1) / (int)gridDim.z;
      m_start = max(m_start, (int)blockIdx.z * qper);
      m_end = min(total_m, ((int)blockIdx.z + 1) * qper);
      if (m_start >= m_end) return;
    } else if (blockIdx.z != 0) {
      return;
    }
  }
  const bool atomic_dkv = split || chunked;
  const int mq = m_end - m_start;
  const int steps = group * mq;
  const float scale_log2 = scale * kLog2e;

  if (threadIdx.x == 0) {
    mbar_init(smem_u32(kv_full), 1);
    for (int i = 0; i < C::STAGES; ++i) {
      mbar_init(smem_u32(&q_full[i]), 1);
      mbar_init(smem_u32(&q_empty[i]), 1);
      mbar_init(smem_u32(&do_full[i]), 1);
      mbar_init(smem_u32(&do_empty[i]), 1);
    }
    mbar_init(smem_u32(s_full), 1);
    mbar_init(smem_u32(p_full), C::SM_WARPS);
    mbar_init(smem_u32(dp_full), 1);
    mbar_init(smem_u32(ds_full), C::SM_WARPS);
    mbar_init(smem_u32(acc_done), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) tmem_alloc(smem_u32(tmem_slot), 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (*tmem_slot != 0) __trap();
  ::kpo::pdl_wait();  // the dQ kernel before us wrote the D vector
  constexpr uint32_t tmem = 0;
  const uint32_t sK = smem_u32(smem + C::OFF_K), sV = smem_u32(smem + C::OFF_V);
  const uint32_t sQ = smem_u32(smem + C::OFF_Q), sDO = smem_u32(smem + C::OFF_DO);

  auto step_coords = [&](int s, int& h, int& m0) {
    h = h_first + s / mq;
    m0 = (m_start + s % mq) * BM;
  };

  if (warp == 0) {
    if (lane == 0) {
      // ------------------------------------------------------------ TMA producer
      mbar_arrive_expect_tx(smem_u32(kv_full), 2 * C::KV_BYTES);
#pragma unroll
      for (int kb = 0; kb < KSUB; ++kb) {
        tma_load_2d(sK + kb * BN * 128, &tmK, smem_u32(kv_full), kvh * D + kb * 64, n0);
        tma_load_2d(sV + kb * BN * 128, &tmV, smem_u32(kv_full), kvh * D + kb * 64, n0);
      }
      for (int s = 0; s < steps; ++s) {
        const int st = s % C::STAGES;
        const uint32_t ph = ((s / C::STAGES) & 1) ^ 1;
        int h, m0;
        step_coords(s, h, m0);
        const uint32_t nstat = (uint32_t)min(BM, T - m0) * 4u;
        mbar_wait(smem_u32(&q_empty[st]), ph);
        const uint32_t fb = smem_u32(&q_full[st]);
        mbar_arrive_expect_tx(fb, C::QT_BYTES + 2 * nstat);
#pragma unroll
        for (int kb = 0; kb < KSUB; ++kb) tma_load_2d(sQ + st * C::QT_BYTES + kb * BM * 128, &tmQ, fb, h * D + kb * 64, m0);
        const uint32_t sst = smem_u32(stat + st * 2 * BM);
        bulk_load(sst, lse + (int64_t)h * T + m0, nstat, fb);
        bulk_load(sst + BM * 4, dvec + (int64_t)h * T + m0, nstat, fb);
        mbar_wait(smem_u32(&do_empty[st]), ph);
        const uint32_t ob = smem_u32(&do_full[st]);
        mbar_arrive_expect_tx(ob, C::QT_BYTES);
#pragma unroll
        for (int kb = 0; kb < KSUB; ++kb) tma_load_2d(sDO + st * C::QT_BYTES + kb * BM * 128, &tmDO, ob, h * D + kb * 64, m0);
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer (whole warp, elect.sync)
    constexpr uint32_t ID_SS = idesc_bf16(BN, BM, false, false);  // S^T, dP^T
    constexpr uint32_t ID_G = idesc_bf16(BN, D, false, true);     // dV, dK: A from TMEM, B MN-major
    const uint32_t k_k = desc_lo(sK, 16), v_k = desc_lo(sV, 16);
    auto mma_ss = [&](uint32_t a_k, uint32_t b_base, uint32_t col_d, uint64_t* done) {
      const uint32_t b_k = desc_lo(b_base, 16);
#pragma unroll
      for (int kb = 0; kb < KSUB; ++kb)
#pragma unroll
        for (int k = 0; k < 4; ++k)
          tc_mma_lo_w(tmem + col_d, a_k + kb * (BN * 8) + k * 2, b_k + kb * (BM * 8) + k * 2, ID_SS, (kb | k) ? 1u : 0u);
      tc_commit_w(smem_u32(done));
    };
    auto mma_s = [&](int s) {
      const int st = s % C::STAGES;
      mbar_wait(smem_u32(&q_full[st]), (s / C::STAGES) & 1);
      tc_fence_after();
      mma_ss(k_k, sQ + st * C::QT_BYTES, C::COL_S, s_full);
    };
    auto mma_dp = [&](int s) {
      const int st = s % C::STAGES;
      mbar_wait(smem_u32(&do_full[st]), (s / C::STAGES) & 1);
      tc_fence_after();
      mma_ss(v_k, sDO + st * C::QT_BYTES, C::COL_DP, dp_full);
    };
    if (steps > 0) {
      mbar_wait(smem_u32(kv_full), 0);
      mma_s(0);
      mma_dp(0);
    }
    for (int s = 0; s < steps; ++s) {
      const int st = s % C::STAGES;
      // dV += P^T(s) dO(s): P^T of queries 16k.. sits in softmax warp (k / 2)'s S columns
      mbar_wait(smem_u32(p_full), s & 1);
      tc_fence_after();
      const uint32_t o_mn = desc_lo(sDO + st * C::QT_BYTES, BM * 128);
#pragma unroll
      for (int k = 0; k < BM / 16; ++k)
        tc_mma_ts_lo_w(tmem + C::COL_DV, tmem + C::COL_S + 32 * (k >> 1) + 8 * (k & 1), o_mn + k * 128, ID_G,
                       (s > 0 || k > 0) ? 1u : 0u);
      tc_commit_w(smem_u32(&do_empty[st]));
      if (s + 1 < steps) mma_s(s + 1);  // over S / P(s): the dV MMA above is its last reader
      // dK += dS^T(s) Q(s): dS^T over the dP^T columns, same per-warp layout
      mbar_wait(smem_u32(ds_full), s & 1);
      tc_fence_after();
      const uint32_t q_mn = desc_lo(sQ + st * C::QT_BYTES, BM * 128);
#pragma unroll
      for (int k = 0; k < BM / 16; ++k)
        tc_mma_ts_lo_w(tmem + C::COL_DK, tmem + C::COL_DP + 32 * (k >> 1) + 8 * (k & 1), q_mn + k * 128, ID_G,
                       (s > 0 || k > 0) ? 1u : 0u);
      tc_commit_w(smem_u32(&q_empty[st]));
      if (s + 1 < steps) mma_dp(s + 1);  // over dP^T / dS^T(s): the dK MMA above is its last reader
    }
    tc_commit_w(smem_u32(acc_done));
  } else {
    // ------------------------------------------------------------ softmax warps: row = key, 32 queries each
    const int quarter = warp & 3;
    const int g = (warp - 2) >> 2;
    const int r = quarter * 32 + lane;
    const int key = n0 + r;
    const uint32_t lane_addr = tmem + ((uint32_t)(quarter * 32) << 16);
    for (int s = 0, mi = 0; s < steps; ++s, mi = (mi + 1 == mq) ? 0 : mi + 1) {
      const int m0 = (m_start + mi) * BM;
      const int st = s % C::STAGES;
      const bool tile_mask = (causal && m0 < n0 + BN - 1) || n0 + BN > T || m0 + BM > T;
      mbar_wait(smem_u32(&q_full[st]), (s / C::STAGES) & 1);  // lse / D rows of this step
      mbar_wait(smem_u32(s_full), s & 1);
      tc_fence_after();
      float p[32];
      tmem_ld32_nowait(lane_addr + C::COL_S + 32 * g, reinterpret_cast<uint32_t*>(p));
      tmem_wait_ld();
      const float* sl = stat + st * 2 * BM + 32 * g;
      {
        uint32_t pp[16];
#pragma unroll
        for (int i = 0; i < 32; i += 4) {
          const float4 nl = *reinterpret_cast<const float4*>(sl + i);
          const float l4[4] = {nl.x, nl.y, nl.z, nl.w};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            float pe = ex2(fmaf(p[i + e], scale_log2, -l4[e] * kLog2e));
            if (tile_mask) {
              const int qi = m0 + 32 * g + i + e;
              pe = (key >= T || qi >= T || (causal && qi < key)) ? 0.f : pe;
            }
            p[i + e] = pe;
          }
          pp[i / 2] = pack_bf16x2(p[i], p[i + 1]);
          pp[i / 2 + 1] = pack_bf16x2(p[i + 2], p[i + 3]);
        }
        tmem_st16(lane_addr + C::COL_S + 32 * g, pp);  // over this warp's own (already read) S columns
        tmem_wait_st();
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_u32(p_full));
      mbar_wait(smem_u32(dp_full), s & 1);
      tc_fence_after();
      uint32_t qq[16];
#pragma unroll
      for (int hf = 0; hf < 2; ++hf) {
        float dp[16];
        tmem_ld16_nowait(lane_addr + C::COL_DP + 32 * g + 16 * hf, reinterpret_cast<uint32_t*>(dp));
        tmem_wait_ld();
#pragma unroll
        for (int i = 0; i < 16; i += 4) {
          const float4 dd = *reinterpret_cast<const float4*>(sl + BM + 16 * hf + i);
          const int b = 16 * hf + i;
          qq[b / 2] = pack_bf16x2(p[b] * (dp[i] - dd.x), p[b + 1] * (dp[i + 1] - dd.y));
          qq[b / 2 + 1] = pack_bf16x2(p[b + 2] * (dp[i + 2] - dd.z), p[b + 3] * (dp[i + 3] - dd.w));
        }
      }
      tmem_st16(lane_addr + C::COL_DP + 32 * g, qq);  // over this warp's own (already read) dP^T columns
      tmem_wait_st();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_u32(ds_full));
    }
    // ------------------------------------------------------------ dK / dV epilogue (all 16 warps)
    mbar_wait(smem_u32(acc_done), 0);
    tc_fence_after();
    const bool ok = key < T && steps > 0;
#pragma unroll 1
    for (int which = 0; which < 2; ++which) {
      const uint32_t col = which ? C::COL_DV : C::COL_DK;
      const float mul = which ? 1.f : scale;
      __nv_bfloat16* row = which ? dv + (int64_t)key * dvs + (int64_t)kvh * D : dk + (int64_t)key * dks + (int64_t)kvh * D;
      if (32 * g >= D) break;  // head_dim 64: warps g = 0, 1 hold the columns
      if (which == 0 && rope_cs != nullptr && !atomic_dkv) {
        // inverse rotary (head_dim 128, host-checked), pairs (i, i + D/2): i in [16g, 16g + 16)
        const float2* cs = rope_cs + (int64_t)(key < T ? key : 0) * (D / 2);
        uint32_t va[16], vb[16];
        tmem_ld16_nowait(lane_addr + col + 16 * g, va);
        tmem_ld16_nowait(lane_addr + col + D / 2 + 16 * g, vb);
        tmem_wait_ld();
        if (ok) {
#pragma unroll
          for (int q8 = 0; q8 < 2; ++q8) {
            float oa[8], ob[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              const float2 tc = cs[16 * g + q8 * 8 + j];
              const float x = __uint_as_float(va[q8 * 8 + j]) * mul, y = __uint_as_float(vb[q8 * 8 + j]) * mul;
              oa[j] = x * tc.x + y * tc.y;
              ob[j] = y * tc.x - x * tc.y;
            }
            *reinterpret_cast<uint4*>(row + 16 * g + q8 * 8) = pack8(oa);
            *reinterpret_cast<uint4*>(row + D / 2 + 16 * g + q8 * 8) = pack8(ob);
          }
        }
      } else {
        uint32_t v[32];
        tmem_ld32_nowait(lane_addr + col + 32 * g, v);
        tmem_wait_ld();
        if (ok && atomic_dkv) {
          float* acc = dkv_acc + (which ? (int64_t)T * hkv * D : 0) + ((int64_t)key * hkv + kvh) * D + 32 * g;
#pragma unroll
          for (int q4 = 0; q4 < 8; ++q4)
            atomicAdd(reinterpret_cast<float4*>(acc + q4 * 4),
                      make_float4(__uint_as_float(v[q4 * 4 + 0]) * mul, __uint_as_float(v[q4 * 4 + 1]) * mul,
                                  __uint_as_float(v[q4 * 4 + 2]) * mul, __uint_as_float(v[q4 * 4 + 3]) * mul));
        } else if (ok) {
#pragma unroll
          for (int q4 = 0; q4 < 4; ++q4) {
            float f[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) f[j] = __uint_as_float(v[q4 * 8 + j]) * mul;
            *reinterpret_cast<uint4*>(row + 32 * g + q4 * 8) = pack8(f);
          }
        }
      }
      if (!atomic_dkv && steps == 0 && key < T) {
        for (int c = 32 * g; c < 32 * g + 32; c += 8) *reinterpret_cast<uint4*>(row + c) = make_uint4(0, 0, 0, 0);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) tmem_dealloc(tmem, 512);
}

// dQ kernel, then the dK / dV kernel (same stream; PDL lets the second one's prologue overlap).
template <int D>
int bwd_split_launch(const void* q, const void* k, const void* v, const void* o, const void* dout, const float* lse,
                     float* dvec, void* dq, void* dk, void* dv, int64_t T, int hq, int hkv, int64_t qs, int64_t ks,
                     int64_t vs, int64_t os, int64_t dqs, int64_t dks, int64_t dvs, float scale, int causal,
                     float* dkv_acc, int split_group, int qsplit_tiles, int qchunks, cudaStream_t st,
                     const float* rope_table) {
  using A = BwdDq<D>;
  using B = BwdKV<D>;
  CUtensorMap mq, mk, mv, mo;
  int e;
  if ((e = make_map_2d(&mq, q, (uint64_t)hq * D, T, qs, 64, B::BM))) return e;
  if ((e = make_map_2d(&mk, k, (uint64_t)hkv * D, T, ks, 64, B::BN))) return e;
  if ((e = make_map_2d(&mv, v, (uint64_t)hkv * D, T, vs, 64, B::BN))) return e;
  if ((e = make_map_2d(&mo, dout, (uint64_t)hq * D, T, os, 64, B::BM))) return e;
  static bool set = false;
  if (!set) {
    KPO_CUDA(cudaFuncSetAttribute(attn_bwd_dq_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, A::SMEM));
    KPO_CUDA(cudaFuncSetAttribute(attn_bwd_dkdv_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, B::SMEM));
    set = true;
  }
  const float2* cs = reinterpret_cast<const float2*>(rope_table);
  const unsigned ntiles = (unsigned)((T + A::BM - 1) / A::BM);
  KPO_CUDA(::kpo::pdl_launch(attn_bwd_dq_kernel<D>, dim3((unsigned)hq, ntiles), A::THREADS, A::SMEM, st, mk, mv,
                             (const __nv_bfloat16*)q, (const __nv_bfloat16*)dout, (const __nv_bfloat16*)o, lse, dvec,
                             (__nv_bfloat16*)dq, (int)T, hq, hkv, qs, os, dqs, scale, causal, cs));
  KPO_LAUNCH_CHECK();
  dim3 grid((unsigned)(split_group ? hq : hkv), (unsigned)((T + B::BN - 1) / B::BN), (unsigned)(qchunks > 1 ? qchunks : 1));
  KPO_CUDA(::kpo::pdl_launch(attn_bwd_dkdv_kernel<D>, grid, B::THREADS, B::SMEM, st, mq, mk, mv, mo, lse,
                             (const float*)dvec, (__nv_bfloat16*)dk, (__nv_bfloat16*)dv, (int)T, hq, hkv, dks, dvs,
                             scale, causal, dkv_acc, split_group, qsplit_tiles, cs));
  KPO_LAUNCH_CHECK();
  return KPO_OK;
}

template <int D>
int bwd_launch(const void* q, const void* k, const void* v, const void* dout, const float* lse, const float* dvec,
               float* dq_acc, void* dk, void* dv, int64_t T, int hq, int hkv, int64_t qs, int64_t ks, int64_t vs,
               int64_t os, int64_t dks, int64_t dvs, float scale, int causal, float* dkv_acc, int split_group,
               int qsplit_tiles, int qchunks, cudaStream_t st,
               const float* rope_table) {
  // head_dim 128: the 64-query kernel (measured faster: its dQ^T has TMEM of its own, so the drain
  // and the dQ reduce-adds stay off the critical path; the 128-query kernel must alias dQ with dP^T
  // and stage through the dS^T buffer).  head_dim 64: the 128-query kernel (3.4x the mma.sync one).
  static const int variant = getenv("KPO_ATTN_BWD") ? atoi(getenv("KPO_ATTN_BWD")) : (D == 64 ? 3 : 2);
  if (variant == 3 || D == 64) {  // 128-query steps
    using C3 = Bwd3<D>;
    CUtensorMap mq, mk, mv, mo, mdq;
    int e;
    if ((e = make_map_2d_f32(&mdq, dq_acc, (uint64_t)hq * D, T, (uint64_t)hq * D, C3::DQC, C3::BM, true))) return e;
    if ((e = make_map_2d(&mq, q, (uint64_t)hq * D, T, qs, 64, C3::BM))) return e;
    if ((e = make_map_2d(&mk, k, (uint64_t)hkv * D, T, ks, 64, C3::BN))) return e;
    if ((e = make_map_2d(&mv, v, (uint64_t)hkv * D, T, vs, 64, C3::BN))) return e;
    if ((e = make_map_2d(&mo, dout, (uint64_t)hq * D, T, os, 64, C3::BM))) return e;
    static bool set3 = false;
    if (!set3) {
      KPO_CUDA(cudaFuncSetAttribute(attn_bwd_tc3_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, C3::SMEM));
      set3 = true;
    }
    const int ntiles = (int)((T + C3::BN - 1) / C3::BN);
    dim3 grid((unsigned)(split_group ? hq : hkv), (unsigned)ntiles, (unsigned)(qchunks > 1 ? qchunks : 1));
    KPO_CUDA(::kpo::pdl_launch(attn_bwd_tc3_kernel<D>, grid, C3::THREADS, C3::SMEM, st, mq, mk, mv, mo, mdq, lse, dvec,
                               (__nv_bfloat16*)dk, (__nv_bfloat16*)dv, (int)T, hq, hkv, dks, dvs, scale, causal,
                               dkv_acc, split_group, qsplit_tiles, reinterpret_cast<const float2*>(rope_table)));
    KPO_LAUNCH_CHECK();
    return KPO_OK;
  }
  if constexpr (D == 64) {
    return KPO_ERR_UNSUPPORTED;  // unreachable: head_dim 64 always takes the 128-query kernel
  } else {
  using C = Bwd<D>;
  CUtensorMap mq, mk, mv, mo, mdq;
  int e;
  // dQ reduce boxes of half a step (32 queries): the two halves of the staging tile drain separately
  if ((e = make_map_2d_f32(&mdq, dq_acc, (uint64_t)hq * D, T, (uint64_t)hq * D, D, C::BM / 2))) return e;
  if ((e = make_map_2d(&mq, q, (uint64_t)hq * D, T, qs, 64, C::BM))) return e;
  if ((e = make_map_2d(&mk, k, (uint64_t)hkv * D, T, ks, 64, C::BN))) return e;
  if ((e = make_map_2d(&mv, v, (uint64_t)hkv * D, T, vs, 64, C::BN))) return e;
  if ((e = make_map_2d(&mo, dout, (uint64_t)hq * D, T, os, 64, C::BM))) return e;
  static bool set = false;
  if (!set) {
    KPO_CUDA(cudaFuncSetAttribute(attn_bwd_tc_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
    set = true;
  }
  const int ntiles = (int)((T + C::BN - 1) / C::BN);
  dim3 grid((unsigned)(split_group ? hq : hkv), (unsigned)ntiles, (unsigned)(qchunks > 1 ? qchunks : 1));
  KPO_CUDA(::kpo::pdl_launch(attn_bwd_tc_kernel<D>, grid, C::THREADS, C::SMEM, st, mq, mk, mv, mo, mdq, lse, dvec, dq_acc, (__nv_bfloat16*)dk,
                                                          (__nv_bfloat16*)dv, (int)T, hq, hkv, dks, dvs, scale, causal,
                                                          dkv_acc, split_group, qsplit_tiles,
                                                          getenv("KPO_ATTN_BWD_ABLATE") ? atoi(getenv("KPO_ATTN_BWD_ABLATE")) : 0,
                                                          reinterpret_cast<const float2*>(rope_table)));
  KPO_LAUNCH_CHECK();
  return KPO_OK;
  }
}
}  // namespace attn_tc

int attn_bwd_tcgen05_split(const void* q, const void* k, const void* v, const void* o, const void* dout,
                           const float* lse, float* dvec, void* dq, void* dk, void* dv, int64_t T, int hq, int hkv,
                           int d, int64_t qs, int64_t ks, int64_t vs, int64_t os, int64_t dqs, int64_t dks,
                           int64_t dvs, float scale, int causal, float* dkv_acc, int split_group, int qsplit_tiles,
                           int qchunks, cudaStream_t st, const float* rope_table) {
  if (d == 128)
    return attn_tc::bwd_split_launch<128>(q, k, v, o, dout, lse, dvec, dq, dk, dv, T, hq, hkv, qs, ks, vs, os, dqs,
                                          dks, dvs, scale, causal, dkv_acc, split_group, qsplit_tiles, qchunks, st,
                                          rope_table);
  if (d == 64 && rope_table == nullptr)
    return attn_tc::bwd_split_launch<64>(q, k, v, o, dout, lse, dvec, dq, dk, dv, T, hq, hkv, qs, ks, vs, os, dqs,
                                         dks, dvs, scale, causal, dkv_acc, split_group, qsplit_tiles, qchunks, st,
                                         rope_table);
  set_error("attn_bwd two-kernel path: head_dim 64 or 128 (fused rotary: 128)");
  return KPO_ERR_UNSUPPORTED;
}

// entry used by attention.cu's kpo_attn_fwd
int attn_fwd_tcgen05(const void* q, const void* k, const void* v, void* o, float* lse, int64_t T, int hq, int hkv,
                     int d, int64_t qs, int64_t ks, int64_t vs, int64_t os, float scale, int causal, cudaStream_t st) {
  if (d == 128) return attn_tc::fwd_launch<128>(q, k, v, o, lse, T, hq, hkv, qs, ks, vs, os, scale, causal, st);
  return attn_tc::fwd_launch<64>(q, k, v, o, lse, T, hq, hkv, qs, ks, vs, os, scale, causal, st);
}

int attn_bwd_tcgen05_main(const void* q, const void* k, const void* v, const void* dout, const float* lse,
                          const float* dvec, float* dq_acc, void* dk, void* dv, int64_t T, int hq, int hkv, int d,
                          int64_t qs, int64_t ks, int64_t vs, int64_t os, int64_t dks, int64_t dvs, float scale,
                          int causal, float* dkv_acc, int split_group, int qsplit_tiles, int qchunks,
                          cudaStream_t st, const float* rope_table) {
  if (d == 64) {
    if (rope_table != nullptr) {
      set_error("attn_bwd tcgen05 path: the fused inverse rotary needs head_dim 128");
      return KPO_ERR_UNSUPPORTED;
    }
    return attn_tc::bwd_launch<64>(q, k, v, dout, lse, dvec, dq_acc, dk, dv, T, hq, hkv, qs, ks, vs, os, dks, dvs,
                                   scale, causal, dkv_acc, split_group, qsplit_tiles, qchunks, st, rope_table);
  }
  if (d != 128) {
    set_error("attn_bwd tcgen05 path needs head_dim 64 or 128");
    return KPO_ERR_UNSUPPORTED;
  }
  return attn_tc::bwd_launch<128>(q, k, v, dout, lse, dvec, dq_acc, dk, dv, T, hq, hkv, qs, ks, vs, os, dks, dvs,
                                  scale, causal, dkv_acc, split_group, qsplit_tiles, qchunks, st, rope_table);
}

}  // namespace kpo
