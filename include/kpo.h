/*
 * kpo.h — C ABI of libkpo.so, the B200 (sm_100a) partitioned-overlap execution engine.
 *
 * The reference (schedfront, Kareus arXiv 2601.17654) has no native code: its hot path is the
 * Python simulator `simgpu.simulate_schedule` / `simgpu.measure`
 * (reference pkg/src/schedfront/simgpu.py:264-286 and :321-364), which turns an abstract
 * `PartitionSpec` (domain.py:201-229) of `KernelSpec`s (domain.py:165-198) plus a
 * `ScheduleConfig` (domain.py:145-162) into a `Measurement`.  This library supplies the real
 * kernels that an executed schedule launches in place of those abstract kernels:
 *
 *   abstract kernel (reference)                    entry point here
 *   ---------------------------------------------  -------------------------------------------
 *   "norm" / "fused_norm" (workloads.py:44,60,87)   kpo_rmsnorm_fwd / kpo_rmsnorm_bwd
 *   "linear_*" (workloads.py:45,48,61-62,73)        kpo_gemm (tcgen05 + TMEM + TMA)
 *   "rope" (workloads.py:46)                        kpo_rope (head_dim 64), fused into kpo_gemm_rope / kpo_attn_bwd_rope (128)
 *   "attention_core" (workloads.py:47)              kpo_attn_fwd / kpo_attn_bwd
 *   SwiGLU (memory-bound unit, compose.py:48-76)    kpo_swiglu_fwd / kpo_swiglu_bwd
 *   "allreduce" (workloads.py:50,64,74,90)          kpo_all_reduce      (SM-budgeted P2P)
 *   FSDP all-gather / reduce-scatter (north_star)   kpo_all_gather / kpo_reduce_scatter
 *   `comm_rate_bps(sm_count)` (simgpu.py:81-82)     the `ncta` argument of every collective
 *
 * Conventions:
 *   - every function returns an int status: KPO_OK (0) or a negative error class;
 *     kpo_last_error() returns a thread-local message for the last failure on this thread;
 *     nothing throws across the ABI;
 *   - all tensors are raw device pointers owned by the caller; sizes are element counts
 *     unless named *_bytes; streams are cudaStream_t passed as void*;
 *   - bf16 data is passed as void* (raw 16-bit bfloat16), fp32 as float*.
 */
#ifndef KPO_H
#define KPO_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define KPO_OK 0
#define KPO_ERR_INVALID (-1)     /* bad argument / shape / alignment                       */
#define KPO_ERR_CUDA (-2)        /* CUDA runtime or driver error                           */
#define KPO_ERR_UNSUPPORTED (-3) /* feature not available on this device / build           */
#define KPO_ERR_STATE (-4)       /* object used in the wrong state (e.g. peers not opened) */

/* ---------------------------------------------------------------- library */
const char* kpo_last_error(void);
int kpo_version(void);
/* Device facts the host-side GpuModel descriptor needs (simgpu.py:35-82 `num_sms`). */
int kpo_device_info(int device, int* num_sms, int* smem_optin_bytes, int* cc_major, int* cc_minor);

/* ---------------------------------------------------------------- memory-bound kernels */
/* y = x * rsqrt(mean(x^2) + eps) * w ; rstd[row] saved for backward.  x,y: [rows, cols] bf16. */
int kpo_rmsnorm_fwd(const void* x, const void* w, void* y, float* rstd, int64_t rows, int64_t cols,
                    float eps, void* stream);
/* dx = rmsnorm'(dy) (+ dres if non-null); dw_partial: [ceil(rows/rows_per_block) , cols] fp32 partial
 * sums reduced by kpo_colsum_f32 into dw (bf16).  rows_per_block is returned through *dw_rows. */
int kpo_rmsnorm_bwd(const void* dy, const void* x, const void* w, const float* rstd, const void* dres,
                    void* dx, float* dw_partial, int64_t rows, int64_t cols, void* stream);
int kpo_rmsnorm_bwd_partial_rows(int64_t rows, int64_t cols, int64_t* n_partials);
/* out[c] = sum_r in[r, c] (fp32 in, bf16 out). */
int kpo_colsum_f32_to_bf16(const float* in, void* out, int64_t rows, int64_t cols, void* stream);

/* Rotary embedding (Llama "rotate half" convention), theta base `theta`, position = pos0 + token.
 * in:  heads [tokens, heads, head_dim] addressed with in_row_stride elements between tokens;
 * out: same layout with out_row_stride.  inverse != 0 applies the transpose rotation (backward). */
int kpo_rope(const void* in, int64_t in_row_stride, void* out, int64_t out_row_stride, int64_t tokens,
             int heads, int head_dim, float theta, int64_t pos0, int inverse, void* stream);

/* SwiGLU on a fused gate|up buffer gu: [rows, 2*ffn] (gate = cols [0,ffn), up = [ffn,2ffn)).
 * act = silu(gate) * up : [rows, ffn]. */
int kpo_swiglu_fwd(const void* gu, void* act, int64_t rows, int64_t ffn, void* stream);
int kpo_swiglu_bwd(const void* dact, const void* gu, void* dgu, int64_t rows, int64_t ffn, void* stream);
/* The same on the blocked gate|up layout of kpo_gemm_swiglu: columns [2*b*block, 2*b*block + block) of
 * gu are gate block b, the next `block` columns the matching up block (block = 0: halves, as above). */
int kpo_swiglu_fwd_blocked(const void* gu, void* act, int64_t rows, int64_t ffn, int block, void* stream);
int kpo_swiglu_bwd_blocked(const void* dact, const void* gu, void* dgu, int64_t rows, int64_t ffn, int block,
                           void* stream);

/* ---------------------------------------------------------------- tensor-core GEMM (tcgen05) */
/* D[M,N] = A[M,K] * B[K,N]  (+ C[M,N] if C != NULL), bf16 in/out, fp32 accumulation in TMEM.
 *   a_mn_major = 0: A stored row-major [M][K] (K contiguous), lda >= K
 *   a_mn_major = 1: A stored as [K][M] (M contiguous),        lda >= M
 *   b_mn_major = 0: B stored as [N][K] (K contiguous, i.e. a torch Linear weight), ldb >= K
 *   b_mn_major = 1: B stored as [K][N] (N contiguous),         ldb >= N
 *   D, C: row-major [M][N] with leading dimension ldd (C shares ldd).
 * max_ctas: persistent grid cap (0 = all SMs).  sched: caller-owned device int32[2] tile-scheduler
 * word, zero-initialised once, reset by the kernel itself (one per concurrently running GEMM). */
int kpo_gemm(const void* A, const void* B, void* D, const void* C, int64_t M, int64_t N, int64_t K,
             int a_mn_major, int b_mn_major, int64_t lda, int64_t ldb, int64_t ldd, int max_ctas,
             int* sched, void* stream);

/* Forward (TN) GEMM whose output columns [0, rope_cols) are rotary-embedded in the epilogue:
 * heads of head_dim = 128 columns, pairs (i, i + 64) rotated by table[row][i] = (cos, sin), before the
 * bf16 rounding.  Fuses the reference's separate "rope" memory-bound KernelSpec (workloads.py:46)
 * into "linear_qkv" (workloads.py:45).  table: fp32 [M][head_dim/2][2] from kpo_rope_table. */
int kpo_gemm_rope(const void* A, const void* B, void* D, int64_t M, int64_t N, int64_t K, int64_t lda, int64_t ldb,
                  int64_t ldd, int max_ctas, int* sched, const float* rope_table, int64_t rope_cols, int head_dim,
                  void* stream);
/* gate|up projection with the SwiGLU fused into the epilogue: gu[M, N] = A[M, K] @ B[N, K]^T (bf16) and
 * act[M, N/2] = silu(gate) * up, where B's rows are 128-row gate / up blocks (gate block b = rows
 * [256b, 256b + 128), its up block the next 128; kpo_swiglu_*_blocked with block = 128 read gu in the
 * same order).  Fuses the reference's "swiglu" memory-bound KernelSpec into "linear_up"
 * (workloads.py:61-62).  CTA-pair 256x256 tiles: M >= 256, N % 256 == 0. */
int kpo_gemm_swiglu(const void* A, const void* B, void* gu, void* act, int64_t M, int64_t N, int64_t K, int64_t lda,
                    int64_t ldb, int64_t ldgu, int64_t ldact, int max_ctas, int* sched, void* stream);
/* down-projection dgrad with the SwiGLU backward fused into the epilogue: dact = dy[M, K] @ w[K, N]
 * (w = the down weight [hidden, ffn], MN-major B) is never written; per tile the epilogue TMA-loads the
 * matching gate / up boxes of gu (128-blocked order of kpo_gemm_swiglu, [M, 2N]) and writes
 * dgu [M, 2N] = (dact * u * sig(g) * (1 + g * (1 - sig(g))), dact * silu(g)) in the same order.
 * Fuses the reference's "swiglu" backward into "linear_down"'s dgrad (workloads.py:61-62).
 * CTA-pair 256x256 tiles: M >= 256, N % 256 == 0. */
int kpo_gemm_swiglu_bwd(const void* dy, const void* w, const void* gu, void* dgu, int64_t M, int64_t N, int64_t K,
                        int64_t lddy, int64_t ldw, int64_t ldgu, int64_t lddgu, int max_ctas, int* sched,
                        void* stream);
/* table[t][i] = (cos, sin)((pos0 + t) * theta^(-2i/head_dim)), fp32, t < tokens, i < head_dim/2. */
int kpo_rope_table(int64_t tokens, int head_dim, float theta, int64_t pos0, float* table, void* stream);

/* ---------------------------------------------------------------- attention */
/* Causal GQA flash attention, bf16 in/out, fp32 softmax statistics.
 * q: [T, hq, d] with token stride q_stride (elements), k/v: [T, hkv, d] with k_stride/v_stride,
 * o: [T, hq, d] with o_stride, lse: [hq, T] fp32 (natural-log logsumexp of scaled scores). */
int kpo_attn_fwd(const void* q, const void* k, const void* v, void* o, float* lse, int64_t T, int hq,
                 int hkv, int d, int64_t q_stride, int64_t k_stride, int64_t v_stride, int64_t o_stride,
                 float scale, int causal, void* stream);
/* The round-1 warp-level (mma.sync) forward, kept as a cross-check / A-B baseline for the
 * tcgen05 kernel behind kpo_attn_fwd.  Same arguments. */
int kpo_attn_fwd_mma(const void* q, const void* k, const void* v, void* o, float* lse, int64_t T, int hq,
                     int hkv, int d, int64_t q_stride, int64_t k_stride, int64_t v_stride, int64_t o_stride,
                     float scale, int causal, void* stream);
/* dq/dk/dv: same layouts as q/k/v (strides dq_stride, dk_stride, dv_stride).
 * workspace: fp32 scratch of kpo_attn_bwd_workspace_bytes(). */
int64_t kpo_attn_bwd_workspace_bytes(int64_t T, int hq, int hkv, int d);
int kpo_attn_bwd(const void* q, const void* k, const void* v, const void* o, const void* dout,
                 const float* lse, void* dq, void* dk, void* dv, int64_t T, int hq, int hkv, int d,
                 int64_t q_stride, int64_t k_stride, int64_t v_stride, int64_t o_stride,
                 int64_t dq_stride, int64_t dk_stride, int64_t dv_stride, float scale, int causal,
                 void* workspace, void* stream);

/* ---------------------------------------------------------------- non-partition work */
/* The work of a microbatch outside its partitions, which the reference costs analytically from
 * per-microbatch "non_partition_kernels" (reference pkg/src/schedfront/cli.py:171-175,227-241 ->
 * MicrobatchSpec.non_partition_costs, compose.py:79-102).  Here it is real kernels measured on the
 * hardware: embedding gather / scatter-add and the fused LM-head cross-entropy (the LM-head GEMMs
 * are kpo_gemm).  ids / labels are int32 [tokens]. */
/* out[t,:] = table[ids[t],:] (bf16, [vocab, hidden]); out-of-range ids give a zero row and set
 * *bad_flag (device int) to 1. */
int kpo_embedding_fwd(const int32_t* ids, const void* table, void* out, int64_t tokens, int64_t hidden,
                      int64_t vocab, int* bad_flag, void* stream);
/* dtable[ids[t],:] += dy[t,:] into an fp32 [vocab, hidden] gradient table (fp32 vector reductions;
 * repeated ids are summed in arbitrary order).  Out-of-range ids are skipped. */
int kpo_embedding_bwd(const int32_t* ids, const void* dy, float* dtable, int64_t tokens, int64_t hidden,
                      int64_t vocab, void* stream);
/* Fused softmax cross-entropy over bf16 logits [tokens, vocab] (row stride ld elements):
 * loss[t] = logsumexp(x_t) - x_t[labels[t]] (fp32, natural log), and
 * dlogits[t,:] = (softmax(x_t) - onehot(labels[t])) * grad_scale in bf16.  dlogits may alias logits.
 * Rows whose label == ignore_index (or is out of range) get loss 0 and zero gradients. */
int kpo_cross_entropy(const void* logits, void* dlogits, const int32_t* labels, float* loss, int64_t tokens,
                      int64_t vocab, int64_t ld, float grad_scale, int ignore_index, void* stream);

/* kpo_attn_bwd for q / k that were rotated by kpo_gemm_rope: dq and dk come out inverse-rotated
 * (gradients w.r.t. the un-rotated projections), fusing the reference's "rope" backward.  head_dim 128. */
int kpo_attn_bwd_rope(const void* q, const void* k, const void* v, const void* o, const void* dout,
                      const float* lse, void* dq, void* dk, void* dv, int64_t T, int hq, int hkv, int d,
                      int64_t q_stride, int64_t k_stride, int64_t v_stride, int64_t o_stride,
                      int64_t dq_stride, int64_t dk_stride, int64_t dv_stride, float scale, int causal,
                      void* workspace, const float* rope_table, void* stream);

/* ---------------------------------------------------------------- SM-budgeted collectives */
/* A communicator owns one symmetric buffer per rank (IPC-exported) plus per-CTA flag words.
 * world > 1, loopback == 0: one process per GPU; exchange kpo_comm_ipc_handle() blobs (out of band,
 *   e.g. torch.distributed all_gather_object) and pass all of them to kpo_comm_open_peers().
 * loopback != 0: `world` virtual ranks whose symmetric buffers all live on this device; the
 *   calling process plays rank `rank` and the virtual peers' data is whatever the caller wrote
 *   into their buffers (kpo_comm_peer_ptr).  Used for single-GPU execution and tests.
 * Collective inputs live in the symmetric buffer at byte offset `sym_off`; outputs are local. */
typedef struct kpo_comm kpo_comm;
#define KPO_IPC_HANDLE_BYTES 64
int kpo_comm_create(int rank, int world, int device, size_t sym_bytes, int loopback, kpo_comm** out);
int kpo_comm_ipc_handle(kpo_comm* c, void* handle_out /* KPO_IPC_HANDLE_BYTES */);
int kpo_comm_open_peers(kpo_comm* c, const void* handles /* world * KPO_IPC_HANDLE_BYTES */);
void* kpo_comm_sym_ptr(kpo_comm* c);                 /* this rank's symmetric buffer    */
void* kpo_comm_peer_ptr(kpo_comm* c, int peer);      /* peer's buffer as mapped here    */
int kpo_comm_max_ctas(kpo_comm* c);                  /* flag slots per rank             */
int kpo_comm_destroy(kpo_comm* c);

/* all-gather: out[p*bytes_per_rank ...] = sym_p[sym_off ...] for every rank p (pull model). */
int kpo_all_gather(kpo_comm* c, size_t sym_off, void* out, size_t bytes_per_rank, int ncta, void* stream);
/* reduce-scatter (bf16, fp32 accumulate in fixed rank order):
 *   out[i] = sum_p sym_p[sym_off + (rank*count + i)*2], i < count, count = elements per rank. */
int kpo_reduce_scatter(kpo_comm* c, size_t sym_off, void* out, size_t count_per_rank, int ncta, void* stream);
/* all-reduce (bf16, fp32 accumulate in fixed rank order), two-shot: reduce-scatter into
 * sym[stage_off] then all-gather; out[i] = sum_p sym_p[sym_off + 2i], count % world == 0. */
int kpo_all_reduce(kpo_comm* c, size_t sym_off, size_t stage_off, void* out, size_t count, int ncta,
                   void* stream);

/* ---------------------------------------------------------------- launch-order instrumentation */
/* Records, per CTA, the SM id and globaltimer at entry/exit of the next `n` comm launches into a
 * caller buffer (int64 [n_slots*4]); used by tests to prove the SM budget.  NULL disables. */
int kpo_comm_trace(kpo_comm* c, int64_t* buf, int n_slots);

/* Launch-completion ordering helper: launches the collective with
 * cudaLaunchAttributeLaunchCompletionEvent = `launched_event` (cudaEvent_t) so the compute stream
 * can wait until every comm CTA is resident before its next kernel is dispatched. */
int kpo_set_launch_completion_event(kpo_comm* c, void* launched_event);
/* Probe: launches one empty kernel with that attribute on `stream`, synchronizes and queries the
 * event.  Non-zero when the runtime (or a tool intercepting it) rejects the attribute; the executor
 * then forks the collective without the launch gate.  No reference counterpart (the simulator's
 * overlap starts instantly, simgpu.py:217-221). */
int kpo_probe_launch_completion(void* launched_event, void* stream);

/* SM blocker for solo-kernel timing at a reduced SM count (reference kernel_duration(k, f, sms),
 * simgpu.py:144-168, whose `sms` argument the executor realises as "the SMs the collective leaves"):
 * `ncta` CTAs that each hold a whole SM (full opt-in shared memory) spin for `spin_ns` on `stream`;
 * `launched_event` (cudaEvent_t, may be null) completes once all of them are resident. */
int kpo_sm_blocker(int ncta, int64_t spin_ns, void* launched_event, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* KPO_H */
