/*
 * infinigen_b200.h -- C ABI of the B200 decode-time KV path (InfiniGen,
 * arXiv 2406.19707).  Plain C types only; every call enqueues on the caller's
 * CUDA stream (passed as void*), never synchronises the host, never allocates
 * device memory, and returns an int status (IG_OK == 0).
 *
 * The reference exposes this path as Python operators that its engine imports
 * by name (reference: pkg/src/speckv/engine.py:27-38).  Each entry point below
 * names the reference interface it replaces; the Python shims in
 * paper_2406_19707_b200/ keep the reference signatures and map statuses back
 * to the reference exception classes (ValueError / IndexError /
 * ArtifactConsistencyError).
 *
 * Layouts (row-major, all per layer unless noted; Hg = heads on this GPU):
 *   host pool   T[B][Hg][S_max][2][d]      K row then V row, T = f32|f16|bf16
 *   partial K   f32[B][Hg][k][S_max]       column-major over tokens (coalesced)
 *   cols        i32[B][Hg][k]              ascending skewed-column indices
 *   scores      f32[B][Hg][S_max]
 *   idx         i32[B][Hg][cap]            selected rows, ascending
 *   stage       T[B][Hg][cap][2][d]        fetched rows in HBM
 *   pool meta   i64 arrival[B][Hg][S_max], i64 last_fetch[...], u8 counter[...]
 */
#ifndef INFINIGEN_B200_H
#define INFINIGEN_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  IG_OK = 0,
  IG_EINVAL = 1,        /* bad shape/argument  -> ValueError (speculation.py:51-54, 124-132) */
  IG_ERANGE = 2,        /* index out of range  -> IndexError (pool.py:91-92)                  */
  IG_ECONSISTENCY = 3,  /* pool / partial-K desync -> ArtifactConsistencyError (speculation.py:107-114) */
  IG_ENOMEM = 4,
  IG_ECUDA = 1000       /* IG_ECUDA + cudaError_t */
};

enum { IG_ELT_F32 = 0, IG_ELT_F16 = 1, IG_ELT_BF16 = 2 };
/* EvictionPolicy (pool.py:22-25) */
enum { IG_POLICY_FIFO = 0, IG_POLICY_LRU = 1, IG_POLICY_COUNTER = 2 };

/* Per-session decode position, resident in device memory so a whole decode
 * step can be enqueued (or graph-captured) without host round trips.
 *   s_len : pool rows before this step's append (len(pool), engine.py:329)
 *   limit : pool_limit, 0 = unlimited (engine.py:58, pool.py:61)
 *   seq   : KvPool._seq of every pool (pool.py:50-51); each decode step does
 *           one append (+1) and one fetch (+1) on every pool.             */
typedef struct ig_step_state {
  int32_t s_len;
  int32_t limit;
  int64_t seq;
  int32_t step;
  int32_t reserved;
} ig_step_state;

int ig_abi_version(void);
const char* ig_status_string(int status);

/* ---- host KV pool storage: replaces KvPool.keys/values (pool.py:37-38) ---- */
/* Pinned, mapped, portable host allocation; *dev_ptr is its device alias.   */
int ig_host_alloc(size_t bytes, void** host_ptr, void** dev_ptr);
int ig_host_free(void* host_ptr);
/* NUMA node holding the pool's first page (-1: unknown).  ig_host_alloc binds
 * the pool to the current GPU's NUMA node when the machine has several nodes
 * (mmap + mbind + cudaHostRegister; IG_HOST_NUMA=0: plain cudaHostAlloc). */
int ig_host_numa_node(const void* host_ptr, int* node);

/* ---- K1 rehearsal: replaces speculate_scores (speculation.py:117-135) -----
 * qspec = x_a(prev layer) @ W_Q(layer)[:, local heads] (f32[B][ldq]).  Per
 * (b, h): score[t] = (sum_j qspec[b, h*d + cols[j]] * pk[j][t]) * scale for
 * t < st->s_len, and maxkey[b,h] = max over t (order-preserving u32 key,
 * atomically max-reduced, so maxkey must be zeroed before the call).        */
int ig_rehearse(const float* qspec, int ldq, const int32_t* cols, const float* pk,
                const ig_step_state* st, int B, int Hg, int d, int k, int S_max,
                float scale, float* scores, uint32_t* maxkey, void* stream);

/* ---- K1+K2a fused (engine path): ig_rehearse + ig_count in one launch ----
 * The rehearsal tiles max-reduce into maxkey[b,h] and take a ticket; the last
 * tile of each (b, h) row counts score > float32(double(max) - alpha) over the
 * row and adds it to count_sum[b] (zero that first).  maxkey and tickets are
 * [B][Hg] scratch that must start zeroed and are left zeroed.  row_range
 * (optional, u32 [B][Hg][2]): that pass also records the row's maximum and
 * minimum score as order keys, which ig_select then takes instead of
 * scanning the row for them.                                                */
int ig_rehearse_count(const float* qspec, int ldq, const int32_t* cols, const float* pk,
                      const ig_step_state* st, int B, int Hg, int d, int k, int S_max,
                      float scale, double alpha, float* scores, uint32_t* maxkey,
                      int32_t* tickets, int32_t* counts, int32_t* count_sum, uint32_t* row_range,
                      void* stream);

/* Row maxima (as order keys) of scores not produced by ig_rehearse (the
 * select_tokens shim, speculation.py:156).                                  */
int ig_score_max(const float* scores, const ig_step_state* st, int B, int Hg, int S_max,
                 uint32_t* maxkey, void* stream);

/* ---- K2a count: select_tokens lines speculation.py:154-157 ---------------
 * counts[b,h] = #{t < s : score[t] > float32(double(max) - alpha)};
 * count_sum[b] += sum_h counts[b,h] (atomic; zero it first).               */
int ig_count(const float* scores, const uint32_t* maxkey, const ig_step_state* st,
             int B, int Hg, int S_max, double alpha, int32_t* counts,
             int32_t* count_sum, void* stream);

/* ---- K2b select: speculation.py:158-163 + topk_indices linalg.py:177-185 --
 * n[b] = min(clamp(floor(count_sum[b]/H_total + 0.5), min_select, cap), s),
 * cap = max(floor(cap_ratio*s), min_select); idx[b,h,0:n] = the top-n rows of
 * score[b,h] (ties -> lower index), written in ASCENDING row order.
 * If n would exceed cap_max (the buffer size) it is clamped and *err_flag set
 * to 1.  row_range (optional): the rows' (max, min) order keys as
 * ig_rehearse_count records them; NULL: computed here.                      */
int ig_select(const float* scores, const int32_t* count_sum, const ig_step_state* st,
              int B, int Hg, int H_total, int S_max, int cap_max, double cap_ratio,
              int min_select, int32_t* idx, int32_t* n_out, int32_t* err_flag,
              const uint32_t* row_range, void* stream);

/* Drop-in ordering: rewrite idx[b,h,0:n] in the reference's stable
 * descending-score order (linalg.py:184).  Used by the select_tokens shim,
 * not by the engine (the engine fetches in ascending order).              */
int ig_order_by_score(const float* scores, const int32_t* n, int B, int Hg,
                      int S_max, int cap, int32_t* idx, void* stream);

/* ig_select + ig_resident_plan of the same (b, h) in one launch (the plan runs
 * in the select's CTA on the selection it just wrote): same arguments as the
 * two calls, same results. */
int ig_select_plan(const float* scores, const int32_t* count_sum, const ig_step_state* st, int B,
                   int Hg, int H_total, int S_max, int cap_max, double cap_ratio, int min_select,
                   int32_t* idx, int32_t* n_out, int32_t* err_flag, const int32_t* pos_prev,
                   int32_t* slot_id, int32_t* slot_used, int32_t* frow, int32_t* fslot,
                   int32_t* fcount, int64_t* moved_rows, const uint32_t* row_range, void* stream);

/* Generic top-k per row (ties -> lower index), ascending output.  Used for
 * build_partial's column choice (speculation.py:41-58).                   */
int ig_topk_rows(const float* values, int rows, int len, int k, int32_t* idx_out,
                 void* stream);

/* ---- K3 fetch: replaces KvPool.fetch's gather (pool.py:83-99) ------------
 * Zero-copy SM gather of the selected rows from the mapped host pool into
 * stage.  pool_dev = device alias of this layer's T[B][Hg][S_max][2][d].   */
int ig_fetch(const void* pool_dev, const int32_t* idx, const int32_t* n, int B, int Hg,
             int S_max, int cap, int row_bytes, void* stage, int ctas, int threads,
             void* stream);   /* threads per CTA: 256, 512 or 1024 */
/* Same gather with TMA bulk copies (host -> smem -> HBM): `warps` (1-4) warps
 * per CTA; each warp moves `rows_per_batch` (<= 32) rows per batch, one per
 * lane, with two batches loading while the previous one drains (shared memory
 * warps * 3 * rows_per_batch * row_bytes).  The bytes in flight live in shared
 * memory, so the gather takes almost no threads/registers from compute.
 * idx == NULL: every row [0, st->s_len) of every (b, h) (a full layer whose
 * size is read on the device -- CUDA-graph capturable; st unused otherwise). */
int ig_fetch_tma(const void* pool_dev, const int32_t* idx, const int32_t* n,
                 const ig_step_state* st, int B, int Hg, int S_max, int cap, int row_bytes,
                 void* stage, int ctas, int warps, int rows_per_batch, void* stream);
/* Layer 0 (engine.py:393-396): every row [0, s) by copy engine, host sizes. */
int ig_fetch_all(const void* pool_host, int B, int Hg, int S_max, int s, int row_bytes,
                 void* stage, int stage_rows, void* stream);

/* ---- K5 append: KvPool.append (pool.py:53-81) + evict_select (:101-109) +
 * append_partial_key (speculation.py:92-114) + the fetch-metadata update of
 * KvPool.fetch (pool.py:93-98) for this layer's fetch set.
 * Per (b, h): pos = s (below limit) or the policy victim; the new K/V row is
 * stored to the host pool, k_cur[cols] into pk[:, pos], metadata reset to
 * seq+1; then (fetch_mode 1) every row, or (fetch_mode 2) the selection
 * idx[0:n] plus pos deduplicated (engine.py:449-453), gets last_fetch = seq+2
 * and a saturating counter bump with "any counter hit 255 -> halve all";
 * fetch_mode 0 is a plain KvPool.append.  pos_out[b,h] receives pos;
 * events[b,h] = {victim, old arrival} on overwrite else {-1, 0}.            */
int ig_append(const float* k_cur, const float* v_cur, int ldkv, void* pool_dev, int elt,
              float* pk, const int32_t* cols, int k, int64_t* arrival, int64_t* last_fetch,
              uint8_t* counter, int policy, int fetch_mode, const int32_t* idx,
              const int32_t* n, int cap, const ig_step_state* st, int B, int Hg, int d,
              int S_max, int32_t* pos_out, int64_t* events, void* stream);

/* KvPool.evict_select (pool.py:101-109) alone: victim[b,h] = argmin over
 * [0, st->s_len) of the policy key, lowest index on ties.                  */
int ig_evict_select(const int64_t* arrival, const int64_t* last_fetch, const uint8_t* counter,
                    int policy, const ig_step_state* st, int B, int Hg, int S_max,
                    int32_t* victim, void* stream);

/* KvPool.fetch metadata alone (pool.py:93-98): rows idx[b,h,0:n[b]] (unique)
 * get last_fetch = seq and a saturating counter bump; halve-all over
 * [0, st->s_len) if any reaches 255.                                       */
int ig_touch(const int32_t* idx, const int32_t* n, int cap, const ig_step_state* st, int B,
             int Hg, int S_max, int64_t seq, int64_t* last_fetch, uint8_t* counter,
             void* stream);

/* ---- K4 attend: replaces attention_head on the fetched set (model.py:156-180,
 * engine.py:352-358).  Per (b, h): softmax((q . K^T) / float32(sqrt(d))) . V
 * over stage rows r < n (n == NULL -> s rows, idx == NULL -> row r) whose row
 * index != pos, plus the GPU-resident current row (k_cur, v_cur).  pos ==
 * NULL means pos = st->s_len for every (b, h) (the append position when no
 * pool limit applies).  Split over row chunks; partial/ticket are scratch
 * sized by ig_attend_scratch.                                              */
int ig_attend_scratch(int B, int Hg, int d, int cap, size_t* partial_floats,
                      size_t* tickets);
int ig_attend(const float* q, int ldq, const float* k_cur, const float* v_cur, int ldkv,
              const void* stage, int elt, const int32_t* idx, const int32_t* n,
              const int32_t* pos, const ig_step_state* st, int B, int Hg, int d, int cap,
              float* partial, int32_t* tickets, float* out, int ldo, void* stream);

/* ---- resident selection (B200 extension of K3/K4) ----------
 * The fetched set of each speculative layer stays in HBM across decode steps
 * in a slot table: stage T[B][Hg][cap][2][d], slot_id i32[B][Hg][cap] (row
 * index held by the slot, -1 = empty), slot_used i32[B][Hg] (slots in use).
 * Only rows that enter the selection are fetched from the host pool, which
 * stays authoritative (the reference refetches every selected row each step,
 * pool.py:83-99 via engine.py:352-356; same rows, fewer link bytes).
 *
 * ig_resident_plan, per (b, h): free every slot whose row is not in the new
 * ascending selection idx[b,h,0:n[b]] or equals pos_prev[b,h] (the row last
 * step's append overwrote; NULL = none), then give the selected rows that are
 * not resident the free slots in ascending order (then slots from slot_used
 * up): fetch list frow/fslot i32[B][Hg][cap], fcount i32[B][Hg].  moved_rows
 * (nullable) accumulates the fetched row count.  Shared memory 5*cap bytes.
 * ig_fetch_slots: stage[b,h,fslot[k]] = pool[b,h,frow[k]] for k < fcount.
 * ig_stage_put: stage[b,h,pos[b,h]] = (k_cur, v_cur) rounded to `elt` exactly
 * like ig_append (layer 0's full mirror, stage rows per (b, h) = stage_rows).
 * ig_attend_slots: ig_attend over slots r < slot_used[b,h] whose id >= 0 and
 * != pos, plus the current row.                                            */
int ig_resident_plan(const int32_t* idx, const int32_t* n, const int32_t* pos_prev,
                     int32_t* slot_id, int32_t* slot_used, int B, int Hg, int cap, int32_t* frow,
                     int32_t* fslot, int32_t* fcount, uint64_t* moved_rows, void* stream);
int ig_fetch_slots(const void* pool_dev, const int32_t* frow, const int32_t* fslot,
                   const int32_t* fcount, int B, int Hg, int S_max, int cap, int row_bytes,
                   void* stage, void* stream);
int ig_stage_put(const float* k_cur, const float* v_cur, int ldkv, const int32_t* pos, void* stage,
                 int elt, int B, int Hg, int d, int stage_rows, void* stream);
int ig_attend_slots(const float* q, int ldq, const float* k_cur, const float* v_cur, int ldkv,
                    const void* stage, int elt, const int32_t* slot_id, const int32_t* slot_used,
                    const int32_t* pos, const ig_step_state* st, int B, int Hg, int d, int cap,
                    float* partial, int32_t* tickets, float* out, int ldo, void* stream);

/* Strided 2-D copy between any UVA addresses (cudaMemcpyDefault): used to
 * write prefill K/V rows into the host pool (engine.py:265-266).          */
int ig_memcpy2d(void* dst, size_t dpitch, const void* src, size_t spitch, size_t width,
                size_t height, void* stream);

/* ---- dense projections of the decode step (engine.py:323-327, 360-364) ----
 * Y[M][N] = X[M][K] . W[K][N], M <= 32 (sequences); epilogue 0 = none,
 * 1 = ReLU, 2 = Y = R + X.W (residual).  f32-level split precision on the
 * tensor cores over weights PACKED once at load time (ig_sgemm_pack: 32-KB
 * blocks in MMA-fragment order, f16 hi/lo pairs -- 11 + 11 significand bits;
 * x split the same way in registers; x.w = hi.hi + (hi.lo + lo.hi) with f32
 * accumulation), contiguous in (column tile, row block) order -- the whole GEMM
 * is one sequential stream.  Persistent stream-K grid:
 * ig_sgemm_packed_sizes gives the packed buffer (floats), the workspace
 * (floats) and ticket (ints, zeroed once, left zeroed) sizes for (M, N, K).
 * X 16-B aligned, ldx and K multiples of 4.  Deterministic on a given device. */
int ig_sgemm_packed_sizes(int M, int N, int K, size_t* packed_floats, size_t* workspace_floats,
                          size_t* tickets);
int ig_sgemm_pack(const float* W, int ldw, int N, int K, float* packed, void* stream);
int ig_sgemm_packed(const float* X, int ldx, const float* packed, int N, int K, float* Y, int ldy,
                    const float* R, int ldr, int M, int epilogue, float* workspace,
                    size_t workspace_floats, int32_t* tickets, size_t ntickets, void* stream);

/* ---- head-parallel output all-reduce over peer memory (N > 1) ----------
 * Replaces the NCCL all-reduce of the row-parallel W_O / FFN-out partials
 * (engine.py:360-364 sums over all heads).  Each rank allocates a receive
 * buffer (2 x world x n 4-B elements) and flags (2 x world u32 + a 16-B ticket) with
 * ig_peer_alloc, shares them by CUDA IPC (ig_ipc_get_handle / _open_handle;
 * 64-B handles), and passes device arrays of the world's receive / flag base
 * pointers.  ig_allreduce_peer pushes `src` (n floats) into every rank's slot,
 * raises its flag, waits for all ranks and writes out = sum over ranks (rank
 * order, identical bits on every rank) + residual (may be NULL).  `call` in
 * [0, calls_per_step) numbers the all-reduces of one step (epoch from
 * st->step: graph-replayable); ticket = flags + 2 * world (u32).          */
int ig_peer_alloc(int n, int world, void** recv, void** flags);
int ig_peer_free(void* recv, void* flags);
int ig_ipc_get_handle(void* dev_ptr, void* handle64);
int ig_ipc_open_handle(const void* handle64, void** dev_ptr);
int ig_ipc_close(void* dev_ptr);
int ig_allreduce_peer(const float* src, int n, const uint64_t* peer_recv, const uint64_t* peer_flags,
                      int rank, int world, const ig_step_state* st, int call, int calls_per_step,
                      const float* residual, float* out, uint32_t* ticket, void* stream);
/* The collective's push folded into the producer: ig_sgemm_packed_peer runs the
 * packed GEMM (epilogue 0) and writes its final values into slot
 * [parity][rank] of every rank's receive buffer (n = M * N, row-major) and
 * raises this rank's flags when the whole grid is done (`done`: a u32 counter,
 * zeroed once, left zeroed -- flags + 2 * world + 1); ig_allreduce_peer_sum
 * then waits and sums (+ residual) without a push phase. */
int ig_sgemm_packed_peer(const float* X, int ldx, const float* packed, int N, int K, int M,
                         const uint64_t* peer_recv, const uint64_t* peer_flags, int rank, int world,
                         const ig_step_state* st, int call, int calls_per_step, uint32_t* done,
                         float* workspace, size_t workspace_floats, int32_t* tickets,
                         size_t ntickets, void* stream);
int ig_allreduce_peer_sum(int n, const uint64_t* peer_recv, const uint64_t* peer_flags, int rank,
                          int world, const ig_step_state* st, int call, int calls_per_step,
                          const float* residual, float* out, void* stream);
/* The same for the per-sequence int32 head-count sums (speculation.py:154-158:
 * n averages over ALL heads); no residual. */
int ig_allreduce_peer_i32(const int32_t* src, int n, const uint64_t* peer_recv,
                          const uint64_t* peer_flags, int rank, int world, const ig_step_state* st,
                          int call, int calls_per_step, int32_t* out, uint32_t* ticket, void* stream);

/* ---- step bookkeeping -------------------------------------------------- */
/* s_len = min(s_len + 1, limit), seq += 2, step += 1 (engine.py:377-378). */
int ig_step_advance(ig_step_state* st, void* stream);

/* Reference layernorm (linalg.py:50-69): (x-mean)/sqrt(var+eps)*g+b, f32. */
int ig_layernorm(const float* x, const float* gain, const float* bias, float eps,
                 int rows, int D, float* out, void* stream);

/* ---- prefill projections on tcgen05 -------------
 * The prompt-length GEMMs of DecodeSession._prefill / forward_block
 * (engine.py:245-291, model.py:195-244: x_a @ W_QKV, attn @ W_O, the FFN) at
 * f32-level accuracy on the 5th-generation tensor cores.  Operands are split
 * once into f16 hi/lo pairs with a power-of-two scale per operand row
 * (ig_split_f16: out [rows][2 Kp] f16 = hi in [0, Kp), lo in [Kp, 2 Kp),
 * Kp = K rounded up to 64; transpose = 1 takes W [K][N] and emits W^T rows),
 * then ig_gemm_tc05 computes C = A @ W (+ ReLU, epilogue 1 / + R, epilogue 2)
 * as hi.hi + hi.lo + lo.hi accumulated in f32 in TMEM (tcgen05.mma kind::f16,
 * TMA-fed 128-B-swizzled tiles).  max_ctas <= 0: one CTA per SM. */
int ig_split_f16(const float* X, int ldx, int rows, int cols, int transpose, int Kp, void* out,
                 float* inv_scale, void* stream);
int ig_gemm_tc05(const void* A_hl, const float* inv_sa, const void* B_hl, const float* inv_sb, int M,
                 int N, int K, int Kp, float* C, int ldc, const float* R, int ldr, int epilogue,
                 int max_ctas, void* stream);

/* Prefill causal attention on tcgen05 (model.py:156-180 causal, as used by
 * forward_block model.py:195-244 in DecodeSession._prefill engine.py:245-291):
 * qkv [nb N][ldqkv] f32 rows of (q | k | v) over Hg heads of d (64 or 128);
 * out [nb N][ldo] f32, head h at columns [h d, (h+1) d).  q, k, v and p are
 * split exactly into f16 hi/lo pairs (work: ig_prefill_attention_scratch bytes). */
int ig_prefill_attention_scratch(int nb, int N, int Hg, int d, size_t* bytes);
int ig_prefill_attention(const float* qkv, int ldqkv, int nb, int N, int Hg, int d, void* work,
                         float* out, int ldo, void* stream);

/* ---- diagnostics --------------------------------------------------------
 * ig_debug_attend_trace: device buffer (u64, >= grid x (8 + 6 x 64)) that the
 * tcgen05 attention fills with %globaltimer stamps per role and tile
 * (tools/attend_trace.py); NULL switches it off (the default). */
int ig_debug_attend_trace(void* buf);

#ifdef __cplusplus
}
#endif
#endif /* INFINIGEN_B200_H */
