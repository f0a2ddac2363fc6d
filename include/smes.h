/*
 * smes.h -- C ABI of the B200-native SMES layer (arXiv 2602.09386) hot path.
 *
 * The reference (taskmoe 0.1.0) exposes this path as NumPy functions, not an
 * FFI; each entry point below replaces one reference function (file:line in
 * /root/reference/pkg/src/taskmoe) and is what a ctypes / cffi binding of the
 * reference's module API binds to.
 *
 * Conventions
 *   - plain device pointers + sizes; no torch types; `stream` is a cudaStream_t.
 *   - functions never allocate; the caller passes outputs and workspaces.
 *   - every launch is stream-ordered and host-sync free (CUDA-graph capturable);
 *     data-dependent sizes (N_act, segment offsets) stay on the device.
 *   - return 0 on success, else an SMES_ERR_* code; smes_last_error() gives the
 *     message.  Codes map 1:1 to taskmoe.errors (errors.py:4-49).
 *   - bf16 = __nv_bfloat16 storage, fp32 accumulation.  Deterministic: no
 *     floating-point atomics, fixed reduction orders.
 */
#ifndef SMES_H_
#define SMES_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SMES_ABI_VERSION 1

#define SMES_OK 0
#define SMES_ERR_SHAPE 1    /* taskmoe.errors.ShapeError    */
#define SMES_ERR_CONFIG 2   /* taskmoe.errors.ConfigError   */
#define SMES_ERR_NUMERICS 3 /* taskmoe.errors.NumericsError */
#define SMES_ERR_STATE 4    /* taskmoe.errors.StateError    */
#define SMES_ERR_CUDA 5     /* CUDA runtime / driver failure */

const char* smes_last_error(void);
int smes_abi_version(void);

/* ---- K1 progressive router: replaces route_batch (routing.py:235-281) incl.
 *      softmax (linalg.py:74-83), _top_k_rows (routing.py:184-187) and
 *      _renormalized_weights_batch (routing.py:203-211); fuses the per-chunk
 *      histograms of build_execution_plan (execution.py:109) and
 *      compute_load_stats (balance.py:65-68).  Stage I in fp64.
 *      z element (t,b,e) at z[t*stride_t + b*stride_b + e].  frozen = 1 reuses the selections in
 *      shared/adaptive and recomputes weights + statistics (model.py:284-300). */
int smes_route_rows_per_warp(int B);
int smes_route_num_chunks(int B, int rows_per_warp);
int smes_route_batch(const float* z, long stride_t, long stride_b, const double* probs_in,
                     const double* task_weights, int T, int B, int E, int k_shared, int k_adaptive,
                     int rows_per_warp, int32_t* shared, int32_t* adaptive, int32_t* active, float* wsel,
                     uint32_t* umask, int32_t* usize, int32_t* chunk_union, int32_t* chunk_active,
                     double* chunk_mass, double* chunk_dmass, double* probs_out, int32_t* flag, int frozen,
                     void* stream);

/* ---- K0+K1 fused router front: RouterBank.logits (routing.py:101-103, via Affine.apply
 *      linalg.py:143-149) on the tensor cores, feeding route_batch (routing.py:235-281) straight
 *      from TMEM, two threads per row.  Same outputs as smes_route_batch (per-chunk histograms
 *      over chunks of sub_rows = 4 * rows_per_warp rows).  Stage I: fp32 exponentials with fp64
 *      sums and a certified error bound; rows whose shared set the bound cannot decide are
 *      recomputed entirely in fp64, so the selections equal an fp64 Stage I.  z_out
 *      (B, T*E) fp32 is optional; chunk_dmass may be null (dense mass not computed).
 *      h (B, ldh) bf16, w_r (T*E, d) bf16, b_r (T*E) fp32.  Supported shapes: see
 *      smes_route_front_supported (E in {16, 32}, T*E <= 256, d in {64, ..., 256}, budget 4+2 or 2+1). */
int smes_route_front_supported(int T, int E, int d, int k_shared, int k_adaptive);
int smes_route_front(const void* h, long ldh, const void* w_r, const float* b_r, const double* task_weights,
                     int T, int B, int E, int d, int k_shared, int k_adaptive, int sub_rows, int32_t* shared,
                     int32_t* adaptive, int32_t* active, float* wsel, uint32_t* umask, int32_t* usize,
                     int32_t* chunk_union, int32_t* chunk_active, double* chunk_mass, double* chunk_dmass,
                     int32_t* flag, float* z_out, void* stream);
/* ---- K1 (row, task) router: smes_route_batch in training / scoring mode (not frozen, no dense
 *      probabilities in or out, chunk_dmass NULL) for E in {16, 32, 64}, T <= min(32, E), budget 4+2
 *      or 2+1 -- smes_route_batch dispatches here itself.  Thread per (row, task); Stage I in fp32
 *      with a certified bound and an fp64 recompute of undecidable rows (selections as fp64). */
int smes_route_rt_supported(int T, int E, int k_shared, int k_adaptive);
int smes_route_rt(const float* z, long stride_t, long stride_b, const double* task_weights, int T, int B, int E,
                  int k_shared, int k_adaptive, int rows_per_warp, int32_t* shared, int32_t* adaptive,
                  int32_t* active, float* wsel, uint32_t* umask, int32_t* usize, int32_t* chunk_union,
                  int32_t* chunk_active, double* chunk_mass, double* chunk_dmass, int32_t* flag, void* stream);
void smes_route_count_exact(int32_t* dev_counter);

/* diagnostic: count (atomically, into *dev_counter) the rows later smes_route_front launches send
 * through the fp64 recompute; NULL turns counting off. */
void smes_route_front_count_exact(int32_t* dev_counter);

/* ---- combine backward from a given upstream gradient of the task reps (the autograd form of the
 *      layer, SMESLayer): training.py:160-179 with d_reps (T, B, d_out) fp32 in place of
 *      dlogit x head_w, plus the sparse-reading LB term lb_coef * w (f - <w, f>) (balance.py:83-99).
 *      Writes d_packed (rows, ldo) bf16 (x relu mask of O when relu_last) and the full dz rows
 *      (B, ldz) bf16, zero off the active sets.  Deterministic (fixed-order sums). */
int smes_combine_bwd_reps(int T, int B, int E, int K, int d_out, int umax, const uint32_t* umask,
                          const int32_t* usize, const int32_t* row_of, const int32_t* active, const float* wsel,
                          const void* O, long ldo, int relu_last, const float* d_reps, const float* freq,
                          float lb_coef, void* dpacked, void* dz, long ldz, void* stream);

/* ---- one-shot all-reduce of a small f64 vector over CUDA-IPC-mapped peer memory (NVLink): the
 *      data-parallel exchange of the 3E LoadStats sums (balance.py:62-70).  recv buffers are
 *      [2][n][count] f64 on every rank, flags [n] int32, epoch_ctr 1 int32 (device-side epoch:
 *      graph capturable).  out may alias in.  Result: sum in rank order, identical on every rank. */
int smes_peer_allreduce_f64(int n, int me, int count, const double* in, void* const* peer_recv_dev,
                            int32_t* const* peer_flags_dev, const double* my_recv, int32_t* my_flags,
                            int32_t* epoch_ctr, double* out, void* stream);

/* ---- K2 execution plan: replaces build_execution_plan (execution.py:85-123)
 *      and the gather hidden[plan.gather_instances] (model.py:301).
 *      Segments are padded to 128 rows (seg_pad); seg_log are the reference's
 *      segment_offsets.  totals = {0, padded rows, N_act}.  seg_half (optional, 2E+1) splits
 *      every padded segment into two 64-row-aligned halves (split-K tables). */
int smes_plan_reduce(int C, int E, const int32_t* chunk_union, const int32_t* chunk_active,
                     const double* chunk_mass, const double* chunk_dmass, int32_t* chunk_base, int32_t* loads,
                     double* stats_raw, int32_t* seg_pad, int32_t* seg_log, int32_t* totals,
                     unsigned int* ticket, int32_t* seg_half, void* stream);
/* smes_plan_reduce + the LoadStats finalize of smes_stats_finalize in the same launch, for steps
 * with no cross-device exchange of the raw sums in between (single GPU). */
int smes_plan_reduce_stats(int C, int E, const int32_t* chunk_union, const int32_t* chunk_active,
                           const double* chunk_mass, const double* chunk_dmass, int32_t* chunk_base, int32_t* loads,
                           double* stats_raw, int32_t* seg_pad, int32_t* seg_log, int32_t* totals,
                           unsigned int* ticket, int32_t* seg_half, int K, int lb_experts, double batch_times_tasks,
                           int dense, double* stats_out, float* freq_f32, void* stream);
/* int32 elements of the ``ticket`` work buffer smes_plan_reduce / smes_plan_reduce_stats need
 * (zero-initialised once by the caller; the kernels keep it replay-safe themselves). */
int smes_plan_reduce_work_ints(int C, int E);
/* plan reduce + LoadStats finalize (as smes_plan_reduce_stats) and the head fold of a training
 * step (as smes_fold_heads) in one launch, for the shapes smes_fold_full_supported accepts (the
 * fold's blocks run in the slack of the reduce's E column-scan blocks). */
int smes_fold_full_supported(int E, int T, int ldg, int d_out, int d_in);
int smes_plan_reduce_stats_fold(int C, int E, const int32_t* chunk_union, const int32_t* chunk_active,
                                const double* chunk_mass, const double* chunk_dmass, int32_t* chunk_base,
                                int32_t* loads, double* stats_raw, int32_t* seg_pad, int32_t* seg_log, int32_t* totals,
                                unsigned int* ticket, int32_t* seg_half, int K, int lb_experts,
                                double batch_times_tasks, int dense, double* stats_out, float* freq_f32, int T,
                                int ldg, int d_out, int d_in, const float* head_w, const void* W, const float* b,
                                void* G, float* c, void* stream);
int smes_plan_counts(int B, int E, int rows_per_warp, const uint32_t* umask, int32_t* chunk_union, int32_t* usize,
                     void* stream);
int smes_plan_scatter(int B, int E, int d, int rows_per_warp, const uint32_t* umask, const int32_t* chunk_base,
                      const int32_t* seg_pad, const int32_t* loads, const void* h_bf16, long ldh, void* X_bf16,
                      long ldx, int32_t* row_of, int umax, int32_t* gather_inst, int32_t* gather_exp,
                      void* zero_rows2_bf16, long ldz2, int d2, void* stream);

/* ---- K3 grouped GEMM (tcgen05 + TMEM + TMA): replaces grouped_gemm
 *      (execution.py:126-158) and the expert part of backward (training.py:180-191).
 *      ragged-M: C[m,n] = act(sum_k A[m,k] W_g[n,k] + bias_g[n])   (b_mn = 0, fwd)
 *                C[m,n] = mask(sum_k A[m,k] W_g[k,n])              (b_mn = 1, dgrad)
 *      ragged-K: C_g[i,j] = sum_{m in g} P[m,i] Q[m,j]           (wgrad, fp32 out)
 *                db_g[i]  = sum_{m in g} P[m,i]   when db_out != NULL (G, I): an extra N=16 MMA per
 *                K-step against a constant ones tile in smem, inside the j0 = 0 output tiles.
 *      seg = padded group offsets (device). */
int smes_gemm_ragged_m(const void* A, long lda, long rows_cap, const void* W, int G, int N, int K, int b_mn,
                       const int* seg, const float* bias, int act, uint32_t* relu_bits_out,
                       const uint32_t* relu_bits_in, long bits_ld, void* C, long ldc, int out_fp32,
                       long m_limit, void* stream);
int smes_gemm_ragged_k(const void* P, long ldp, const void* Q, long ldq, long rows_cap, int G, int I, int J,
                       const int* seg, float* C, float* db_out, void* stream);
/* ragged-K with one P shared by every group: P row m is read as row (m % a_period) of a
 * (p_rows, I) matrix (a_period a multiple of 64; 0 = ordinary ragged-K). */
int smes_gemm_ragged_k_periodic(const void* P, long ldp, long p_rows, const void* Q, long ldq, long rows_cap, int G,
                                int I, int J, const int* seg, float* C, float* db_out, int a_period, void* stream);
/* ragged-K with Q gathered: packed row r of Q is row gather[r] of src ((n_src, ld_src) bf16; -1 =
 * a zero row), read by TMA gather4 -- the packed copy of the layer input (the reference's
 * `hidden[plan.gather_instances]`, model.py:301) is never written (the fc1 weight gradient,
 * training.py:184-191).  gather: rows_cap int32, 16-byte aligned. */
int smes_gemm_ragged_k_gather(const void* P, long ldp, const void* src, long ld_src, long n_src, const int32_t* gather,
                              long rows_cap, int G, int I, int J, const int* seg, float* C, float* db_out,
                              void* stream);

/* ragged-K with the K range of every group split into `splits` contiguous parts (more work units
 * than SMs for few, long groups): fp32 partials in `work` (smes_gemm_ragged_k_split_work floats),
 * then summed over the splits in order into C (and db_out). */
long smes_gemm_ragged_k_split_work(int G, int I, int J, int splits, int with_db);
int smes_gemm_ragged_k_split(const void* P, long ldp, const void* Q, long ldq, long rows_cap, int G, int I, int J,
                             const int* seg, float* C, float* db_out, int splits, float* work, void* stream);

/* ---- K4 combine + heads + BCE: replaces reconstruct_task_reps (execution.py:161-191),
 *      _heads (model.py:202-208) and _weighted_bce (training.py:54-57). */
int smes_combine_grid(int B, int T, int d_out);
int smes_combine_fwd(int T, int B, int E, int K, int d_out, int umax, const uint32_t* umask, const int32_t* usize,
                     const int32_t* row_of, const int32_t* active, const float* wsel, const void* O, long ldo,
                     const float* head_w, const float* head_b, const float* P, long ldp, void* reps, float* logits, float* preds,
                     const float* labels, const float* lam, double* loss_part, int grid, void* stream);

/* ---- K6+K7 heads/combine backward + LB gradient: replaces backward
 *      (training.py:146-179) and lb_loss_gradient (balance.py:83-99). */
int smes_combine_bwd(int T, int B, int E, int K, int d_out, int umax, const uint32_t* umask, const int32_t* usize,
                     const int32_t* row_of, const int32_t* active, const float* wsel, const void* O, long ldo,
                     const float* head_w, const float* P, long ldp, const void* reps, const float* preds,
                     const float* labels, const float* lam, float inv_b, int relu_last, void* dpacked, void* dz,
                     const float* freq, float lb_coef, int dense_probs, const float* z, float* part_dw,
                     float* part_db, int grid, void* stream);

/* ---- K4+K6+K7 for a training step (sparse LB reading): logits/preds/loss from the head
 *      projections P, dlogit, the (row, task) coefficient matrix C = w * dlogit (bf16) and the
 *      router-logit gradient dz (training.py:146-179, balance.py:83-99).  The dense parts,
 *      d_packed = C head_W and dW_head = C^T O, are tcgen05 GEMMs (smes_gemm_*). */
int smes_combine_train(int T, int B, int E, int K, int umax, const uint32_t* umask, const int32_t* usize,
                       const int32_t* row_of, const int32_t* active, const float* wsel, const float* head_b,
                       const float* P, long ldp, float* logits, float* preds, const float* labels, const float* lam,
                       double* loss_part, float inv_b, void* cmat, long ldc, void* dz, const float* freq,
                       float lb_coef, float* part_db, float* part_csum, float* part_rb, int grid, void* stream);
/* last-pool bias grad when the last pool is identity: db[e] = (sum_rows_of_e C) head_W. part_csum
 * (grid, E, T) and part_rb (grid, T*E: router bias grad = column sums of dz) are per-CTA partials
 * from smes_combine_train (optional, may be NULL). */
int smes_bias_from_csum(int E, int T, int d_out, const float* csum, const float* head_w, float* out, void* stream);

/* ---- head folding for the training step when the last expert pool is the identity
 *      (model.py:202-208 composed with execution.py:126-158; backward training.py:146-191):
 *      G (E, ldg, d_in) bf16 = head_w W_e (rows >= T zero), c (E, ldg) = head_w b_e, so the head
 *      projections are P = H G_e^T + c_e (an N = ldg GEMM) and d_packed never materialises.
 *      smes_unfold_grads expands Q = per-expert C^T H (element (e, t, k) at e*q_expert_stride +
 *      t*q_task_stride + k*q_k_stride: (E, ldg, d_in) or (E, d_in(+1), ldg) layouts) and
 *      csum (per-expert column sums of C) into dW = head_w^T Q_e, db = head_w^T csum_e and
 *      dW_head = sum_e (Q_e W_e^T + csum_e b_e^T).  Large banks (E*d_out*d_in >= 2^24) run both as
 *      grouped tcgen05 GEMMs (Q split into bf16 hi + lo rows), small ones as split-K CUDA-core tiles.
 *      work: fp32 scratch of smes_fold_work_floats(E, T, d_out, d_in) floats (split-K partials). */
int smes_fold_work_floats(int E, int T, int d_out, int d_in);
int smes_fold_gemm_path(int E, int T, int d_out, int d_in);   /* 1: tensor-core fold/unfold path */
int smes_fold_heads(int E, int T, int ldg, int d_out, int d_in, const float* head_w, const void* W_bf16,
                    const float* b, void* G_bf16, float* c, float* work, void* stream);
int smes_unfold_grads(int E, int T, int ldg, int d_out, int d_in, const float* Q, long q_expert_stride,
                      long q_task_stride, long q_k_stride, const float* csum, long csum_expert_stride,
                      const float* head_w, const void* W_bf16,
                      const float* b, float* dW, float* db, float* work, float* d_head_w, void* stream);

/* ---- fused expert MLP for training steps (csrc/mlp.cu): two chained tcgen05 MMAs per 128-row
 *      tile with the d_ff-wide intermediate handed over in shared memory.
 *      smes_mlp_fwd:   H = relu(X W1_e^T + b1_e) (+ relu bit-mask, H optional), P = H G_e^T + c_e
 *                      (execution.py:126-158 for both pools + the folded heads model.py:202-208).
 *      smes_mlp_dgrad: dH = (C G_e) * mask, dX = dH W1_e (training.py:180-192); dH optional.
 *      d in {64, 128, 256, 512} (dgrad: <= 256), d_ff % 128 == 0, ldg <= 16. */
int smes_mlp_fwd(const void* X, long ldx, long rows_cap, const void* W1, const float* b1, const void* G,
                 const float* c, int ldg, int E, int d, int d_ff, const int* seg, uint32_t* relu_bits,
                 long bits_ld, void* H, long ldh, float* P, long ldp, void* stream);
/* smes_mlp_fwd_pack: the same, its X rows copied by an in-kernel gather warp from src[gather[r]]
 * (LDGSTS; -1 = a zero row) and also stored as the packed X (rows_cap, ldx) for the weight
 * gradient: the plan scatter then only places rows (model.py:301 inside the expert kernel). */
int smes_mlp_fwd_pack(const void* src, long ld_src, const int32_t* gather, void* X, long ldx, long rows_cap,
                      const void* W1, const float* b1, const void* G, const float* c, int ldg, int E, int d, int d_ff,
                      const int* seg, uint32_t* relu_bits, long bits_ld, void* H, long ldh, float* P, long ldp,
                      void* stream);
/* smes_mlp_fwd_gather: the same with X gathered from its source rows (X row r = src row gather[r],
 * -1 = zeros; TMA gather4), replacing the gather of model.py:301 -- no packed X in HBM. */
int smes_mlp_fwd_gather(const void* src, long ld_src, long n_src, const int32_t* gather, long rows_cap,
                        const void* W1, const float* b1, const void* G, const float* c, int ldg, int E, int d,
                        int d_ff, const int* seg, uint32_t* relu_bits, long bits_ld, void* H, long ldh, float* P,
                        long ldp, void* stream);
/* smes_mlp_fwd2: the same forward on 2-CTA clusters (cta_group::2, M = 256 per MMA over two
 * consecutive tiles of one expert; each CTA loads half of every W1 / G k-block). */
int smes_mlp_fwd2(const void* X, long ldx, long rows_cap, const void* W1, const float* b1, const void* G,
                  const float* c, int ldg, int E, int d, int d_ff, const int* seg, uint32_t* relu_bits,
                  long bits_ld, void* H, long ldh, float* P, long ldp, void* stream);
int smes_mlp_dgrad(const void* C, long ldc, long rows_cap, const void* G, int ldg, const void* W1, int E, int d,
                   int d_ff, const int* seg, const uint32_t* relu_bits, long bits_ld, void* dX, long lddx,
                   void* dH, long lddh, void* stream);
/* smes_mlp_dgrad2: the same dgrad on 2-CTA clusters (each CTA loads half of every W1 / G k-block);
 * d in {128, 256}. */
int smes_mlp_dgrad2(const void* C, long ldc, long rows_cap, const void* G, int ldg, const void* W1, int E, int d,
                    int d_ff, const int* seg, const uint32_t* relu_bits, long bits_ld, void* dX, long lddx,
                    void* dH, long lddh, void* stream);
/* fc1 weight gradient with dH recomputed per 128-row block (dH never stored): one CTA per
 * (expert, 128-wide d_ff chunk); dW (E, d_ff, d) fp32, db (E, d_ff) fp32; d <= 256. */
int smes_mlp_wgrad(const void* C, long ldc, long rows_cap, const void* G, int ldg, const void* X, long ldx, int E,
                   int d, int d_ff, const int* seg, const uint32_t* relu_bits, long bits_ld, float* dW, float* db,
                   void* stream);

/* ---- expert parallelism (csrc/ep.cu; BASELINE config c5).  Rank r owns experts [r*El, (r+1)*El),
 *      El % 32 == 0 (whole union-mask words).  Fixed-slot buffers: every count stays on the device.
 *      smes_ep_pack:       per owner r, the instances whose union meets r's words (ascending b):
 *                          idx (n, B), pos (n, B) (-1 if absent), cnt (n), mask words (n, B, wpr), h rows (n, B, d)
 *      smes_ep_segments:   (packed row, slot row, rows) per (peer, local expert); mode 0 owner, 1 source
 *      smes_ep_copy_rows:  dir 0 packed -> slots, dir 1 slots -> packed (16-byte rows)
 *      smes_ep_combine_dh: d_hidden[b] = dh_router[b] + sum_r dh_recv[r][pos[r][b]] (fixed owner order)
 *      smes_ep_capacity_guard: empty the owner plan and raise flag if its rows exceed the workspace
 *      smes_ep_put_slots / smes_ep_signal_wait: peer-memory all-to-all (CUDA IPC pointers, flag epochs)
 *      smes_ipc_handle / smes_ipc_open / smes_ipc_close: CUDA IPC plumbing (64-byte handles).
 *      smes_ipc_handle also returns dev_ptr's offset inside its allocation: the peer maps the
 *      allocation base and must add it. */
int smes_ep_pack(int B, int EW, const uint32_t* umask, int n, int wpr, const void* h_bf16, long ldh, int d,
                 int32_t* idx, int32_t* pos, int32_t* cnt, uint32_t* mask_out, void* h_out_bf16, void* stream);
int smes_ep_segments(int mode, int n, int El, const int32_t* cnt, const int32_t* seg_pad, long slot_rows,
                     int32_t* tab, void* stream);
int smes_ep_copy_rows(int nseg, const int32_t* tab, int dir, const void* src, long src_ld_bytes, void* dst,
                      long dst_ld_bytes, int row_bytes, void* stream);
int smes_ep_combine_dh(int B, int d, int n, long slot_rows, const int32_t* pos, const float* dh_recv,
                       const float* dh_router, float* out, void* stream);
int smes_ep_capacity_guard(int E, long cap, const int32_t* totals, int32_t* seg_pad, int32_t* loads,
                           uint32_t* umask, long n_mask_words, int32_t* usize, long n_inst, int32_t* flag,
                           void* stream);
/* fused dispatch / return over peer memory: the pack (resp. the segment gather) writes straight into
 * slot `self` of every owner's (resp. source's) receive buffer through the peer pointer tables. */
int smes_ep_pack_put(int B, int EW, const uint32_t* umask, int n, int wpr, const void* h_bf16, long ldh, int d,
                     int self, int32_t* idx, int32_t* pos, int32_t* cnt, void* const* peer_mask_recv,
                     void* const* peer_h_recv, void* stream);
int smes_ep_copy_rows_put(int nseg, const int32_t* tab, int El, long slot_rows, int self, const void* src,
                          long src_ld_bytes, void* const* peer_dst, long dst_ld_bytes, int row_bytes, void* stream);
int smes_ep_put_slots(int n, int self, const void* send, long slot_bytes, long row_bytes, const int32_t* rows_used,
                      void* const* peer_recv_dev, void* stream);
int smes_ep_signal_wait(int n, int self, void* const* peer_flags_dev, int32_t* my_flags, int epoch, void* stream);
int smes_ipc_handle(void* dev_ptr, void* handle_out, long* offset_out);
int smes_ipc_open(const void* handle, void** dev_ptr_out);
int smes_ipc_close(void* dev_ptr);

/* ---- K5 LoadStats / loss: compute_load_stats (balance.py:54-80), total_loss (training.py:90-94). */
/* every reduction of the training combine's per-CTA partials in one launch: loss_out {task, L_lb,
 * total}, per-(expert, task) sums of C (optional), router bias grads (optional), head bias grads. */
int smes_post_combine(int nparts, const float* part_csum, int n_csum, float* csum, const float* part_rb, int n_rb,
                      float* rb, const float* part_db, int n_db, float* db, const double* loss_part, double inv_b,
                      double beta, const double* stats_value, double* loss_out, void* stream);
/* lb_experts: the E of the load-balancing value (E / K) <f, p> (balance.py:69-70); 0 = E.  It differs
 * from E when the shim pads the expert count with never-selected experts (model.py). */
int smes_stats_finalize(int E, int K, int lb_experts, double batch_times_tasks, int dense, const double* raw,
                        double* out, float* freq_f32, void* stream);
int smes_loss_finalize(int nparts, const double* part, double inv_b, double beta, const double* stats_value,
                       double* out, void* stream);

/* ---- reductions: bias grads (training.py:190), un-permute (training.py:192 + :212),
 *      per-CTA partials (training.py:151-152). */
int smes_seg_colsum(const void* M, long ld, long rows_cap, int N, const int32_t* seg, int G, float* part, float* out,
                    void* stream);
int smes_unpermute(int B, int d, const int32_t* usize, const int32_t* row_of, int umax, const void* dX, long ldx,
                   const float* dh_router, float* dh, void* stream);
int smes_part_reduce(const float* part, int nparts, int n, float* out, void* stream);

/* ---- standalone reference entry points: lb_loss_gradient (balance.py:83-99) as a dense
 *      (T,B,E) tensor; task_loss (training.py:60-87) partial sums + validity flags
 *      (bit 1: prediction outside [0,1], bit 2: label not in {0,1}). */
int smes_lb_grad(int T, int B, int E, int K, const int32_t* active, const float* wsel, const float* z, long zst,
                 long zsb, const float* freq, float coef, int dense, float* out, void* stream);
int smes_bce_loss(int T, int B, const float* pred, const float* labels, const float* lam, double* part, int nparts,
                  int32_t* bad, void* stream);

/* ---- fp32 arithmetic mode (BASELINE c1, the north star's fp32 1e-5 contract; the reference is
 *      float64 NumPy, linalg.py:3-8).  Dense contractions run on the tensor cores as bf16x3
 *      products: every fp32 operand is stored as three bf16 planes [x0 | x1 | x2] along K
 *      (x = x0 + x1 + x2, 24 significant bits) and the six leading cross terms accumulate in fp32.
 *      smes_gemm_ragged_m_x3: C = act(A W_g^T + b_g), A (rows, >= 3K) and W (G, N, 3K) in planes,
 *        fp32 out; replaces grouped_gemm (execution.py:126-158) and RouterBank.logits
 *        (routing.py:101-103) in fp32.  K % 64 == 0.
 *      smes_split_bf16x3: fp32 (rows, cols) -> planes (rows, 3 cols); rows_dev (optional, device)
 *        caps the row count (the plan's padded row total).
 *      smes_combine_fwd_f32: reconstruct_task_reps (execution.py:161-191) + _heads
 *        (model.py:202-208) + clamped BCE partials (training.py:54-57), fp32 O and reps. */
int smes_gemm_ragged_m_x3(const void* A3, long lda, long rows_cap, const void* W3, int G, int N, int K,
                          const int* seg, const float* bias, int act, float* C, long ldc, long m_limit, void* stream);
int smes_split_bf16x3(long rows, int cols, const float* src, long lds, void* dst, long ldd, const int32_t* rows_dev,
                      void* stream);
int smes_combine_fwd_f32_grid(int B);
int smes_combine_fwd_f32(int T, int B, int E, int K, int d_out, int umax, const uint32_t* umask, const int32_t* usize,
                         const int32_t* row_of, const int32_t* active, const float* wsel, const float* O, long ldo,
                         const float* head_w, const float* head_b, float* reps, float* logits, float* preds,
                         const float* labels, const float* lam, double* loss_part, int grid, void* stream);
/* the same with the loss finalize (smes_loss_finalize) done by the last CTA to finish: loss_out =
 * [task, L_lb, task + beta L_lb] (training.py:60-94); ticket: one int32, zero before the first
 * launch (the kernel resets it). */
int smes_combine_fwd_f32_loss(int T, int B, int E, int K, int d_out, int umax, const uint32_t* umask,
                              const int32_t* usize, const int32_t* row_of, const int32_t* active, const float* wsel,
                              const float* O, long ldo, const float* head_w, const float* head_b, float* reps,
                              float* logits, float* preds, const float* labels, const float* lam, double* loss_part,
                              int grid, int32_t* ticket, double inv_b, double beta, const double* stats_value,
                              double* loss_out, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* SMES_H_ */
