// K4 / K6+K7 -- combine, task heads, BCE, and their backward (gather form, no atomics).
//
// Forward restates `reconstruct_task_reps` (taskmoe/execution.py:161-191) fused
// with `_heads` (taskmoe/model.py:202-208) and the clamped BCE
// (taskmoe/training.py:54-57).  Each packed row O[u] of an instance is loaded
// ONCE; it is accumulated into all T task representations and projected onto
// all T heads:  P[u, t] = <head_w_t, O[u]>  (so logit_t = sum_u w[u,t] P[u,t] + b_t).
// P is kept (rows x T fp32) for the backward.
//
// Backward restates training.py:146-179 (+ the LB term of :155-157 and
// balance.py:83-99) without touching O (identity last pool):
//   dlogit_t  = lambda_t / B (yhat - y) [clamp inactive]                       (:147-148)
//   d_packed[u] = sum_t w[u,t] dlogit_t head_w_t  (x [O>0] if last act relu)   (:172-176, :180-181)
//   g[t,k]    = dlogit_t P[u(t,k), t]                                           (:171)
//   dz[t,e_k] = w_k (g_k - sum_j g_j w_j) + beta * coef * w_k (f[e_k] - <w, f>) (:178-179, balance.py:97-99)
//   dW_head_t = sum_b dlogit_t reps_t                                           (:151)
// A CTA of 8 warps owns 8/S instances at a time (S warps per instance, each
// thread 4..16 columns); head-grad partials stay in registers across instances
// and are combined in a fixed order (deterministic).
#include "ptx.cuh"
#include "smes_capi.h"

namespace smes {

constexpr int CB_MAX_U = 128;
constexpr int CB_MAX_T = 32;
constexpr int CB_THREADS = 256;
constexpr int CB_WARPS = CB_THREADS / 32;
constexpr int CB_MAX_TK = 1024;

__device__ __forceinline__ int union_rank(const uint32_t* um, int e) {
  int r = 0;
  for (int j = 0; j < (e >> 5); ++j) r += __popc(um[j]);
  return r + __popc(um[e >> 5] & ((1u << (e & 31)) - 1u));
}

// bf16 row slice -> fp32 registers (generic load: used on the shared-memory row stages)
template <int VPL>
__device__ __forceinline__ void load_bf(const __nv_bfloat16* p, float (&x)[VPL]) {
  if constexpr (VPL == 4) {
    const uint2 v = *reinterpret_cast<const uint2*>(p);
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&v);
#pragma unroll
    for (int j = 0; j < 2; ++j) { float2 f = __bfloat1622float2(h[j]); x[2 * j] = f.x; x[2 * j + 1] = f.y; }
  } else {
#pragma unroll
    for (int i = 0; i < VPL; i += 8) {
      const uint4 v = *reinterpret_cast<const uint4*>(p + i);
      const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&v);
#pragma unroll
      for (int j = 0; j < 4; ++j) { float2 f = __bfloat1622float2(h[j]); x[i + 2 * j] = f.x; x[i + 2 * j + 1] = f.y; }
    }
  }
}
template <int VPL>
__device__ __forceinline__ void store_bf(__nv_bfloat16* p, const float (&x)[VPL]) {
  if constexpr (VPL == 4) {
    *reinterpret_cast<uint2*>(p) = make_uint2(pack_bf16(x[0], x[1]), pack_bf16(x[2], x[3]));
  } else {
#pragma unroll
    for (int i = 0; i < VPL; i += 8)
      *reinterpret_cast<uint4*>(p + i) = make_uint4(pack_bf16(x[i], x[i + 1]), pack_bf16(x[i + 2], x[i + 3]),
                                                    pack_bf16(x[i + 4], x[i + 5]), pack_bf16(x[i + 6], x[i + 7]));
  }
}
template <int VPL>
__device__ __forceinline__ void load_f32(const float* p, float (&x)[VPL]) {
#pragma unroll
  for (int i = 0; i < VPL; i += 4) {
    float4 v = __ldg(reinterpret_cast<const float4*>(p + i));
    x[i] = v.x; x[i + 1] = v.y; x[i + 2] = v.z; x[i + 3] = v.w;
  }
}

// Butterfly reduce-scatter of N (power of two <= 32) per-lane values over a warp.
// Returns the warp total of index t = (lane >> (5 - log2 N)) & (N - 1).
template <int N>
__device__ __forceinline__ float warp_reduce_scatter(float (&v)[N], int lane) {
  constexpr int lg = N == 1 ? 0 : N == 2 ? 1 : N == 4 ? 2 : N == 8 ? 3 : N == 16 ? 4 : 5;
#pragma unroll
  for (int s = 0; s < lg; ++s) {
    const int half = N >> (s + 1);
    const int o = 16 >> s;
    const bool upper = (lane & o) != 0;
#pragma unroll
    for (int i = 0; i < half; ++i) {
      const float send = upper ? v[i] : v[i + half];
      const float keep = upper ? v[i + half] : v[i];
      v[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
    }
  }
#pragma unroll
  for (int o = 16 >> lg; o > 0; o >>= 1) v[0] += __shfl_xor_sync(0xffffffffu, v[0], o);
  return v[0];
}
template <int N>
__device__ __forceinline__ int rs_index(int lane) {
  constexpr int lg = N == 1 ? 0 : N == 2 ? 1 : N == 4 ? 2 : N == 8 ? 3 : N == 16 ? 4 : 5;
  return (lane >> (5 - lg)) & (N - 1);
}

struct CombineArgs {
  int T, B, E, K, d_out, umax;
  const uint32_t* umask;   // (B, EW)
  const int32_t* usize;    // (B,)
  const int32_t* row_of;   // (B, umax)
  const int32_t* active;   // (T, B, K)
  const float* wsel;       // (T, B, K)
  const __nv_bfloat16* O;  // packed expert outputs (rows, ldo)
  long ldo;
  const float* head_w;     // (T, d_out)
  const float* head_b;     // (T,)
  float* P;                // (rows, ldp) head projections of every packed row
  int ldp;
  __nv_bfloat16* reps;     // (T, B, d_out)
  float* logits;           // (T, B)
  float* preds;            // (T, B)
  const float* labels;     // optional (T, B)
  const float* lam;        // (T,)
  double* loss_part;       // (grid,) per-CTA sum of lambda-weighted BCE
  // backward
  float inv_b;
  int relu_last;
  __nv_bfloat16* dpacked;  // (rows, ldo)
  __nv_bfloat16* dz;       // (B, T*E) dense
  const float* freq;       // (E,)
  float lb_coef;           // beta * E / (K * B * T)
  int dense_probs;
  const float* z;          // logits (B, T*E) (dense mode only)
  float* part_dw;          // (grid, T, d_out)
  float* part_db;          // (grid, T)
};

// cp_async16: ptx.cuh
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
}

// Per-instance-group shared memory (sized at run time by umax):
//   um[32] | rows[umax] | wt[umax][MAXT] | dl[MAXT] | P stage [umax][ldp] | row stage [nrow][d_out] bf16
struct GroupLayout {
  int off_rows, off_wt, off_dl, off_p, off_stage, bytes;
  __host__ __device__ GroupLayout(int umax, int maxt, int ldp, int stage_rows, int d_out) {
    auto al = [](int x) { return (x + 15) & ~15; };
    off_rows = 128;
    off_wt = al(off_rows + umax * 4);
    off_dl = al(off_wt + umax * maxt * 4);
    off_p = al(off_dl + maxt * 4);
    off_stage = al(off_p + umax * ldp * 4);
    bytes = al(off_stage + stage_rows * d_out * 2);
  }
};

// Scoring without task reps (P only, no labels): a warp per instance, TPL = 32 / next_pow2(T) lanes
// per task, each lane summing w * P[row(e), t] over its share of the task's K active experts in k
// order, then a fixed xor tree over the task's lanes (model.py:202-208 on the folded heads).  No
// shared memory, no block barriers: the per-instance gathers are the whole cost.
template <int TPL>
__global__ void __launch_bounds__(256) combine_score_kernel(const CombineArgs a) {
  pdl_wait();
  const int lane = threadIdx.x & 31;
  const int t = lane / TPL, sub = lane % TPL;
  const int EW = (a.E + 31) >> 5, K = a.K;
  const int nw = gridDim.x * (blockDim.x >> 5);
  for (int b = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); b < a.B; b += nw) {
    float acc = 0.f;
    if (t < a.T) {
      const uint32_t* um = a.umask + (long)b * EW;
      const long o0 = ((long)t * a.B + b) * K;
      for (int k = sub; k < K; k += TPL) {
        const int e = __ldg(a.active + o0 + k);
        const float w = __ldg(a.wsel + o0 + k);
        const int row = __ldg(a.row_of + (long)b * a.umax + union_rank(um, e));
        acc = fmaf(w, __ldg(a.P + (long)row * a.ldp + t), acc);
      }
    }
#pragma unroll
    for (int o = TPL / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (sub == 0 && t < a.T) {
      const float lg = acc + a.head_b[t];
      const float ez = expf(-fabsf(lg));               // stable sigmoid (linalg.py:108-113)
      const float pos = 1.f / (1.f + ez);
      a.logits[(long)t * a.B + b] = lg;
      a.preds[(long)t * a.B + b] = lg >= 0.f ? pos : 1.f - pos;
    }
  }
}

template <int VPL, int MAXT>
__global__ void __launch_bounds__(CB_THREADS) combine_fwd_kernel(const CombineArgs a) {
  pdl_wait();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int S = a.d_out / (32 * VPL);        // warps per instance
  const int G = CB_WARPS / S;                 // instances per CTA iteration
  const int gi = warp / S, ws = warp % S;
  const int col = (ws * 32 + lane) * VPL;
  const int T = a.T, K = a.K, EW = (a.E + 31) >> 5, umax = a.umax;
  const int ldp = a.ldp;
  const bool has_p = a.P != nullptr;
  const bool has_o = a.O != nullptr;           // scoring (no task reps): logits from P only
  extern __shared__ __align__(16) uint8_t smraw[];
  const GroupLayout L(umax, MAXT, ldp, umax, a.d_out);
  uint8_t* g0 = smraw + (size_t)gi * L.bytes;
  uint32_t* s_um = reinterpret_cast<uint32_t*>(g0);
  int32_t* s_rows = reinterpret_cast<int32_t*>(g0 + L.off_rows);
  float* s_wt = reinterpret_cast<float*>(g0 + L.off_wt);
  float* s_p = reinterpret_cast<float*>(g0 + L.off_p);
  __nv_bfloat16* s_o = reinterpret_cast<__nv_bfloat16*>(g0 + L.off_stage);
  const int gthreads = S * 32, gtid = ws * 32 + lane;
  const int lt = lane & (MAXT - 1), ug = lane / MAXT;
  constexpr int NG = 32 / MAXT;
  const int cpr = a.d_out / 8;                 // 16-byte chunks per O row
  const int pcr = ldp / 4;                     // 16-byte chunks per P row
  double my_loss = 0.0;
  const int iters = (a.B + (long)gridDim.x * G - 1) / ((long)gridDim.x * G);
  for (int it = 0; it < iters; ++it) {
    const int b = (it * gridDim.x + blockIdx.x) * G + gi;
    const bool valid = b < a.B;
    const int U = valid ? a.usize[b] : 0;
    if (valid) {
      for (int j = gtid; j < EW; j += gthreads) s_um[j] = a.umask[(long)b * EW + j];
      for (int u = gtid; u < U; u += gthreads) s_rows[u] = a.row_of[(long)b * a.umax + u];
      for (int i = gtid; i < U * MAXT; i += gthreads) s_wt[i] = 0.f;
    }
    __syncthreads();
    if (valid) {
      // gather every packed row of the instance (and its head projections) into smem at once
      if (has_o)
        for (int i = gtid; i < U * cpr; i += gthreads) {
          const int u = i / cpr, c = i - u * cpr;
          cp_async16(s_o + (long)u * a.d_out + c * 8, a.O + (long)s_rows[u] * a.ldo + c * 8);
        }
      if (has_p)
        for (int i = gtid; i < U * pcr; i += gthreads) {
          const int u = i / pcr, c = i - u * pcr;
          cp_async16(s_p + (long)u * ldp + c * 4, a.P + (long)s_rows[u] * ldp + c * 4);
        }
      for (int i = gtid; i < T * K; i += gthreads) {
        const int t = i / K;
        const long o = ((long)t * a.B + b) * K + (i - t * K);
        s_wt[union_rank(s_um, a.active[o]) * MAXT + t] = a.wsel[o];
      }
      cp_async_wait_all();
    }
    __syncthreads();
    if (valid) {
      // reps_t = sum_u w[u,t] O[u]   (every packed row read once)
      if (has_o) {
      float acc[MAXT][VPL];
#pragma unroll
      for (int t = 0; t < MAXT; ++t)
#pragma unroll
        for (int v = 0; v < VPL; ++v) acc[t][v] = 0.f;
      for (int u = 0; u < U; ++u) {
        float x[VPL];
        load_bf<VPL>(s_o + (long)u * a.d_out + col, x);
#pragma unroll
        for (int t = 0; t < MAXT; ++t) {
          const float w = s_wt[u * MAXT + t];
#pragma unroll
          for (int v = 0; v < VPL; ++v) acc[t][v] = fmaf(w, x[v], acc[t][v]);
        }
      }
#pragma unroll
      for (int t = 0; t < MAXT; ++t)
        if (t < T) store_bf<VPL>(a.reps + ((long)t * a.B + b) * a.d_out + col, acc[t]);
      }
      // logit_t = b_t + sum_u w[u,t] P[u,t]   (P = O head_W^T from the tensor-core GEMM)
      if (ws == 0 && has_p) {
        float sacc = 0.f;
        if (lt < T)
          for (int u = ug; u < U; u += NG) sacc = fmaf(s_wt[u * MAXT + lt], s_p[u * ldp + lt], sacc);
#pragma unroll
        for (int o = 16; o >= MAXT; o >>= 1) sacc += __shfl_xor_sync(0xffffffffu, sacc, o);
        if (ug == 0 && lt < T) {
          const int t = lt;
          const float lg = sacc + a.head_b[t];
          const float ez = expf(-fabsf(lg));               // stable sigmoid (linalg.py:108-113)
          const float pos = 1.f / (1.f + ez);
          const float pr = lg >= 0.f ? pos : 1.f - pos;
          a.logits[(long)t * a.B + b] = lg;
          a.preds[(long)t * a.B + b] = pr;
          if (a.labels) {
            const double y = a.labels[(long)t * a.B + b];
            double pc = (double)pr;
            pc = pc < 1e-7 ? 1e-7 : (pc > 1.0 - 1e-7 ? 1.0 - 1e-7 : pc);
            my_loss += (double)a.lam[t] * -(y * log(pc) + (1.0 - y) * log1p(-pc));
          }
        }
      }
    }
    __syncthreads();
  }
  if (a.loss_part) {
    double* s_l = reinterpret_cast<double*>(smraw);
    s_l[threadIdx.x] = my_loss;
    __syncthreads();
    if (threadIdx.x == 0) {
      double s = 0.0;
      for (int i = 0; i < CB_THREADS; ++i) s += s_l[i];
      a.loss_part[blockIdx.x] = s;
    }
  }
}

// Training-step combine (sparse LB reading).  Labels and the global selection frequency
// are known when the forward combine runs, so one pass produces the forward outputs
// (logits, preds, loss) and every backward term that is not a dense contraction:
//   dlogit_t = lambda_t / B (yhat - y) [clamp inactive]                      (training.py:147-148)
//   C[row, t] = w[row, t] dlogit_t            (bf16, one (rows, ldc) matrix)
//   dz[t, e_k] = w_k (g_k - sum_j g_j w_j) + beta coef w_k (f_k - sum_j w_j f_j),
//                g_k = dlogit_t P[row_k, t]                                   (training.py:171-179, balance.py:97-99)
// The two dense contractions run on the tcgen05 GEMM afterwards:
//   d_packed = C head_W   (K = T)         and      dW_head = C^T O   (split-K over expert halves).
// Nothing per-column is computed here, so the kernel only touches T*K pairs per instance.
template <int MAXT>
__global__ void __launch_bounds__(CB_THREADS) combine_train_kernel(const CombineArgs a, __nv_bfloat16* cmat, int ldc,
                                                                 float* part_csum, float* part_rb) {
  pdl_wait();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int T = a.T, K = a.K, E = a.E, EW = (E + 31) >> 5, TE = T * E, TK = T * K, umax = a.umax;
  const int ldp = a.ldp;
  extern __shared__ __align__(16) uint8_t smraw[];
  // per-warp (one instance per warp) tables
  const int per_warp = 128 + umax * 4 + TK * 4 * 4 + MAXT * 4 + 64;
  uint8_t* w0 = smraw + (size_t)warp * ((per_warp + 15) & ~15);
  uint32_t* s_um = reinterpret_cast<uint32_t*>(w0);
  int32_t* s_rows = reinterpret_cast<int32_t*>(w0 + 128);
  int32_t* s_act = s_rows + umax;
  float* s_w = reinterpret_cast<float*>(s_act + TK);
  float* s_gw = s_w + TK;
  float* s_wf = s_gw + TK;
  float* s_dl = s_wf + TK;
  // per-warp accumulators (conflict-free: within one instance every (task, expert) pair is distinct)
  const size_t acc_base = (size_t)CB_WARPS * ((per_warp + 15) & ~15);
  float* s_cs = part_csum ? reinterpret_cast<float*>(smraw + acc_base) + (size_t)warp * E * T : nullptr;  // [E][T]
  float* s_rb = part_rb ? reinterpret_cast<float*>(smraw + acc_base) + (size_t)CB_WARPS * E * T * (part_csum ? 1 : 0) +
                              (size_t)warp * TE : nullptr;                                                     // [T][E]
  if (s_cs) for (int i = lane; i < E * T; i += 32) s_cs[i] = 0.f;
  if (s_rb) for (int i = lane; i < TE; i += 32) s_rb[i] = 0.f;
  float my_db = 0.f;
  double my_loss = 0.0;
  const float lam_t = lane < T ? a.lam[lane] : 0.f, hb = lane < T ? a.head_b[lane] : 0.f;
  // The per-instance tables (usize, union mask, row_of over its full umax width, active, weights,
  // labels) of the NEXT instance are fetched into registers while this one is processed, so each
  // instance waits only on its P gathers.  Register path for E <= 64, umax <= 64, T*K <= 64.
  const bool pf = EW <= 2 && umax <= 64 && TK <= 64;
  const int stride = gridDim.x * CB_WARPS;
  int pU = 0, pRows[2] = {0, 0}, pAct[2] = {0, 0};
  uint32_t pUm[2] = {0u, 0u};
  float pW[2] = {0.f, 0.f}, pY = 0.f;
  auto fetch = [&](int b) {
    pU = a.usize[b];
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const int j = lane + 32 * k;
      if (j < EW) pUm[k] = a.umask[(long)b * EW + j];
      if (j < umax) pRows[k] = a.row_of[(long)b * a.umax + j];
      if (j < TK) {
        const int t = j / K;
        const long o = ((long)t * a.B + b) * K + (j - t * K);
        pAct[k] = a.active[o];
        pW[k] = a.wsel[o];
      }
    }
    if (lane < T) pY = a.labels[(long)lane * a.B + b];
  };
  // P / freq gathers of an instance whose tables sit in registers (pUm, pRows, pAct): issued for
  // the NEXT instance in the middle of this one, so their latency overlaps its tail
  float gn[2] = {0.f, 0.f}, fn[2] = {0.f, 0.f};
  auto gather_next = [&]() {
    const uint32_t w0 = __shfl_sync(0xffffffffu, pUm[0], 0), w1 = EW > 1 ? __shfl_sync(0xffffffffu, pUm[0], 1) : 0u;
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const int j = lane + 32 * k;
      const int e = pAct[k];
      const int rank = e < 32 ? __popc(w0 & ((1u << e) - 1u)) : __popc(w0) + __popc(w1 & ((1u << (e - 32)) - 1u));
      const int r0 = __shfl_sync(0xffffffffu, pRows[0], rank & 31), r1 = __shfl_sync(0xffffffffu, pRows[1], rank & 31);
      if (j < TK) {
        gn[k] = __ldg(a.P + (long)(rank < 32 ? r0 : r1) * ldp + j / K);
        fn[k] = __ldg(a.freq + e);
      }
    }
  };
  if (pf && blockIdx.x * CB_WARPS + warp < a.B) {
    fetch(blockIdx.x * CB_WARPS + warp);
    gather_next();
  }
  for (int b = blockIdx.x * CB_WARPS + warp; b < a.B; b += stride) {
    int U;
    float y = 0.f;
    if (pf) {
      U = pU;
      y = pY;
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        const int j = lane + 32 * k;
        if (j < EW) s_um[j] = pUm[k];
        if (j < umax) s_rows[j] = pRows[k];
        if (j < TK) { s_act[j] = pAct[k]; s_w[j] = pW[k]; }
      }
      if (b + stride < a.B) fetch(b + stride);   // next instance's tables, in flight from here
    } else {
      // one round trip for every per-instance table
      U = a.usize[b];
      for (int j = lane; j < EW; j += 32) s_um[j] = a.umask[(long)b * EW + j];
      for (int u = lane; u < umax; u += 32) s_rows[u] = a.row_of[(long)b * a.umax + u];
      for (int i = lane; i < TK; i += 32) {
        const int t = i / K;
        const long o = ((long)t * a.B + b) * K + (i - t * K);
        s_act[i] = a.active[o];
        s_w[i] = a.wsel[o];
      }
      if (lane < T) y = a.labels[(long)lane * a.B + b];
    }
    __syncwarp();
    // logits from the head projections: logit_t = b_t + sum_k w_k P[row_k, t]; the gathers of a
    // lane's (task, slot) pairs are issued together (second and last round trip)
    if (pf) {
      // this instance's gathers were issued during the previous one
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        const int i = lane + 32 * k;
        if (i < TK) {
          const float w = s_w[i];
          s_gw[i] = w * gn[k];
          s_wf[i] = w * fn[k];
        }
      }
      // next instance's gathers: its tables were fetched at the top of this iteration; the loads
      // overlap the rest of this instance (loss, dlogit, C rows, dz)
      if (b + stride < a.B) gather_next();
    } else {
      constexpr int kMaxI = 4;                  // TK <= 128 per warp pass
      float gv[kMaxI], fv[kMaxI];
#pragma unroll
      for (int r = 0; r < kMaxI; ++r) {
        const int i = lane + 32 * r;
        gv[r] = 0.f; fv[r] = 0.f;
        if (i < TK) {
          const int t = i / K;
          const int e = s_act[i];
          gv[r] = __ldg(a.P + (long)s_rows[union_rank(s_um, e)] * ldp + t);
          fv[r] = __ldg(a.freq + e);
        }
      }
#pragma unroll
      for (int r = 0; r < kMaxI; ++r) {
        const int i = lane + 32 * r;
        if (i < TK) {
          const float w = s_w[i];
          s_gw[i] = w * gv[r];                  // w_k P_k  (scaled by dlogit below)
          s_wf[i] = w * fv[r];
        }
      }
      for (int i = lane + 32 * kMaxI; i < TK; i += 32) {
        const int t = i / K;
        const float w = s_w[i];
        s_gw[i] = w * __ldg(a.P + (long)s_rows[union_rank(s_um, s_act[i])] * ldp + t);
        s_wf[i] = w * __ldg(a.freq + s_act[i]);
      }
    }
    __syncwarp();
    if (lane < T) {
      const int t = lane;
      float lg = hb;
      for (int k = 0; k < K; ++k) lg += s_gw[t * K + k];
      const float ez = expf(-fabsf(lg));                 // stable sigmoid (linalg.py:108-113)
      const float pos = 1.f / (1.f + ez);
      const float pr = lg >= 0.f ? pos : 1.f - pos;
      a.logits[(long)t * a.B + b] = lg;
      a.preds[(long)t * a.B + b] = pr;
      // BCE with the reference's clamp (training.py:54-71); logs in fp32, accumulated in fp64
      const float pc = fminf(fmaxf(pr, 1e-7f), 1.f - 1e-7f);
      my_loss += (double)lam_t * -((double)y * (double)logf(pc) + (1.0 - (double)y) * (double)log1pf(-pc));
      const bool inside = pr > 1e-7f && pr < 1.f - 1e-7f;
      const float dl = inside ? lam_t * a.inv_b * (pr - y) : 0.f;
      s_dl[t] = dl;
      my_db += dl;
    }
    __syncwarp();
    // C rows: every (row, task) coefficient; rows of an instance are zeroed first (tasks that
    // do not select the row's expert contribute 0)
    for (int i = lane; i < U * (ldc / 8); i += 32) {
      const int u = i / (ldc / 8), c = i - u * (ldc / 8);
      *reinterpret_cast<uint4*>(cmat + (long)s_rows[u] * ldc + c * 8) = make_uint4(0, 0, 0, 0);
    }
    __nv_bfloat16* dzr = a.dz + (long)b * TE;
    for (int i = lane * 8; i < TE; i += 256) *reinterpret_cast<uint4*>(dzr + i) = make_uint4(0, 0, 0, 0);
    __syncwarp();
    for (int i = lane; i < TK; i += 32) {
      const int t = i / K;
      const int row = s_rows[union_rank(s_um, s_act[i])];
      const float w = s_w[i], dl = s_dl[t];
      cmat[(long)row * ldc + t] = __float2bfloat16_rn(w * dl);
      float Gt = 0.f, Ft = 0.f;
      for (int k = 0; k < K; ++k) { Gt += s_gw[t * K + k]; Ft += s_wf[t * K + k]; }
      // w (g - G) with g = dl P, G = dl sum_j w_j P_j ;  coef w (f - F)
      const float dzv = dl * (s_gw[i] - w * Gt) + a.lb_coef * (s_wf[i] - w * Ft);
      dzr[t * E + s_act[i]] = __float2bfloat16_rn(dzv);
      if (s_cs) s_cs[s_act[i] * T + t] += w * dl;     // per-(expert, task) sum of C   -> last-pool bias grad
      if (s_rb) s_rb[t * E + s_act[i]] += dzv;        // column sum of dz              -> router bias grad
    }
    __syncwarp();
  }
  // per-CTA partials (fixed order)
  __shared__ float s_db[CB_WARPS][CB_MAX_T];
  __shared__ double s_l[CB_THREADS];
  if (lane < T) s_db[warp][lane] = my_db;
  s_l[threadIdx.x] = my_loss;
  __syncthreads();
  if (threadIdx.x < T) {
    float sum = 0.f;
    for (int w = 0; w < CB_WARPS; ++w) sum += s_db[w][threadIdx.x];
    a.part_db[(long)blockIdx.x * T + threadIdx.x] = sum;
  }
  if (threadIdx.x == 0 && a.loss_part) {
    double sum = 0.0;
    for (int i = 0; i < CB_THREADS; ++i) sum += s_l[i];
    a.loss_part[blockIdx.x] = sum;
  }
  if (part_csum) {
    const float* base = reinterpret_cast<const float*>(smraw + acc_base);
    for (int i = threadIdx.x; i < E * T; i += CB_THREADS) {
      float sum = 0.f;
      for (int w = 0; w < CB_WARPS; ++w) sum += base[(size_t)w * E * T + i];
      part_csum[(size_t)blockIdx.x * E * T + i] = sum;
    }
  }
  if (part_rb) {
    const float* base = reinterpret_cast<const float*>(smraw + acc_base) + (size_t)CB_WARPS * E * T * (part_csum ? 1 : 0);
    for (int i = threadIdx.x; i < TE; i += CB_THREADS) {
      float sum = 0.f;
      for (int w = 0; w < CB_WARPS; ++w) sum += base[(size_t)w * TE + i];
      part_rb[(size_t)blockIdx.x * TE + i] = sum;
    }
  }
}

// db[e][n] = sum_t csum[e][t] head_w[t][n]   (bias grad of an identity last pool: dO = C head_W)
__global__ void bias_from_csum_kernel(int E, int T, int d_out, const float* __restrict__ csum,
                                      const float* __restrict__ head_w, float* __restrict__ out) {
  pdl_wait();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= E * d_out) return;
  const int e = i / d_out, n = i - e * d_out;
  float s = 0.f;
  for (int t = 0; t < T; ++t) s = fmaf(csum[e * T + t], head_w[(long)t * d_out + n], s);
  out[i] = s;
}

template <int VPL, int MAXT>
__global__ void __launch_bounds__(CB_THREADS) combine_bwd_kernel(const CombineArgs a) {
  pdl_wait();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int S = a.d_out / (32 * VPL);
  const int G = CB_WARPS / S;
  const int gi = warp / S, ws = warp % S;
  const int col = (ws * 32 + lane) * VPL;
  const int T = a.T, K = a.K, E = a.E, EW = (E + 31) >> 5, TE = T * E, TK = T * K, umax = a.umax;
  const int ldp = a.ldp;
  const int n = T * a.d_out;
  extern __shared__ __align__(16) uint8_t smraw[];
  const int stage_rows = T + (a.relu_last ? umax : 0);
  const GroupLayout L(umax, MAXT, ldp, stage_rows, a.d_out);
  float* s_hw = reinterpret_cast<float*>(smraw);                                   // [T][d_out]
  float* s_pair = s_hw + n;                                                        // [G][2][T*K]
  uint8_t* g0 = reinterpret_cast<uint8_t*>(s_pair + (size_t)G * 2 * TK) + 0;
  g0 = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(g0) + 15) & ~uintptr_t(15)) + (size_t)gi * L.bytes;
  uint32_t* s_um = reinterpret_cast<uint32_t*>(g0);
  int32_t* s_rows = reinterpret_cast<int32_t*>(g0 + L.off_rows);
  float* s_wt = reinterpret_cast<float*>(g0 + L.off_wt);
  float* s_dl = reinterpret_cast<float*>(g0 + L.off_dl);
  float* s_p = reinterpret_cast<float*>(g0 + L.off_p);
  __nv_bfloat16* s_reps = reinterpret_cast<__nv_bfloat16*>(g0 + L.off_stage);      // [T][d_out]
  __nv_bfloat16* s_o = s_reps + (size_t)T * a.d_out;                                // [umax][d_out] (relu_last)
  float* gw_s = s_pair + (long)gi * 2 * TK;
  float* wf_s = gw_s + TK;
  for (int i = threadIdx.x; i < n; i += CB_THREADS) s_hw[i] = a.head_w[i];
  float acc_dw[MAXT][VPL];
#pragma unroll
  for (int t = 0; t < MAXT; ++t)
#pragma unroll
    for (int v = 0; v < VPL; ++v) acc_dw[t][v] = 0.f;
  float my_db = 0.f;
  const int gthreads = S * 32, gtid = ws * 32 + lane;
  const int cpr = a.d_out / 8, pcr = ldp / 4;
  const int iters = (a.B + (long)gridDim.x * G - 1) / ((long)gridDim.x * G);
  for (int it = 0; it < iters; ++it) {
    const int b = (it * gridDim.x + blockIdx.x) * G + gi;
    const bool valid = b < a.B;
    const int U = valid ? a.usize[b] : 0;
    if (valid) {
      for (int j = gtid; j < EW; j += gthreads) s_um[j] = a.umask[(long)b * EW + j];
      for (int u = gtid; u < U; u += gthreads) s_rows[u] = a.row_of[(long)b * a.umax + u];
      for (int i = gtid; i < U * MAXT; i += gthreads) s_wt[i] = 0.f;
      if (gtid < T) {
        const int t = gtid;
        const float p = a.preds[(long)t * a.B + b], y = a.labels[(long)t * a.B + b];
        const bool inside = p > 1e-7f && p < 1.f - 1e-7f;
        const float dl = inside ? a.lam[t] * a.inv_b * (p - y) : 0.f;
        s_dl[t] = dl;
        my_db += dl;
      }
      for (int i = gtid; i < T * cpr; i += gthreads) {
        const int t = i / cpr, c = i - t * cpr;
        cp_async16(s_reps + (long)t * a.d_out + c * 8, a.reps + ((long)t * a.B + b) * a.d_out + c * 8);
      }
    }
    __syncthreads();
    if (valid) {
      for (int i = gtid; i < U * pcr; i += gthreads) {
        const int u = i / pcr, c = i - u * pcr;
        cp_async16(s_p + (long)u * ldp + c * 4, a.P + (long)s_rows[u] * ldp + c * 4);
      }
      if (a.relu_last)
        for (int i = gtid; i < U * cpr; i += gthreads) {
          const int u = i / cpr, c = i - u * cpr;
          cp_async16(s_o + (long)u * a.d_out + c * 8, a.O + (long)s_rows[u] * a.ldo + c * 8);
        }
      for (int i = gtid; i < TK; i += gthreads) {
        const int t = i / K;
        const long o = ((long)t * a.B + b) * K + (i - t * K);
        s_wt[union_rank(s_um, a.active[o]) * MAXT + t] = a.wsel[o];
      }
      cp_async_wait_all();
    }
    __syncthreads();
    if (valid) {
      float dl[MAXT];
#pragma unroll
      for (int t = 0; t < MAXT; ++t) dl[t] = t < T ? s_dl[t] : 0.f;
      // d_packed[u] = sum_t w[u,t] dlogit_t head_w_t   (x relu mask of O if the last pool is relu)
      for (int u = 0; u < U; ++u) {
        asm volatile("" ::: "memory");   // keep head_w in smem (do not hoist T*VPL values into registers)
        const long r = s_rows[u];
        float dp[VPL];
#pragma unroll
        for (int v = 0; v < VPL; ++v) dp[v] = 0.f;
#pragma unroll
        for (int t = 0; t < MAXT; ++t) {
          if (t < T) {
            const float c = s_wt[u * MAXT + t] * dl[t];
            float hw[VPL];
#pragma unroll
            for (int v = 0; v < VPL; v += 4) {
              const float4 h4 = *reinterpret_cast<const float4*>(s_hw + (long)t * a.d_out + col + v);
              hw[v] = h4.x; hw[v + 1] = h4.y; hw[v + 2] = h4.z; hw[v + 3] = h4.w;
            }
#pragma unroll
            for (int v = 0; v < VPL; ++v) dp[v] = fmaf(c, hw[v], dp[v]);
          }
        }
        if (a.relu_last) {
          float x[VPL];
          load_bf<VPL>(s_o + (long)u * a.d_out + col, x);
#pragma unroll
          for (int v = 0; v < VPL; ++v) dp[v] = x[v] > 0.f ? dp[v] : 0.f;
        }
        store_bf<VPL>(a.dpacked + r * a.ldo + col, dp);
      }
      // dW_head_t += dlogit_t * reps_t
#pragma unroll
      for (int t = 0; t < MAXT; ++t) {
        if (t < T) {
          float x[VPL];
          load_bf<VPL>(s_reps + (long)t * a.d_out + col, x);
#pragma unroll
          for (int v = 0; v < VPL; ++v) acc_dw[t][v] = fmaf(dl[t], x[v], acc_dw[t][v]);
        }
      }
      // router-logit gradient over the (task, pick) pairs (softmax over the active set only)
      if (ws == 0) {
        __nv_bfloat16* dzr = a.dz + (long)b * TE;
        for (int i = lane * 8; i < TE; i += 256) *reinterpret_cast<uint4*>(dzr + i) = make_uint4(0, 0, 0, 0);
        __syncwarp();
        if (!a.dense_probs) {
          for (int i = lane; i < TK; i += 32) {
            const int t = i / K;
            const long o = ((long)t * a.B + b) * K + (i - t * K);
            const int e = a.active[o];
            const float w = a.wsel[o];
            const float p = s_p[union_rank(s_um, e) * ldp + t];
            gw_s[i] = s_dl[t] * p * w;             // g_k w_k
            wf_s[i] = w * __ldg(a.freq + e);       // w_k f_k
          }
          __syncwarp();
          for (int i = lane; i < TK; i += 32) {
            const int t = i / K;
            const long o = ((long)t * a.B + b) * K + (i - t * K);
            float Gt = 0.f, Ft = 0.f;
            for (int k = 0; k < K; ++k) { Gt += gw_s[t * K + k]; Ft += wf_s[t * K + k]; }
            const int e = a.active[o];
            const float w = a.wsel[o];
            // w (g - G) + coef w (f - F)
            dzr[t * E + e] = __float2bfloat16_rn((gw_s[i] - w * Gt) + a.lb_coef * (wf_s[i] - w * Ft));
          }
          __syncwarp();
        } else if (lane < T) {
          const int t = lane;
          const long ob = ((long)t * a.B + b) * K;
          float G2 = 0.f;
          for (int k = 0; k < K; ++k) {
            const int e = a.active[ob + k];
            G2 += s_dl[t] * s_p[union_rank(s_um, e) * ldp + t] * a.wsel[ob + k];
          }
          const float* zr = a.z + (long)b * TE + (long)t * E;
          float mx = -INFINITY;
          for (int e = 0; e < E; ++e) mx = fmaxf(mx, zr[e]);
          float s = 0.f, Fd = 0.f;
          for (int e = 0; e < E; ++e) { float q = expf(zr[e] - mx); s += q; Fd += q * a.freq[e]; }
          Fd /= s;
          __nv_bfloat16* dzt = dzr + (long)t * E;
          for (int e = 0; e < E; ++e) dzt[e] = __float2bfloat16_rn(a.lb_coef * (expf(zr[e] - mx) / s) * (a.freq[e] - Fd));
          for (int k = 0; k < K; ++k) {
            const int e = a.active[ob + k];
            const float w = a.wsel[ob + k];
            const float g = s_dl[t] * s_p[union_rank(s_um, e) * ldp + t];
            dzt[e] = __float2bfloat16_rn(w * (g - G2) + __bfloat162float(dzt[e]));
          }
        }
      }
    }
    __syncthreads();
  }
  // per-CTA head-grad partials: the G groups summed in fixed order through smem
  float* s_red = reinterpret_cast<float*>(smraw);          // reuse: [G][T*d_out] (fits, see combine_smem)
  __syncthreads();
#pragma unroll
  for (int t = 0; t < MAXT; ++t)
    if (t < T)
#pragma unroll
      for (int v = 0; v < VPL; ++v) s_red[(long)gi * n + (long)t * a.d_out + col + v] = acc_dw[t][v];
  float* s_db = s_red + (long)G * n;
  if (gtid < T) s_db[gi * MAXT + gtid] = my_db;
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += CB_THREADS) {
    float s = 0.f;
    for (int g = 0; g < G; ++g) s += s_red[(long)g * n + i];
    a.part_dw[(long)blockIdx.x * n + i] = s;
  }
  if (threadIdx.x < T) {
    float s = 0.f;
    for (int g = 0; g < G; ++g) s += s_db[g * MAXT + threadIdx.x];
    a.part_db[(long)blockIdx.x * T + threadIdx.x] = s;
  }
}

}  // namespace smes

using namespace smes;

static int pick_vpl(int T, int d_out) {
  // VPL columns per thread, S = d_out / (32 VPL) warps per instance (1, 2, 4 or 8)
  int mt = T <= 4 ? 4 : T <= 8 ? 8 : T <= 16 ? 16 : 32;
  int vpl = mt <= 4 ? 8 : 4;      // keep MAXT*VPL <= 32 accumulators per thread (occupancy)
  while (vpl > 4 && d_out / (32 * vpl) < 1) vpl /= 2;
  if (d_out % (32 * vpl)) return -1;
  int s = d_out / (32 * vpl);
  if (s != 1 && s != 2 && s != 4 && s != 8) return -1;
  return vpl;
}

static size_t combine_smem(bool bwd, int T, int K, int d_out, int vpl, int mt, int umax, int ldp, int relu_last) {
  const int S = d_out / (32 * vpl), G = CB_WARPS / S;
  size_t s;
  if (!bwd) {
    GroupLayout L(umax, mt, ldp, umax, d_out);
    s = (size_t)G * L.bytes;
    size_t tail = (size_t)CB_THREADS * 8;
    return s > tail ? s : tail;
  }
  GroupLayout L(umax, mt, ldp, T + (relu_last ? umax : 0), d_out);
  s = (size_t)T * d_out * 4 + (size_t)G * 2 * T * K * 4 + 16 + (size_t)G * L.bytes;
  size_t tail = (size_t)G * T * d_out * 4 + (size_t)G * mt * 4;
  return s > tail ? s : tail;
}

static int combine_launch(bool bwd, CombineArgs& a, int grid, void* stream) {
  if (a.T > CB_MAX_T) return set_error(SMES_ERR_SHAPE, "combine: T=%d exceeds %d", a.T, CB_MAX_T);
  if (a.umax > CB_MAX_U) return set_error(SMES_ERR_SHAPE, "combine: union bound %d exceeds %d", a.umax, CB_MAX_U);
  if (a.E > 1024) return set_error(SMES_ERR_SHAPE, "combine: E=%d exceeds 1024", a.E);
  const int vpl = pick_vpl(a.T, a.d_out);
  if (vpl < 0) return set_error(SMES_ERR_SHAPE, "combine: unsupported d_out=%d for T=%d", a.d_out, a.T);
  if (bwd && ((a.T * a.E) % 8)) return set_error(SMES_ERR_SHAPE, "combine_bwd: T*E must be a multiple of 8");
  if (a.ldp % 4) return set_error(SMES_ERR_SHAPE, "combine: P row stride %d must be a multiple of 4", a.ldp);
  if (a.T * a.K > CB_MAX_TK) return set_error(SMES_ERR_SHAPE, "combine: T*K=%d exceeds %d", a.T * a.K, CB_MAX_TK);
  const int mt = a.T <= 4 ? 4 : a.T <= 8 ? 8 : a.T <= 16 ? 16 : 32;
  const size_t smem = combine_smem(bwd, a.T, a.K, a.d_out, vpl, mt, a.umax, a.ldp > 0 ? a.ldp : 4, a.relu_last);
  if (smem > 227 * 1024) return set_error(SMES_ERR_SHAPE, "combine: shared memory %zu too large", smem);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
#define CB_CASE(V, M)                                                                                    \
  if (vpl == V && mt == M) {                                                                             \
    auto kf = bwd ? combine_bwd_kernel<V, M> : combine_fwd_kernel<V, M>;                                 \
    if (smem > 48 * 1024) cudaFuncSetAttribute(kf, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
    smes_launch(kf, grid, CB_THREADS, smem, st, a);                                                               \
  } else
  CB_CASE(8, 4) CB_CASE(8, 8) CB_CASE(4, 4) CB_CASE(4, 8) CB_CASE(4, 16) CB_CASE(4, 32) {
    return set_error(SMES_ERR_SHAPE, "combine: unsupported T=%d d_out=%d", a.T, a.d_out);
  }
#undef CB_CASE
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_error(SMES_ERR_CUDA, "combine launch: %s", cudaGetErrorString(e));
  return SMES_OK;
}

extern "C" {

int smes_combine_grid(int B, int T, int d_out) {
  const int vpl = pick_vpl(T, d_out);
  const int S = vpl > 0 ? d_out / (32 * vpl) : 1;
  const int G = CB_WARPS / (S > 0 ? S : 1);
  int need = (B + G - 1) / G;
  int g = 148 * 4;     // 4 resident CTAs per SM (register bound): latency hiding for the per-row gathers
  return need < g ? need : g;
}

// SMES_SCORE_KERNEL=0 keeps scoring on the staged combine kernel (A/B)
static bool score_kernel_enabled() {
  static const int on = [] {
    const char* v = std::getenv("SMES_SCORE_KERNEL");
    return (v == nullptr || v[0] != '0') ? 1 : 0;
  }();
  return on != 0;
}

int smes_combine_fwd(int T, int B, int E, int K, int d_out, int umax, const uint32_t* umask, const int32_t* usize,
                     const int32_t* row_of, const int32_t* active, const float* wsel, const void* O, long ldo,
                     const float* head_w, const float* head_b, const float* P, long ldp, void* reps, float* logits, float* preds,
                     const float* labels, const float* lam, double* loss_part, int grid, void* stream) {
  CombineArgs a{};
  a.T = T; a.B = B; a.E = E; a.K = K; a.d_out = d_out; a.umax = umax;
  a.umask = umask; a.usize = usize; a.row_of = row_of; a.active = active; a.wsel = wsel;
  a.O = reinterpret_cast<const __nv_bfloat16*>(O); a.ldo = ldo; a.head_w = head_w; a.head_b = head_b;
  a.P = const_cast<float*>(P); a.ldp = (int)ldp;
  a.reps = reinterpret_cast<__nv_bfloat16*>(reps); a.logits = logits; a.preds = preds; a.labels = labels;
  a.lam = lam; a.loss_part = loss_part;
  if (!reps && O) return set_error(SMES_ERR_STATE, "combine_fwd: reps buffer is required with O");
  if (!O && !P) return set_error(SMES_ERR_STATE, "combine_fwd: scoring without O needs the head projections P");
  if (!O && !labels && !loss_part && T <= 32 && score_kernel_enabled()) {
    // scoring: warp per instance (combine_score_kernel)
    const int tp = T <= 1 ? 1 : T <= 2 ? 2 : T <= 4 ? 4 : T <= 8 ? 8 : T <= 16 ? 16 : 32;
    const int warps = 8;
    long want = ((long)B + warps - 1) / warps;
    const int g = (int)(want < 148L * 8 ? want : 148L * 8);
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    switch (32 / tp) {
      case 32: smes_launch(combine_score_kernel<32>, g, warps * 32, 0, st, a); break;
      case 16: smes_launch(combine_score_kernel<16>, g, warps * 32, 0, st, a); break;
      case 8: smes_launch(combine_score_kernel<8>, g, warps * 32, 0, st, a); break;
      case 4: smes_launch(combine_score_kernel<4>, g, warps * 32, 0, st, a); break;
      case 2: smes_launch(combine_score_kernel<2>, g, warps * 32, 0, st, a); break;
      default: smes_launch(combine_score_kernel<1>, g, warps * 32, 0, st, a); break;
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return set_error(SMES_ERR_CUDA, "combine_score launch: %s", cudaGetErrorString(e));
    return SMES_OK;
  }
  return combine_launch(false, a, grid, stream);
}

int smes_combine_train(int T, int B, int E, int K, int umax, const uint32_t* umask, const int32_t* usize,
                       const int32_t* row_of, const int32_t* active, const float* wsel, const float* head_b,
                       const float* P, long ldp, float* logits, float* preds, const float* labels, const float* lam,
                       double* loss_part, float inv_b, void* cmat, long ldc, void* dz, const float* freq,
                       float lb_coef, float* part_db, float* part_csum, float* part_rb, int grid, void* stream) {
  if (!P || !labels || !cmat || !dz) return set_error(SMES_ERR_STATE, "combine_train: P, labels, C and dz are required");
  if (T > CB_MAX_T) return set_error(SMES_ERR_SHAPE, "combine_train: T=%d exceeds %d", T, CB_MAX_T);
  if (ldc % 8 || ldc < T) return set_error(SMES_ERR_SHAPE, "combine_train: ldc=%ld must be >= T and a multiple of 8", ldc);
  if ((T * E) % 8) return set_error(SMES_ERR_SHAPE, "combine_train: T*E must be a multiple of 8");
  if (umax > CB_MAX_U || T * K > CB_MAX_TK) return set_error(SMES_ERR_SHAPE, "combine_train: union/budget too large");
  CombineArgs a{};
  a.T = T; a.B = B; a.E = E; a.K = K; a.umax = umax;
  a.umask = umask; a.usize = usize; a.row_of = row_of; a.active = active; a.wsel = wsel; a.head_b = head_b;
  a.P = const_cast<float*>(P); a.ldp = (int)ldp; a.logits = logits; a.preds = preds; a.labels = labels; a.lam = lam;
  a.loss_part = loss_part; a.inv_b = inv_b; a.dz = reinterpret_cast<__nv_bfloat16*>(dz); a.freq = freq;
  a.lb_coef = lb_coef; a.part_db = part_db;
  const int mt = T <= 4 ? 4 : T <= 8 ? 8 : T <= 16 ? 16 : 32;
  const int per_warp = 128 + umax * 4 + T * K * 16 + mt * 4 + 64;
  const size_t smem = (size_t)CB_WARPS * ((per_warp + 15) & ~15) +
                      (size_t)CB_WARPS * ((part_csum ? E * T : 0) + (part_rb ? T * E : 0)) * 4;
  if (smem > 200 * 1024) return set_error(SMES_ERR_SHAPE, "combine_train: E*T too large for the fused bias sums");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  auto* cm = reinterpret_cast<__nv_bfloat16*>(cmat);
#define CT_CASE(M)                                                                                      \
  if (mt == M) {                                                                                        \
    if (smem > 48 * 1024) cudaFuncSetAttribute(combine_train_kernel<M>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
    smes_launch(combine_train_kernel<M>, grid, CB_THREADS, smem, st, a, cm, (int)ldc, part_csum, part_rb);      \
  } else
  CT_CASE(4) CT_CASE(8) CT_CASE(16) CT_CASE(32) {}
#undef CT_CASE
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_error(SMES_ERR_CUDA, "combine_train launch: %s", cudaGetErrorString(e));
  return SMES_OK;
}

int smes_bias_from_csum(int E, int T, int d_out, const float* csum, const float* head_w, float* out, void* stream) {
  const int n = E * d_out;
  smes_launch(bias_from_csum_kernel, (n + 255) / 256, 256, 0, reinterpret_cast<cudaStream_t>(stream), E, T, d_out, csum, head_w,
                                                                                           out);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_error(SMES_ERR_CUDA, "bias_from_csum launch: %s", cudaGetErrorString(e));
  return SMES_OK;
}

int smes_combine_bwd(int T, int B, int E, int K, int d_out, int umax, const uint32_t* umask, const int32_t* usize,
                     const int32_t* row_of, const int32_t* active, const float* wsel, const void* O, long ldo,
                     const float* head_w, const float* P, long ldp, const void* reps, const float* preds, const float* labels,
                     const float* lam, float inv_b, int relu_last, void* dpacked, void* dz, const float* freq,
                     float lb_coef, int dense_probs, const float* z, float* part_dw, float* part_db, int grid,
                     void* stream) {
  CombineArgs a{};
  a.T = T; a.B = B; a.E = E; a.K = K; a.d_out = d_out; a.umax = umax;
  a.umask = umask; a.usize = usize; a.row_of = row_of; a.active = active; a.wsel = wsel;
  a.O = reinterpret_cast<const __nv_bfloat16*>(O); a.ldo = ldo; a.head_w = head_w; a.P = const_cast<float*>(P);
  a.ldp = (int)ldp;
  a.reps = reinterpret_cast<__nv_bfloat16*>(const_cast<void*>(reps));
  a.preds = const_cast<float*>(preds); a.labels = labels; a.lam = lam; a.inv_b = inv_b; a.relu_last = relu_last;
  a.dpacked = reinterpret_cast<__nv_bfloat16*>(dpacked); a.dz = reinterpret_cast<__nv_bfloat16*>(dz);
  a.freq = freq; a.lb_coef = lb_coef; a.dense_probs = dense_probs; a.z = z; a.part_dw = part_dw; a.part_db = part_db;
  return combine_launch(true, a, grid, stream);
}

}  // extern "C"
