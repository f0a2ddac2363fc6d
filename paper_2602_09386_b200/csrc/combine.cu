// K4 / K6+K7 -- combine, task heads, BCE, and their backward (gather form, no atomics).
//
// Forward restates `reconstruct_task_reps` (taskmoe/execution.py:161-191) fused
// with `_heads` (taskmoe/model.py:202-208) and the clamped BCE
// (taskmoe/training.py:54-57): every packed row of an instance is loaded ONCE
// and accumulated into all T task representations with the renormalised
// weights; the head dot products, sigmoid and per-instance loss follow in
// registers.
//
// Backward restates training.py:146-179 (+ the LB term of :155-157 and
// balance.py:83-99):
//   dlogit    = lambda_t / B * (yhat - y) * [clamp inactive]                   (:147-148)
//   d_packed  = sum_t w[t,e] dlogit_t head_w_t  (x relu mask if last act relu) (:172-176, :180-181)
//   g[t,k]    = dlogit_t <head_w_t, O[row]>,  dz = w (g - <g,w>) + beta dLB/dz  (:171, :178-179)
//   dW_head_t = sum_b dlogit_t reps_t = sum_rows (w dlogit_t) O[row]            (:151)
// One CTA of S warps owns one instance at a time (persistent grid); head-grad
// partials stay in registers across instances and are reduced in fixed order.
#include "ptx.cuh"
#include "smes_capi.h"

namespace smes {

constexpr int CB_MAX_U = 128;
constexpr int CB_MAX_T = 32;

__device__ __forceinline__ int union_rank(const uint32_t* um, int e) {
  int r = 0;
  for (int j = 0; j < (e >> 5); ++j) r += __popc(um[j]);
  return r + __popc(um[e >> 5] & ((1u << (e & 31)) - 1u));
}

template <int VPL>
__device__ __forceinline__ void load_row(const __nv_bfloat16* p, float (&x)[VPL]) {
  if constexpr (VPL == 8) {
    uint4 v = __ldg(reinterpret_cast<const uint4*>(p));
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&v);
#pragma unroll
    for (int i = 0; i < 4; ++i) { float2 f = __bfloat1622float2(h[i]); x[2 * i] = f.x; x[2 * i + 1] = f.y; }
  } else {
    uint2 v = __ldg(reinterpret_cast<const uint2*>(p));
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&v);
#pragma unroll
    for (int i = 0; i < 2; ++i) { float2 f = __bfloat1622float2(h[i]); x[2 * i] = f.x; x[2 * i + 1] = f.y; }
  }
}
template <int VPL>
__device__ __forceinline__ void store_row(__nv_bfloat16* p, const float (&x)[VPL]) {
  if constexpr (VPL == 8) {
    uint4 v = make_uint4(pack_bf16(x[0], x[1]), pack_bf16(x[2], x[3]), pack_bf16(x[4], x[5]), pack_bf16(x[6], x[7]));
    *reinterpret_cast<uint4*>(p) = v;
  } else {
    uint2 v = make_uint2(pack_bf16(x[0], x[1]), pack_bf16(x[2], x[3]));
    *reinterpret_cast<uint2*>(p) = v;
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
  // forward outputs
  __nv_bfloat16* reps;     // optional (T, B, d_out)
  float* logits;           // (T, B)
  float* preds;            // (T, B)
  const float* labels;     // optional (T, B)
  const float* lam;        // (T,)
  double* loss_part;       // (grid,) per-CTA sum of lambda-weighted BCE
  // backward
  float inv_b;             // 1 / B used in dlogit (training.py:148)
  int relu_last;           // last expert pool is relu: mask d_packed by O > 0 (training.py:180-181)
  __nv_bfloat16* dpacked;  // (rows, ldo)
  __nv_bfloat16* dz;       // (B, T*E) dense
  const float* freq;       // (E,) global selection frequency (balance.py:66)
  float lb_coef;           // beta * E / (K * B * T)  (balance.py:97, training.py:157)
  int dense_probs;         // LB gradient through full_probs (balance.py:96)
  const float* z;          // logits (B, T*E) (dense mode only)
  float* part_dw;          // (grid, T, d_out)
  float* part_db;          // (grid, T)
};

template <int VPL, int MAXT>
__global__ void __launch_bounds__(256) combine_fwd_kernel(const CombineArgs a) {
  const int S = blockDim.x >> 5;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int T = a.T, K = a.K, EW = (a.E + 31) >> 5;
  const int col = threadIdx.x * VPL;
  __shared__ uint32_t s_um[32];
  __shared__ int32_t s_rows[CB_MAX_U];
  __shared__ float s_wt[CB_MAX_U * CB_MAX_T];
  __shared__ float s_red[8][CB_MAX_T];
  double my_loss = 0.0;
  for (int b = blockIdx.x; b < a.B; b += gridDim.x) {
    const int U = a.usize[b];
    for (int j = threadIdx.x; j < EW; j += blockDim.x) s_um[j] = a.umask[(long)b * EW + j];
    for (int u = threadIdx.x; u < U; u += blockDim.x) s_rows[u] = a.row_of[(long)b * a.umax + u];
    for (int i = threadIdx.x; i < U * T; i += blockDim.x) s_wt[i] = 0.f;
    __syncthreads();
    for (int i = threadIdx.x; i < T * K; i += blockDim.x) {
      const int t = i / K;
      const long o = ((long)t * a.B + b) * K + (i - t * K);
      const int u = union_rank(s_um, a.active[o]);
      s_wt[u * T + t] = a.wsel[o];
    }
    __syncthreads();
    float acc[MAXT][VPL];
#pragma unroll
    for (int t = 0; t < MAXT; ++t)
#pragma unroll
      for (int v = 0; v < VPL; ++v) acc[t][v] = 0.f;
    for (int u = 0; u < U; ++u) {
      float x[VPL];
      load_row<VPL>(a.O + (long)s_rows[u] * a.ldo + col, x);
#pragma unroll
      for (int t = 0; t < MAXT; ++t) {
        if (t < T) {
          const float w = s_wt[u * T + t];
#pragma unroll
          for (int v = 0; v < VPL; ++v) acc[t][v] = fmaf(w, x[v], acc[t][v]);
        }
      }
    }
    // heads: logit_t = <head_w_t, reps_t> + head_b_t
#pragma unroll
    for (int t = 0; t < MAXT; ++t) {
      if (t < T) {
        if (a.reps) store_row<VPL>(a.reps + ((long)t * a.B + b) * a.d_out + col, acc[t]);
        float hw[VPL];
        load_f32<VPL>(a.head_w + (long)t * a.d_out + col, hw);
        float p = 0.f;
#pragma unroll
        for (int v = 0; v < VPL; ++v) p = fmaf(hw[v], acc[t][v], p);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) p += __shfl_xor_sync(0xffffffffu, p, o);
        if (lane == 0) s_red[warp][t] = p;
      }
    }
    __syncthreads();
    if (threadIdx.x < T) {
      const int t = threadIdx.x;
      float lg = a.head_b[t];
      for (int w = 0; w < S; ++w) lg += s_red[w][t];
      // stable sigmoid (linalg.py:108-113)
      const float ez = expf(-fabsf(lg));
      const float pos = 1.f / (1.f + ez);
      const float pr = lg >= 0.f ? pos : 1.f - pos;
      a.logits[(long)t * a.B + b] = lg;
      a.preds[(long)t * a.B + b] = pr;
      if (a.labels) {
        // clamped BCE (training.py:54-57), accumulated in fp64
        const double y = a.labels[(long)t * a.B + b];
        double pc = (double)pr;
        pc = pc < 1e-7 ? 1e-7 : (pc > 1.0 - 1e-7 ? 1.0 - 1e-7 : pc);
        my_loss += (double)a.lam[t] * -(y * log(pc) + (1.0 - y) * log1p(-pc));
      }
    }
    __syncthreads();
  }
  if (a.loss_part) {
    // fixed-order CTA reduction of the per-task-thread sums
    __shared__ double s_l[CB_MAX_T];
    if (threadIdx.x < CB_MAX_T) s_l[threadIdx.x] = 0.0;
    __syncthreads();
    if (threadIdx.x < T) s_l[threadIdx.x] = my_loss;
    __syncthreads();
    if (threadIdx.x == 0) {
      double s = 0.0;
      for (int t = 0; t < T; ++t) s += s_l[t];
      a.loss_part[blockIdx.x] = s;
    }
  }
}

template <int VPL, int MAXT>
__global__ void __launch_bounds__(256) combine_bwd_kernel(const CombineArgs a) {
  const int S = blockDim.x >> 5;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int T = a.T, K = a.K, E = a.E, EW = (E + 31) >> 5, TE = T * E;
  const int col = threadIdx.x * VPL;
  __shared__ uint32_t s_um[32];
  __shared__ int32_t s_rows[CB_MAX_U];
  __shared__ float s_wt[CB_MAX_U * CB_MAX_T];
  __shared__ float s_proj[CB_MAX_U * CB_MAX_T];
  __shared__ float s_dl[CB_MAX_T];
  __shared__ float s_red[8][CB_MAX_T];
  float acc_dw[MAXT][VPL];
#pragma unroll
  for (int t = 0; t < MAXT; ++t)
#pragma unroll
    for (int v = 0; v < VPL; ++v) acc_dw[t][v] = 0.f;
  float my_db = 0.f;
  for (int b = blockIdx.x; b < a.B; b += gridDim.x) {
    const int U = a.usize[b];
    for (int j = threadIdx.x; j < EW; j += blockDim.x) s_um[j] = a.umask[(long)b * EW + j];
    for (int u = threadIdx.x; u < U; u += blockDim.x) s_rows[u] = a.row_of[(long)b * a.umax + u];
    for (int i = threadIdx.x; i < U * T; i += blockDim.x) s_wt[i] = 0.f;
    if (threadIdx.x < T) {
      const int t = threadIdx.x;
      const float p = a.preds[(long)t * a.B + b], y = a.labels[(long)t * a.B + b];
      const bool inside = p > 1e-7f && p < 1.f - 1e-7f;
      const float dl = inside ? a.lam[t] * a.inv_b * (p - y) : 0.f;
      s_dl[t] = dl;
      my_db += dl;
    }
    // zero this instance's dz row (dense (B, T*E) operand of the router GEMMs)
    for (int i = threadIdx.x * 8; i < TE; i += blockDim.x * 8)
      *reinterpret_cast<uint4*>(a.dz + (long)b * TE + i) = make_uint4(0, 0, 0, 0);
    __syncthreads();
    for (int i = threadIdx.x; i < T * K; i += blockDim.x) {
      const int t = i / K;
      const long o = ((long)t * a.B + b) * K + (i - t * K);
      const int u = union_rank(s_um, a.active[o]);
      s_wt[u * T + t] = a.wsel[o];
    }
    __syncthreads();
    for (int u = 0; u < U; ++u) {
      const long r = s_rows[u];
      float x[VPL], dp[VPL];
      load_row<VPL>(a.O + r * a.ldo + col, x);
#pragma unroll
      for (int v = 0; v < VPL; ++v) dp[v] = 0.f;
#pragma unroll
      for (int t = 0; t < MAXT; ++t) {
        if (t < T) {
          float hw[VPL];
          load_f32<VPL>(a.head_w + (long)t * a.d_out + col, hw);
          const float c = s_wt[u * T + t] * s_dl[t];
          float p = 0.f;
#pragma unroll
          for (int v = 0; v < VPL; ++v) {
            dp[v] = fmaf(c, hw[v], dp[v]);
            acc_dw[t][v] = fmaf(c, x[v], acc_dw[t][v]);
            p = fmaf(hw[v], x[v], p);
          }
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) p += __shfl_xor_sync(0xffffffffu, p, o);
          if (lane == 0) s_red[warp][t] = p;
        }
      }
      if (a.relu_last) {
#pragma unroll
        for (int v = 0; v < VPL; ++v) dp[v] = x[v] > 0.f ? dp[v] : 0.f;
      }
      store_row<VPL>(a.dpacked + r * a.ldo + col, dp);
      __syncthreads();
      if (threadIdx.x < T) {
        float p = 0.f;
        for (int w = 0; w < S; ++w) p += s_red[w][threadIdx.x];
        s_proj[u * T + threadIdx.x] = p;
      }
      __syncthreads();
    }
    // router-logit gradient, one thread per task (softmax over the active set only)
    if (threadIdx.x < T) {
      const int t = threadIdx.x;
      const long ob = ((long)t * a.B + b) * K;
      float G = 0.f, F = 0.f;
      for (int k = 0; k < K; ++k) {
        const int e = a.active[ob + k];
        const float w = a.wsel[ob + k];
        G += s_dl[t] * s_proj[union_rank(s_um, e) * T + t] * w;
        F += w * a.freq[e];
      }
      __nv_bfloat16* dzr = a.dz + (long)b * TE + (long)t * E;
      if (a.dense_probs) {
        // balance.py:96-99 with full_probs: dense over all E
        const float* zr = a.z + (long)b * TE + (long)t * E;
        float mx = -INFINITY;
        for (int e = 0; e < E; ++e) mx = fmaxf(mx, zr[e]);
        float s = 0.f, Fd = 0.f;
        for (int e = 0; e < E; ++e) { float q = expf(zr[e] - mx); s += q; Fd += q * a.freq[e]; }
        Fd /= s;
        for (int e = 0; e < E; ++e) {
          const float q = expf(zr[e] - mx) / s;
          dzr[e] = __float2bfloat16_rn(a.lb_coef * q * (a.freq[e] - Fd));
        }
      }
      for (int k = 0; k < K; ++k) {
        const int e = a.active[ob + k];
        const float w = a.wsel[ob + k];
        const float g = s_dl[t] * s_proj[union_rank(s_um, e) * T + t];
        float v = w * (g - G);
        if (a.dense_probs) v += __bfloat162float(dzr[e]);
        else v += a.lb_coef * w * (a.freq[e] - F);
        dzr[e] = __float2bfloat16_rn(v);
      }
    }
    __syncthreads();
  }
  // per-CTA head-grad partials
  float* pw = a.part_dw + (long)blockIdx.x * T * a.d_out;
#pragma unroll
  for (int t = 0; t < MAXT; ++t)
    if (t < T)
#pragma unroll
      for (int v = 0; v < VPL; ++v) pw[(long)t * a.d_out + col + v] = acc_dw[t][v];
  if (threadIdx.x < T) a.part_db[(long)blockIdx.x * T + threadIdx.x] = my_db;
}

static int pick_vpl(int T, int d_out) {
  // keep MAXT * VPL <= 128 accumulators per thread
  int vpl = (T <= 8) ? 8 : 4;
  if (d_out / vpl < 32) vpl = 4;
  return vpl;
}

}  // namespace smes

using namespace smes;

static int combine_launch(bool bwd, CombineArgs& a, int grid, void* stream) {
  if (a.T > CB_MAX_T) return set_error(SMES_ERR_SHAPE, "combine: T=%d exceeds %d", a.T, CB_MAX_T);
  if (a.umax > CB_MAX_U) return set_error(SMES_ERR_SHAPE, "combine: union bound %d exceeds %d", a.umax, CB_MAX_U);
  if (a.E > 1024) return set_error(SMES_ERR_SHAPE, "combine: E=%d exceeds 1024", a.E);
  const int vpl = pick_vpl(a.T, a.d_out);
  if (a.d_out % (32 * vpl)) return set_error(SMES_ERR_SHAPE, "combine: d_out=%d must be a multiple of %d", a.d_out, 32 * vpl);
  const int threads = a.d_out / vpl;
  if (threads > 256) return set_error(SMES_ERR_SHAPE, "combine: d_out=%d too large", a.d_out);
  if (bwd && ((a.T * a.E) % 8)) return set_error(SMES_ERR_SHAPE, "combine_bwd: T*E must be a multiple of 8");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const int mt = a.T <= 4 ? 4 : a.T <= 8 ? 8 : a.T <= 16 ? 16 : 32;
#define CB_CASE(V, M)                                                        \
  if (vpl == V && mt == M) {                                                 \
    if (bwd) combine_bwd_kernel<V, M><<<grid, threads, 0, st>>>(a);          \
    else combine_fwd_kernel<V, M><<<grid, threads, 0, st>>>(a);              \
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

int smes_combine_grid(int B) {
  int g = 148 * 16;
  return B < g ? B : g;
}

int smes_combine_fwd(int T, int B, int E, int K, int d_out, int umax, const uint32_t* umask, const int32_t* usize,
                     const int32_t* row_of, const int32_t* active, const float* wsel, const void* O, long ldo,
                     const float* head_w, const float* head_b, void* reps, float* logits, float* preds,
                     const float* labels, const float* lam, double* loss_part, int grid, void* stream) {
  CombineArgs a{};
  a.T = T; a.B = B; a.E = E; a.K = K; a.d_out = d_out; a.umax = umax;
  a.umask = umask; a.usize = usize; a.row_of = row_of; a.active = active; a.wsel = wsel;
  a.O = reinterpret_cast<const __nv_bfloat16*>(O); a.ldo = ldo; a.head_w = head_w; a.head_b = head_b;
  a.reps = reinterpret_cast<__nv_bfloat16*>(reps); a.logits = logits; a.preds = preds; a.labels = labels;
  a.lam = lam; a.loss_part = loss_part;
  return combine_launch(false, a, grid, stream);
}

int smes_combine_bwd(int T, int B, int E, int K, int d_out, int umax, const uint32_t* umask, const int32_t* usize,
                     const int32_t* row_of, const int32_t* active, const float* wsel, const void* O, long ldo,
                     const float* head_w, const float* preds, const float* labels, const float* lam, float inv_b,
                     int relu_last, void* dpacked, void* dz, const float* freq, float lb_coef, int dense_probs,
                     const float* z, float* part_dw, float* part_db, int grid, void* stream) {
  CombineArgs a{};
  a.T = T; a.B = B; a.E = E; a.K = K; a.d_out = d_out; a.umax = umax;
  a.umask = umask; a.usize = usize; a.row_of = row_of; a.active = active; a.wsel = wsel;
  a.O = reinterpret_cast<const __nv_bfloat16*>(O); a.ldo = ldo; a.head_w = head_w;
  a.preds = const_cast<float*>(preds); a.labels = labels; a.lam = lam; a.inv_b = inv_b; a.relu_last = relu_last;
  a.dpacked = reinterpret_cast<__nv_bfloat16*>(dpacked); a.dz = reinterpret_cast<__nv_bfloat16*>(dz);
  a.freq = freq; a.lb_coef = lb_coef; a.dense_probs = dense_probs; a.z = z; a.part_dw = part_dw; a.part_db = part_db;
  return combine_launch(true, a, grid, stream);
}

}  // extern "C"
