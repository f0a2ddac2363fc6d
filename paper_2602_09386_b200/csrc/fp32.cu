// fp32 arithmetic mode of the SMES forward (BASELINE c1; the north star's "fp32 1e-5" contract).
//
// The reference computes in float64 NumPy (taskmoe/linalg.py:3-8).  The fp32 mode keeps every
// operand in fp32 and runs the dense contractions on the tensor cores as bf16x3 products
// (smes_gemm_ragged_m_x3 in gemm.cu): each fp32 operand is split into three bf16 planes
// x = x0 + x1 + x2 (24 significant bits, exact for normal fp32 values), and the six leading cross
// products accumulate in the fp32 TMEM accumulator, so the GEMM matches an fp32 FFMA GEMM to
// within fp32 rounding.  This file holds the two pieces around those GEMMs:
//
//   split_bf16x3      fp32 (rows, cols) -> bf16 planes [x0 | x1 | x2] (rows, 3 cols)   (HBM-bound)
//   combine_fwd_f32   reconstruct_task_reps (execution.py:161-191) + _heads (model.py:202-208)
//                     + clamped BCE (training.py:54-57) in fp32 with a double loss sum
#include "ptx.cuh"
#include "smes_capi.h"

namespace smes {

__global__ void __launch_bounds__(256) split_bf16x3_kernel(long rows, int cols, const float* __restrict__ src,
                                                            long lds, __nv_bfloat16* __restrict__ dst, long ldd,
                                                            const int32_t* __restrict__ rows_dev) {
  pdl_wait();
  if (rows_dev != nullptr) rows = min(rows, (long)*rows_dev);
  const int q = cols >> 2;                       // float4 groups per row
  const long n = rows * q;
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) {
    const long r = i / q;
    const int c = (int)(i - r * q) * 4;
    const float4 v = __ldg(reinterpret_cast<const float4*>(src + r * lds + c));
    const float x[4] = {v.x, v.y, v.z, v.w};
    uint32_t p[3][2];
#pragma unroll
    for (int j = 0; j < 4; j += 2) {
      float a = x[j], b = x[j + 1];
#pragma unroll
      for (int s = 0; s < 3; ++s) {
        const __nv_bfloat16 ha = __float2bfloat16_rn(a), hb = __float2bfloat16_rn(b);
        p[s][j >> 1] = (uint32_t)__bfloat16_as_ushort(ha) | ((uint32_t)__bfloat16_as_ushort(hb) << 16);
        a -= __bfloat162float(ha);              // exact: the residual of a round-to-nearest
        b -= __bfloat162float(hb);
      }
    }
    __nv_bfloat16* o = dst + r * ldd + c;
#pragma unroll
    for (int s = 0; s < 3; ++s) *reinterpret_cast<uint2*>(o + (long)s * cols) = make_uint2(p[s][0], p[s][1]);
  }
}

constexpr int CF_THREADS = 128;

__device__ __forceinline__ int union_rank_f32(const uint32_t* um, int e) {
  int r = 0;
  for (int j = 0; j < (e >> 5); ++j) r += __popc(um[j]);
  return r + __popc(um[e >> 5] & ((1u << (e & 31)) - 1u));
}

// optional loss finalize by the last CTA (smes_combine_fwd_f32_loss)
struct LossTail {
  int* ticket;                   // zero before the launch; the last CTA resets it
  double inv_b, beta;
  const double* stats_value;     // L_lb (LoadStats value) or null
  double* loss_out;              // [task, lb, total]
};

// One instance per CTA iteration (grid-stride).  Thread = columns col, col + 128, ...; the union's
// packed rows are read from L2 once per task (d_out * U * 4 bytes, L1-resident across tasks).
__global__ void __launch_bounds__(CF_THREADS)
    combine_fwd_f32_kernel(int T, int B, int E, int K, int d_out, int umax, const uint32_t* __restrict__ umask,
                           const int32_t* __restrict__ usize, const int32_t* __restrict__ row_of,
                           const int32_t* __restrict__ active, const float* __restrict__ wsel,
                           const float* __restrict__ O, long ldo, const float* __restrict__ head_w,
                           const float* __restrict__ head_b, float* __restrict__ reps, float* __restrict__ logits,
                           float* __restrict__ preds, const float* __restrict__ labels, const float* __restrict__ lam,
                           double* __restrict__ loss_part, const LossTail tail) {
  pdl_wait();
  extern __shared__ __align__(16) uint8_t sm[];
  const int EW = (E + 31) >> 5;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint32_t* s_um = reinterpret_cast<uint32_t*>(sm);
  int32_t* s_rows = reinterpret_cast<int32_t*>(s_um + EW);
  float* s_wt = reinterpret_cast<float*>(s_rows + umax);            // [umax][T]
  float* s_part = s_wt + (size_t)umax * T;                           // [T][4 warps]
  double* s_loss = reinterpret_cast<double*>(sm);                    // reused after the loop
  double my_loss = 0.0;
  for (int b = blockIdx.x; b < B; b += gridDim.x) {
    const int U = usize[b];
    for (int j = threadIdx.x; j < EW; j += CF_THREADS) s_um[j] = umask[(long)b * EW + j];
    for (int u = threadIdx.x; u < U; u += CF_THREADS) s_rows[u] = row_of[(long)b * umax + u];
    for (int i = threadIdx.x; i < U * T; i += CF_THREADS) s_wt[i] = 0.f;
    __syncthreads();
    for (int i = threadIdx.x; i < T * K; i += CF_THREADS) {
      const int t = i / K;
      const long o = ((long)t * B + b) * K + (i - t * K);
      s_wt[union_rank_f32(s_um, active[o]) * T + t] = wsel[o];
    }
    __syncthreads();
    for (int t = 0; t < T; ++t) {
      float part = 0.f;
      for (int col = threadIdx.x; col < d_out; col += CF_THREADS) {
        float acc = 0.f;
        for (int u = 0; u < U; ++u) {
          const float w = s_wt[u * T + t];
          if (w != 0.f) acc = fmaf(w, __ldg(O + (long)s_rows[u] * ldo + col), acc);
        }
        reps[((long)t * B + b) * d_out + col] = acc;
        part = fmaf(acc, __ldg(head_w + (long)t * d_out + col), part);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
      if (lane == 0) s_part[t * (CF_THREADS / 32) + warp] = part;
    }
    __syncthreads();
    for (int t = threadIdx.x; t < T; t += CF_THREADS) {
      float lg = head_b[t];
#pragma unroll
      for (int w = 0; w < CF_THREADS / 32; ++w) lg += s_part[t * (CF_THREADS / 32) + w];
      const float ez = expf(-fabsf(lg));                 // stable sigmoid (linalg.py:108-113)
      const float pos = 1.f / (1.f + ez);
      const float pr = lg >= 0.f ? pos : 1.f - pos;
      logits[(long)t * B + b] = lg;
      preds[(long)t * B + b] = pr;
      if (labels != nullptr) {
        const double y = labels[(long)t * B + b];
        double pc = (double)pr;
        pc = pc < 1e-7 ? 1e-7 : (pc > 1.0 - 1e-7 ? 1.0 - 1e-7 : pc);
        my_loss += (double)lam[t] * -(y * log(pc) + (1.0 - y) * log1p(-pc));
      }
    }
    __syncthreads();
  }
  if (loss_part != nullptr) {
    __syncthreads();
    s_loss[threadIdx.x] = my_loss;
    __syncthreads();
    if (threadIdx.x == 0) {
      double s = 0.0;
      for (int i = 0; i < CF_THREADS; ++i) s += s_loss[i];
      loss_part[blockIdx.x] = s;
    }
    if (tail.ticket != nullptr) {
      // loss finalize in the last CTA to finish (training.py:60-94): the partials in a fixed order
      __shared__ int s_last;
      if (threadIdx.x == 0) {
        __threadfence();
        s_last = atomicAdd(tail.ticket, 1) == (int)gridDim.x - 1;
      }
      __syncthreads();
      if (s_last) {
        __threadfence();
        double v = 0.0;
        for (int i = threadIdx.x; i < (int)gridDim.x; i += CF_THREADS) v += __ldcg(loss_part + i);
        s_loss[threadIdx.x] = v;
        __syncthreads();
        if (threadIdx.x == 0) {
          double t = 0.0;
          for (int i = 0; i < CF_THREADS; ++i) t += s_loss[i];
          const double task = t * tail.inv_b;
          const double lb = tail.stats_value ? *tail.stats_value : 0.0;
          tail.loss_out[0] = task;
          tail.loss_out[1] = lb;
          tail.loss_out[2] = task + tail.beta * lb;
          *tail.ticket = 0;                          // ready for the next launch (graph replays)
        }
      }
    }
  }
}

}  // namespace smes

using namespace smes;

extern "C" {

int smes_split_bf16x3(long rows, int cols, const float* src, long lds, void* dst, long ldd, const int32_t* rows_dev,
                      void* stream) {
  if (rows < 0 || cols <= 0 || cols % 4 || lds % 4 || ldd % 4 || ldd < 3L * cols)
    return set_error(SMES_ERR_SHAPE, "split_bf16x3: cols=%d, lds=%ld, ldd=%ld (need cols %% 4 == 0, ldd >= 3 cols)",
                     cols, lds, ldd);
  if (rows == 0) return SMES_OK;
  const long n = rows * (cols / 4);
  const long want = (n + 255) / 256;
  const int grid = (int)(want < 148L * 16 ? want : 148L * 16);
  smes_launch(split_bf16x3_kernel, grid, 256, 0, reinterpret_cast<cudaStream_t>(stream), 
      rows, cols, src, lds, reinterpret_cast<__nv_bfloat16*>(dst), ldd, rows_dev);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_error(SMES_ERR_CUDA, "split_bf16x3 launch: %s", cudaGetErrorString(e));
  return SMES_OK;
}

int smes_combine_fwd_f32_grid(int B) { return B < 148 * 8 ? B : 148 * 8; }

static int combine_f32_impl(int T, int B, int E, int K, int d_out, int umax, const uint32_t* umask,
                            const int32_t* usize, const int32_t* row_of, const int32_t* active, const float* wsel,
                            const float* O, long ldo, const float* head_w, const float* head_b, float* reps,
                            float* logits, float* preds, const float* labels, const float* lam, double* loss_part,
                            int grid, const LossTail& tail, void* stream) {
  if (T < 1 || B < 1 || E < 1 || K < 1 || d_out < 1 || umax < 1)
    return set_error(SMES_ERR_SHAPE, "combine_fwd_f32: empty shape");
  if (!O || !reps || !logits || !preds) return set_error(SMES_ERR_STATE, "combine_fwd_f32: missing buffer");
  const int EW = (E + 31) / 32;
  size_t smem = (size_t)(EW + umax) * 4 + (size_t)umax * T * 4 + (size_t)T * (CF_THREADS / 32) * 4;
  smem = (smem + 15) & ~(size_t)15;
  if (smem < CF_THREADS * sizeof(double)) smem = CF_THREADS * sizeof(double);
  if (smem > 227 * 1024) return set_error(SMES_ERR_SHAPE, "combine_fwd_f32: union x tasks too large");
  if (smem > 48 * 1024) {
    cudaError_t ea = cudaFuncSetAttribute(combine_fwd_f32_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)smem);
    if (ea != cudaSuccess) return set_error(SMES_ERR_CUDA, "combine_fwd_f32 smem: %s", cudaGetErrorString(ea));
  }
  smes_launch(combine_fwd_f32_kernel, grid, CF_THREADS, smem, reinterpret_cast<cudaStream_t>(stream), 
      T, B, E, K, d_out, umax, umask, usize, row_of, active, wsel, O, ldo, head_w, head_b, reps, logits, preds, labels,
      lam, loss_part, tail);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_error(SMES_ERR_CUDA, "combine_fwd_f32 launch: %s", cudaGetErrorString(e));
  return SMES_OK;
}

int smes_combine_fwd_f32(int T, int B, int E, int K, int d_out, int umax, const uint32_t* umask, const int32_t* usize,
                         const int32_t* row_of, const int32_t* active, const float* wsel, const float* O, long ldo,
                         const float* head_w, const float* head_b, float* reps, float* logits, float* preds,
                         const float* labels, const float* lam, double* loss_part, int grid, void* stream) {
  return combine_f32_impl(T, B, E, K, d_out, umax, umask, usize, row_of, active, wsel, O, ldo, head_w, head_b, reps,
                          logits, preds, labels, lam, loss_part, grid, LossTail{nullptr, 0.0, 0.0, nullptr, nullptr},
                          stream);
}

int smes_combine_fwd_f32_loss(int T, int B, int E, int K, int d_out, int umax, const uint32_t* umask,
                              const int32_t* usize, const int32_t* row_of, const int32_t* active, const float* wsel,
                              const float* O, long ldo, const float* head_w, const float* head_b, float* reps,
                              float* logits, float* preds, const float* labels, const float* lam, double* loss_part,
                              int grid, int32_t* ticket, double inv_b, double beta, const double* stats_value,
                              double* loss_out, void* stream) {
  if (labels == nullptr || loss_part == nullptr || ticket == nullptr || loss_out == nullptr)
    return set_error(SMES_ERR_STATE, "combine_fwd_f32_loss: labels, partials, ticket and loss_out are required");
  return combine_f32_impl(T, B, E, K, d_out, umax, umask, usize, row_of, active, wsel, O, ldo, head_w, head_b, reps,
                          logits, preds, labels, lam, loss_part, grid,
                          LossTail{ticket, inv_b, beta, stats_value, loss_out}, stream);
}

}  // extern "C"
