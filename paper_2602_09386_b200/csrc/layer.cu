// Combine backward from an arbitrary upstream gradient of the task representations: the reverse
// of reconstruct_task_reps (execution.py:161-191) plus the load-balancing term, for the
// nn.Module / autograd.Function form of the layer (SMESLayer), where the heads and the loss live
// outside the layer.  Restates training.py:160-179 with d_reps given instead of dlogit x head_w:
//
//   d_packed[row(b, e)] = sum_t w[t, b, e] d_reps[t, b]          (x relu mask of O if the last pool is relu)
//   g[t, b, e]          = <d_reps[t, b], O[row(b, e)]>
//   dz[t, b, e]         = w (g - sum_k w_k g_k) + c_lb w (f_e - sum_k w_k f_k)     for e in active_t(b)
//
// with c_lb = dL/dL_lb * E / (K B T) (balance.py:83-99, sparse reading) and dz = 0 off the active
// sets.  One warp per instance; every sum runs in a fixed order (deterministic, no atomics).
#include "ptx.cuh"
#include "smes_capi.h"

namespace smes {

constexpr int LB_WARPS = 4;

struct RepsBwdArgs {
  int T, B, E, K, d_out, umax;
  const uint32_t* umask;       // (B, EW)
  const int32_t* usize;        // (B,)
  const int32_t* row_of;       // (B, umax) packed row of the u-th union member
  const int32_t* active;       // (T, B, K) ascending
  const float* wsel;           // (T, B, K)
  const __nv_bfloat16* O;      // (rows, ldo) packed expert outputs
  long ldo;
  int relu_last;
  const float* d_reps;         // (T, B, d_out)
  const float* freq;           // (E,) LB frequency f
  float lb_coef;
  __nv_bfloat16* dpacked;      // (rows, ldo)
  __nv_bfloat16* dz;           // (B, ldz) row b: [t * E + e]
  long ldz;
};

__device__ __forceinline__ int union_rank_of(const uint32_t* um, int e) {
  int r = 0;
  for (int w = 0; w < (e >> 5); ++w) r += __popc(um[w]);
  return r + __popc(um[e >> 5] & ((1u << (e & 31)) - 1u));
}

__global__ void __launch_bounds__(LB_WARPS * 32) combine_bwd_reps_kernel(const RepsBwdArgs a) {
  pdl_wait();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int b = blockIdx.x * LB_WARPS + warp;
  if (b >= a.B) return;
  const int T = a.T, K = a.K, E = a.E, EW = (E + 31) >> 5;
  extern __shared__ __align__(16) uint8_t smraw[];
  // per warp: union words [EW] | weights [umax][T] | dots [umax][T]
  const int per_warp = EW + 2 * a.umax * T;
  uint32_t* s_um = reinterpret_cast<uint32_t*>(smraw) + (size_t)warp * per_warp;
  float* s_w = reinterpret_cast<float*>(s_um + EW);
  float* s_g = s_w + a.umax * T;
  const int U = a.usize[b];
  for (int j = lane; j < EW; j += 32) s_um[j] = a.umask[(size_t)b * EW + j];
  for (int i = lane; i < U * T; i += 32) { s_w[i] = 0.f; s_g[i] = 0.f; }
  __syncwarp();
  for (int i = lane; i < T * K; i += 32) {
    const int t = i / K;
    const size_t o = ((size_t)t * a.B + b) * K + (i - t * K);
    s_w[union_rank_of(s_um, a.active[o]) * T + t] = a.wsel[o];
  }
  __syncwarp();
  // d_packed rows and the dot products g[u, t]
  for (int u = 0; u < U; ++u) {
    const long r = a.row_of[(size_t)b * a.umax + u];
    float g[32];
#pragma unroll
    for (int t = 0; t < 32; ++t) g[t] = 0.f;
    for (int c = lane; c < a.d_out; c += 32) {
      const float o = __bfloat162float(a.O[r * a.ldo + c]);
      float dp = 0.f;
#pragma unroll
      for (int t = 0; t < 32; ++t) {
        if (t < T) {
          const float w = s_w[u * T + t];
          const float dr = a.d_reps[((size_t)t * a.B + b) * a.d_out + c];
          dp = fmaf(w, dr, dp);
          g[t] = fmaf(dr, o, g[t]);
        }
      }
      a.dpacked[r * a.ldo + c] = __float2bfloat16_rn((a.relu_last && !(o > 0.f)) ? 0.f : dp);
    }
#pragma unroll
    for (int t = 0; t < 32; ++t) {
      if (t < T) {
        float v = g[t];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0) s_g[u * T + t] = v;
      }
    }
  }
  // dz row: zero, then the active entries (lane per task)
  __nv_bfloat16* dzr = a.dz + (size_t)b * a.ldz;
  for (int i = lane; i < T * E; i += 32) dzr[i] = __float2bfloat16_rn(0.f);
  __syncwarp();
  for (int t = lane; t < T; t += 32) {
    const size_t base = ((size_t)t * a.B + b) * K;
    float mg = 0.f, mf = 0.f;
    for (int k = 0; k < K; ++k) {
      const int e = a.active[base + k];
      const float w = a.wsel[base + k];
      mg = fmaf(w, s_g[union_rank_of(s_um, e) * T + t], mg);
      mf = fmaf(w, a.freq[e], mf);
    }
    for (int k = 0; k < K; ++k) {
      const int e = a.active[base + k];
      const float w = a.wsel[base + k];
      const float gk = s_g[union_rank_of(s_um, e) * T + t];
      dzr[t * E + e] = __float2bfloat16_rn(w * (gk - mg) + a.lb_coef * w * (a.freq[e] - mf));
    }
  }
}

}  // namespace smes

using namespace smes;

extern "C" {

int smes_combine_bwd_reps(int T, int B, int E, int K, int d_out, int umax, const uint32_t* umask,
                          const int32_t* usize, const int32_t* row_of, const int32_t* active, const float* wsel,
                          const void* O, long ldo, int relu_last, const float* d_reps, const float* freq,
                          float lb_coef, void* dpacked, void* dz, long ldz, void* stream) {
  if (T < 1 || T > 32) return set_error(SMES_ERR_SHAPE, "combine_bwd_reps: T=%d outside [1, 32]", T);
  if (B < 1 || K < 1 || K > E) return set_error(SMES_ERR_SHAPE, "combine_bwd_reps: B=%d K=%d E=%d", B, K, E);
  if (ldz < (long)T * E) return set_error(SMES_ERR_SHAPE, "combine_bwd_reps: dz stride %ld < T*E", ldz);
  const size_t per_warp = ((size_t)(E + 31) / 32 + 2 * (size_t)umax * T) * 4;
  const size_t smem = per_warp * LB_WARPS;
  if (smem > 200 * 1024) return set_error(SMES_ERR_SHAPE, "combine_bwd_reps: union x tasks too large");
  RepsBwdArgs a{T, B, E, K, d_out, umax, umask, usize, row_of, active, wsel,
                reinterpret_cast<const __nv_bfloat16*>(O), ldo, relu_last, d_reps, freq, lb_coef,
                reinterpret_cast<__nv_bfloat16*>(dpacked), reinterpret_cast<__nv_bfloat16*>(dz), ldz};
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(combine_bwd_reps_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  smes_launch(combine_bwd_reps_kernel, (B + LB_WARPS - 1) / LB_WARPS, LB_WARPS * 32, smem, st, a);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_error(SMES_ERR_CUDA, "combine_bwd_reps launch: %s", cudaGetErrorString(e));
  return SMES_OK;
}

}  // extern "C"
