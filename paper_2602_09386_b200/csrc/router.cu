// K1 -- fused progressive router (one warp per instance row).
//
// Restates `route_batch` (taskmoe/routing.py:235-281) for a whole batch:
//   Stage I   pooled[e] = sum_t w_t softmax(z_t)[e]          (routing.py:256-260)  -- fp64
//             shared    = top_{K_s}(pooled), ties -> lowest index (routing.py:261, :184-187)
//   Stage II  adaptive_t = top_{K_a}(z_t with shared = -inf)    (routing.py:263-268) -- exact fp32 compare
//   active_t  = sort(shared U adaptive_t)                       (routing.py:270-271)
//   weights   = softmax of z_t over active_t                    (routing.py:203-211, :273)
//   union     = OR_t active_t as a bitmask                      (routing.py:272)
// and fuses, per chunk of rows, the histograms the rest of the path needs:
//   union membership per expert   -> plan loads / stable scatter (execution.py:109-113)
//   active counts, sparse mass, dense mass per expert -> LoadStats (balance.py:65-68)
// Stage I is fp64 because reference-init routers give pooled-score gaps down
// to 1e-10; all chunk reductions run in a fixed order (no atomics).
#include "ptx.cuh"
#include "smes_capi.h"

namespace smes {

constexpr int RT_WARPS = 4;
constexpr int RT_MAX_E = 1024;
constexpr int RT_MAX_EPL = RT_MAX_E / 32;

struct RouteArgs {
  const float* z;          // logits, element (t,b,e) at z[t*st + b*sb + e]
  long st, sb;
  const double* probs_in;  // optional (T,B,E) contiguous fp64 (route_batch full_probs=)
  const double* tw;        // (T,) Stage-I pooling weights
  int T, B, E, ks, ka;
  int rows_per_warp;
  int32_t* shared;         // (B, ks)
  int32_t* adaptive;       // (T, B, ka)
  int32_t* active;         // (T, B, K)
  float* wsel;             // (T, B, K) renormalised weights aligned with active
  uint32_t* umask;         // (B, EW)
  int32_t* usize;          // (B,)
  int32_t* chunk_union;    // (C, E)
  int32_t* chunk_active;   // (C, E)
  double* chunk_mass;      // (C, E) sparse mass
  double* chunk_dmass;     // (C, E) dense mass
  double* probs_out;       // optional (T,B,E) fp64 dense softmax
  int32_t* flag;           // non-finite logits seen (sticky)
  int frozen;              // 1: shared/adaptive are inputs (model.py:284-300), weights/stats recomputed
};

template <int EPL>
__device__ __forceinline__ void warp_argmax_f64(const double (&v)[EPL], const uint32_t taken, int lane, int E,
                                                double& best_v, int& best_i) {
  best_v = -INFINITY;
  best_i = 0x7fffffff;
#pragma unroll
  for (int j = 0; j < EPL; ++j) {
    int e = lane + 32 * j;
    if (e < E && !((taken >> j) & 1u)) {
      if (v[j] > best_v || (v[j] == best_v && e < best_i)) { best_v = v[j]; best_i = e; }
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    double ov = __shfl_xor_sync(0xffffffffu, best_v, o);
    int oi = __shfl_xor_sync(0xffffffffu, best_i, o);
    if (ov > best_v || (ov == best_v && oi < best_i)) { best_v = ov; best_i = oi; }
  }
}

template <int EPL>
__device__ __forceinline__ void warp_argmax_f32(const float (&v)[EPL], const uint32_t excl, int lane, int E,
                                                float& best_v, int& best_i) {
  best_v = -INFINITY;
  best_i = 0x7fffffff;
#pragma unroll
  for (int j = 0; j < EPL; ++j) {
    int e = lane + 32 * j;
    if (e < E && !((excl >> j) & 1u)) {
      // -inf (masked shared) entries can still be chosen last, like argsort of +inf (routing.py:265)
      if (best_i == 0x7fffffff || v[j] > best_v || (v[j] == best_v && e < best_i)) { best_v = v[j]; best_i = e; }
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    float ov = __shfl_xor_sync(0xffffffffu, best_v, o);
    int oi = __shfl_xor_sync(0xffffffffu, best_i, o);
    bool ovalid = oi != 0x7fffffff, svalid = best_i != 0x7fffffff;
    if (ovalid && (!svalid || ov > best_v || (ov == best_v && oi < best_i))) { best_v = ov; best_i = oi; }
  }
}

template <int EPL, int TP>
__global__ void __launch_bounds__(RT_WARPS * 32) route_kernel(const RouteArgs a) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int T = a.T, E = a.E, ks = a.ks, ka = a.ka, K = ks + ka;
  const int EW = (E + 31) >> 5;
  extern __shared__ __align__(16) uint8_t sm[];
  // per-warp private accumulators [warp][E]
  int32_t* s_union = reinterpret_cast<int32_t*>(sm);
  int32_t* s_act = s_union + RT_WARPS * E;
  double* s_mass = reinterpret_cast<double*>(s_act + RT_WARPS * E + (E & 1) * RT_WARPS);
  double* s_dmass = s_mass + RT_WARPS * E;
  for (int i = threadIdx.x; i < RT_WARPS * E; i += blockDim.x) {
    s_union[i] = 0; s_act[i] = 0; s_mass[i] = 0.0; s_dmass[i] = 0.0;
  }
  __syncthreads();
  int32_t* w_union = s_union + warp * E;
  int32_t* w_act = s_act + warp * E;
  double* w_mass = s_mass + warp * E;
  double* w_dmass = s_dmass + warp * E;

  const int chunk_rows = RT_WARPS * a.rows_per_warp;
  const int row0 = blockIdx.x * chunk_rows + warp * a.rows_per_warp;
  int bad = 0;
  for (int r = 0; r < a.rows_per_warp; ++r) {
    const int b = row0 + r;
    if (b >= a.B) break;
    // ---------------- load the row's logits (all tasks when T*EPL fits in registers)
    float zpre[TP > 0 ? TP : 1][EPL];
    if (TP > 0) {
#pragma unroll
      for (int t = 0; t < TP; ++t) {
        const float* zr = a.z + (long)t * a.st + (long)b * a.sb;
#pragma unroll
        for (int j = 0; j < EPL; ++j) {
          int e = lane + 32 * j;
          zpre[t][j] = (t < T && e < E) ? __ldg(zr + e) : -INFINITY;
        }
      }
    }
    // ---------------- Stage I (fp64)
    double pooled[EPL];
    double dsum[EPL];
#pragma unroll
    for (int j = 0; j < EPL; ++j) { pooled[j] = 0.0; dsum[j] = 0.0; }
#pragma unroll
    for (int t = 0; t < (TP > 0 ? TP : 1024); ++t) {
      if (t >= T) break;
      const float* zr = a.z + (long)t * a.st + (long)b * a.sb;
      float zv[EPL];
      float mx = -INFINITY;
#pragma unroll
      for (int j = 0; j < EPL; ++j) {
        int e = lane + 32 * j;
        if (TP > 0) zv[j] = zpre[TP > 0 ? t : 0][j];
        else zv[j] = e < E ? __ldg(zr + e) : -INFINITY;
        if (e < E && !isfinite(zv[j])) bad = 1;
        mx = fmaxf(mx, zv[j]);
      }
      const double wt = a.tw[t];
      double p[EPL];
      if (a.probs_in == nullptr) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        double s = 0.0;
#pragma unroll
        for (int j = 0; j < EPL; ++j) {
          int e = lane + 32 * j;
          p[j] = e < E ? exp((double)zv[j] - (double)mx) : 0.0;
          s += p[j];
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        const double inv = 1.0 / s;
#pragma unroll
        for (int j = 0; j < EPL; ++j) p[j] = p[j] / s;
        (void)inv;
      } else {
        const double* pr = a.probs_in + ((long)t * a.B + b) * E;
#pragma unroll
        for (int j = 0; j < EPL; ++j) {
          int e = lane + 32 * j;
          p[j] = e < E ? pr[e] : 0.0;
        }
      }
#pragma unroll
      for (int j = 0; j < EPL; ++j) {
        pooled[j] += wt * p[j];
        dsum[j] += p[j];
      }
      if (a.probs_out != nullptr) {
        double* po = a.probs_out + ((long)t * a.B + b) * E;
#pragma unroll
        for (int j = 0; j < EPL; ++j) {
          int e = lane + 32 * j;
          if (e < E) po[e] = p[j];
        }
      }
    }
    // shared set: K_s rounds of warp argmax on (pooled desc, index asc)
    uint32_t taken = 0;  // bit j: expert lane+32j is shared
    int my_shared = -1;  // lane i < ks holds the i-th pick
    if (a.frozen) {
      const int v = lane < ks ? a.shared[(long)b * ks + lane] : -1;
      for (int i = 0; i < ks; ++i) {
        const int bi = __shfl_sync(0xffffffffu, v, i);
        if ((bi & 31) == lane) taken |= 1u << (bi >> 5);
      }
      my_shared = v;
    } else {
      for (int i = 0; i < ks; ++i) {
        double bv;
        int bi;
        warp_argmax_f64<EPL>(pooled, taken, lane, E, bv, bi);
        if ((bi & 31) == lane) taken |= 1u << (bi >> 5);
        if (lane == i) my_shared = bi;
      }
    }
    // sort the shared picks ascending (rank among the ks lanes)
    int srank = 0;
    for (int j = 0; j < ks; ++j) {
      int o = __shfl_sync(0xffffffffu, my_shared, j);
      if (lane < ks && o < my_shared) ++srank;
    }
    __syncwarp();
    if (lane < ks) a.shared[(long)b * ks + srank] = my_shared;

    // ---------------- Stage II, per task
    uint32_t in_union = taken;  // union bits owned by this lane
#pragma unroll
    for (int t = 0; t < (TP > 0 ? TP : 1024); ++t) {
      if (t >= T) break;
      const float* zr = a.z + (long)t * a.st + (long)b * a.sb;
      float zv[EPL];
#pragma unroll
      for (int j = 0; j < EPL; ++j) {
        int e = lane + 32 * j;
        if (TP > 0) zv[j] = zpre[TP > 0 ? t : 0][j];
        else zv[j] = e < E ? __ldg(zr + e) : -INFINITY;
        if ((taken >> j) & 1u) zv[j] = -INFINITY;
      }
      uint32_t picked = 0;
      int my_pick = -1;  // lane i < ka holds the i-th adaptive pick
      if (a.frozen) {
        const int v = lane < ka ? a.adaptive[((long)t * a.B + b) * ka + lane] : -1;
        for (int i = 0; i < ka; ++i) {
          const int bi = __shfl_sync(0xffffffffu, v, i);
          if ((bi & 31) == lane) picked |= 1u << (bi >> 5);
        }
        my_pick = v;
      } else {
        for (int i = 0; i < ka; ++i) {
          float bv;
          int bi;
          warp_argmax_f32<EPL>(zv, taken | picked, lane, E, bv, bi);
          if ((bi & 31) == lane) picked |= 1u << (bi >> 5);
          if (lane == i) my_pick = bi;
        }
      }
      in_union |= picked;
      int arank = 0;
      for (int j = 0; j < ka; ++j) {
        int o = __shfl_sync(0xffffffffu, my_pick, j);
        if (lane < ka && o < my_pick) ++arank;
      }
      __syncwarp();
      if (lane < ka) a.adaptive[((long)t * a.B + b) * ka + arank] = my_pick;
      // active = sorted(shared U adaptive): lanes 0..K-1 each hold one member
      int val = -1;
      {
        int sv = __shfl_sync(0xffffffffu, my_shared, lane < ks ? lane : 0);
        int av = __shfl_sync(0xffffffffu, my_pick, (lane >= ks && lane < K) ? lane - ks : 0);
        val = lane < ks ? sv : (lane < K ? av : 0x7fffffff);
      }
      int pos = 0;
      for (int j = 0; j < K; ++j) {
        int o = __shfl_sync(0xffffffffu, val, j);
        if (o < val) ++pos;
      }
      float zsel;
      if (TP > 0) {
        // owner lane of expert val holds it in zpre[t][val / 32]
        float mine = 0.f;
        const int src = lane < K ? (val & 31) : 0, jj = lane < K ? (val >> 5) : 0;
#pragma unroll
        for (int j = 0; j < EPL; ++j) {
          float cand = __shfl_sync(0xffffffffu, zpre[TP > 0 ? t : 0][j], src);
          if (j == jj) mine = cand;
        }
        zsel = lane < K ? mine : -INFINITY;
      } else {
        zsel = lane < K ? __ldg(zr + val) : -INFINITY;
      }
      float mx = zsel;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      float ex = lane < K ? expf(zsel - mx) : 0.f;
      float s = ex;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      float w = ex / s;
      if (lane < K) {
        long o = ((long)t * a.B + b) * K + pos;
        a.active[o] = val;
        a.wsel[o] = w;
        w_act[val] += 1;       // distinct vals within a task: no intra-warp race
        w_mass[val] += w;
      }
      __syncwarp();
    }
    // union bitmask words and size; per-expert union / dense-mass accumulation
    int usz = 0;
    for (int j = 0; j < EW; ++j) {
      uint32_t bit = 0;
      if (j < EPL) bit = (in_union >> j) & 1u;
      uint32_t word = __ballot_sync(0xffffffffu, bit != 0);
      usz += __popc(word);
      if (lane == 0) a.umask[(long)b * EW + j] = word;
    }
    if (lane == 0) a.usize[b] = usz;
#pragma unroll
    for (int j = 0; j < EPL; ++j) {
      int e = lane + 32 * j;
      if (e < E) {
        w_union[e] += (in_union >> j) & 1u;
        w_dmass[e] += dsum[j];
      }
    }
    __syncwarp();
  }
  bad = __any_sync(0xffffffffu, bad);
  if (bad && lane == 0) atomicOr(a.flag, 1);
  __syncthreads();
  // chunk partials in fixed warp order
  for (int e = threadIdx.x; e < E; e += blockDim.x) {
    int cu = 0, ca = 0;
    double m = 0.0, dm = 0.0;
    for (int w = 0; w < RT_WARPS; ++w) {
      cu += s_union[w * E + e];
      ca += s_act[w * E + e];
      m += s_mass[w * E + e];
      dm += s_dmass[w * E + e];
    }
    long o = (long)blockIdx.x * E + e;
    a.chunk_union[o] = cu;
    a.chunk_active[o] = ca;
    a.chunk_mass[o] = m;
    a.chunk_dmass[o] = dm;
  }
}

}  // namespace smes

using namespace smes;

extern "C" {

int smes_route_rows_per_warp(int B) {
  int target = B / (148 * 4 * RT_WARPS);
  int rpw = 1;
  while (rpw * 2 <= target && rpw < 64) rpw *= 2;
  return rpw;
}

int smes_route_num_chunks(int B, int rows_per_warp) {
  int cr = RT_WARPS * rows_per_warp;
  return (B + cr - 1) / cr;
}

int smes_route_batch(const float* z, long stride_t, long stride_b, const double* probs_in, const double* task_weights,
                     int T, int B, int E, int k_shared, int k_adaptive, int rows_per_warp, int32_t* shared,
                     int32_t* adaptive, int32_t* active, float* wsel, uint32_t* umask, int32_t* usize,
                     int32_t* chunk_union, int32_t* chunk_active, double* chunk_mass, double* chunk_dmass,
                     double* probs_out, int32_t* flag, int frozen, void* stream) {
  if (T < 1 || B < 1 || E < 1) return set_error(SMES_ERR_SHAPE, "route_batch: empty logits T=%d B=%d E=%d", T, B, E);
  if (E > RT_MAX_E) return set_error(SMES_ERR_SHAPE, "route_batch: E=%d exceeds %d", E, RT_MAX_E);
  if (k_shared < 0 || k_adaptive < 0) return set_error(SMES_ERR_CONFIG, "budget counts must be non-negative");
  if (k_shared + k_adaptive < 1) return set_error(SMES_ERR_CONFIG, "budget must activate at least one expert per task");
  if (k_shared + k_adaptive > E)
    return set_error(SMES_ERR_CONFIG,
                     "budget k=%d exceeds expert count %d: stage-II would have only %d candidates for %d adaptive picks",
                     k_shared + k_adaptive, E, E - k_shared, k_adaptive);
  if (k_shared + k_adaptive > 32) return set_error(SMES_ERR_CONFIG, "budget k=%d exceeds 32", k_shared + k_adaptive);
  RouteArgs a{z, stride_t, stride_b, probs_in, task_weights, T, B, E, k_shared, k_adaptive, rows_per_warp,
              shared, adaptive, active, wsel, umask, usize, chunk_union, chunk_active, chunk_mass, chunk_dmass,
              probs_out, flag, frozen};
  const int C = smes_route_num_chunks(B, rows_per_warp);
  const size_t smem = (size_t)RT_WARPS * (E + 1) * 24 + 64;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const int epl = (E + 31) / 32;
#define RT_LAUNCH_T(N, TPV)                                                                       \
  {                                                                                               \
    if (smem > 48 * 1024)                                                                         \
      cudaFuncSetAttribute(route_kernel<N, TPV>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
    route_kernel<N, TPV><<<C, RT_WARPS * 32, smem, st>>>(a);                                     \
  }
#define RT_LAUNCH(N)                                                                              \
  if (epl <= N) {                                                                                 \
    if (T * N <= 8 && T <= 8 / N) RT_LAUNCH_T(N, (8 / N > 0 ? 8 / N : 1))                         \
    else if (T * N <= 32 && T <= 32 / N) RT_LAUNCH_T(N, (32 / N > 0 ? 32 / N : 1))               \
    else RT_LAUNCH_T(N, 0)                                                                        \
  } else
  RT_LAUNCH(1) RT_LAUNCH(2) RT_LAUNCH(4) RT_LAUNCH(8) RT_LAUNCH(16) RT_LAUNCH(32) {}
#undef RT_LAUNCH
#undef RT_LAUNCH_T
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_error(SMES_ERR_CUDA, "route_batch launch: %s", cudaGetErrorString(e));
  return SMES_OK;
}

}  // extern "C"
