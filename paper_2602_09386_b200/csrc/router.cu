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
#ifndef SMES_RPW_DIV
#define SMES_RPW_DIV 4      // plan chunks: ~SMES_RPW_DIV CTAs of RT_WARPS warps per SM
#endif

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

// ---- order-preserving keys so warp arg-max runs on the REDUX unit (__reduce_max_sync)
__device__ __forceinline__ uint32_t fkey(float f) {
  const uint32_t u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float fkey_inv(uint32_t k) {
  return __uint_as_float((k & 0x80000000u) ? (k & 0x7fffffffu) : ~k);
}
__device__ __forceinline__ uint64_t dkey(double d) {
  const uint64_t u = (uint64_t)__double_as_longlong(d);
  return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}

// arg-max over the warp of (value desc, expert index asc); lane owns experts lane + 32 j.
// Candidates with a set bit in `excl` (bit j) or e >= E are ignored.  Returns the expert.
// e^x - 1 for x <= 0 with relative accuracy (the front / route_rt helper): degree-8 Taylor for
// |x| < 1/4, else ex2.approx(x log2 e) - 1; kRtEpsY bounds the relative error with margin
constexpr float kRtEpsY = 16.f * 0x1p-23f;
__device__ __forceinline__ float rt_expm1_neg(float x) {
  float p = fmaf(x, 1.f / 40320.f, 1.f / 5040.f);
  p = fmaf(x, p, 1.f / 720.f);
  p = fmaf(x, p, 1.f / 120.f);
  p = fmaf(x, p, 1.f / 24.f);
  p = fmaf(x, p, 1.f / 6.f);
  p = fmaf(x, p, 0.5f);
  p = fmaf(x, p, 1.f);
  p *= x;
  float e;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(x * 1.4426950408889634f));
  e -= 1.f;
  return x > -0.25f ? p : e;
}

template <int EPL>
__device__ __forceinline__ int warp_argmax_key32(const uint32_t (&k)[EPL], uint32_t excl, int lane, int E) {
  uint32_t bk = 0;
  int bi = 0x7fffffff;
#pragma unroll
  for (int j = 0; j < EPL; ++j) {
    const int e = lane + 32 * j;
    if (e < E && !((excl >> j) & 1u) && k[j] > bk) { bk = k[j]; bi = e; }   // j ascending: ties keep lower e
  }
  const uint32_t m = __reduce_max_sync(0xffffffffu, bk);
  return __reduce_min_sync(0xffffffffu, (bk == m) ? bi : 0x7fffffff);
}
template <int EPL>
__device__ __forceinline__ int warp_argmax_key64(const uint64_t (&k)[EPL], uint32_t excl, int lane, int E) {
  uint64_t bk = 0;
  int bi = 0x7fffffff;
#pragma unroll
  for (int j = 0; j < EPL; ++j) {
    const int e = lane + 32 * j;
    if (e < E && !((excl >> j) & 1u) && k[j] > bk) { bk = k[j]; bi = e; }
  }
  const uint32_t hi = (uint32_t)(bk >> 32), lo = (uint32_t)bk;
  const uint32_t mh = __reduce_max_sync(0xffffffffu, hi);
  const uint32_t ml = __reduce_max_sync(0xffffffffu, hi == mh ? lo : 0u);
  return __reduce_min_sync(0xffffffffu, (hi == mh && lo == ml) ? bi : 0x7fffffff);
}

// position of each owned expert inside a sorted set given as per-lane bits (bit j: expert lane+32j)
template <int EPL>
__device__ __forceinline__ void sorted_positions(uint32_t bits, int lane, int (&pos)[EPL]) {
  int base = 0;
  const uint32_t lt = (1u << lane) - 1u;
#pragma unroll
  for (int j = 0; j < EPL; ++j) {
    const uint32_t w = __ballot_sync(0xffffffffu, (bits >> j) & 1u);
    pos[j] = base + __popc(w & lt);
    base += __popc(w);
  }
}

// E > 224 (EPL = 8): 8 CTAs per SM (64 registers, a few spills) beat 4 CTAs at 125 registers,
// 1.77 vs 2.07 ms at T = 32, E = 256, B = 32768.
// KS/KA > 0: budget fixed at compile time (selection loops unrolled); PLAIN: not frozen, no
// probs_in / probs_out (the training and scoring path) -- the branches compile away.
template <int EPL, int TP, int KS, int KA, bool PLAIN>
__global__ void __launch_bounds__(RT_WARPS * 32, EPL >= 8 ? 8 : 1) route_kernel(const RouteArgs a) {
  pdl_wait();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int T = a.T, E = a.E, ks = KS > 0 ? KS : a.ks, ka = KA > 0 ? KA : a.ka, K = ks + ka;
  const bool frozen = !PLAIN && a.frozen;
  const double* probs_in = PLAIN ? nullptr : a.probs_in;
  double* probs_out = PLAIN ? nullptr : a.probs_out;
  const int EW = (E + 31) >> 5;
  extern __shared__ __align__(16) uint8_t sm[];
  // per-warp partials [warp][E]: union count, active count, sparse mass, dense mass
  int32_t* s_union = reinterpret_cast<int32_t*>(sm);
  int32_t* s_act = s_union + RT_WARPS * E;
  double* s_mass = reinterpret_cast<double*>(s_act + RT_WARPS * E + (E & 1) * RT_WARPS);
  double* s_dmass = s_mass + RT_WARPS * E;
  // lane-owned accumulators over this warp's rows
  int c_union[EPL], c_act[EPL];
  double c_mass[EPL], c_dmass[EPL];
#pragma unroll
  for (int j = 0; j < EPL; ++j) { c_union[j] = 0; c_act[j] = 0; c_mass[j] = 0.0; c_dmass[j] = 0.0; }

  const int chunk_rows = RT_WARPS * a.rows_per_warp;
  const int row0 = blockIdx.x * chunk_rows + warp * a.rows_per_warp;
  int bad = 0;
  for (int r = 0; r < a.rows_per_warp; ++r) {
    const int b = row0 + r;
    if (b >= a.B) break;
    // ---------------- the row's logits (registers when T * EPL is small)
    float zpre[TP > 0 ? TP : 1][EPL];
    if (TP > 0) {
#pragma unroll
      for (int t = 0; t < TP; ++t) {
        const float* zr = a.z + (long)t * a.st + (long)b * a.sb;
#pragma unroll
        for (int j = 0; j < EPL; ++j) {
          const int e = lane + 32 * j;
          zpre[t][j] = (t < T && e < E) ? __ldg(zr + e) : -INFINITY;
        }
      }
    }
    auto load_task = [&](int t, float (&zv)[EPL]) {
      if (TP > 0) {
#pragma unroll
        for (int tt = 0; tt < (TP > 0 ? TP : 1); ++tt)
          if (tt == t) {
#pragma unroll
            for (int j = 0; j < EPL; ++j) zv[j] = zpre[tt][j];
          }
      } else {
        const float* zr = a.z + (long)t * a.st + (long)b * a.sb;
#pragma unroll
        for (int j = 0; j < EPL; ++j) {
          const int e = lane + 32 * j;
          zv[j] = e < E ? __ldg(zr + e) : -INFINITY;
        }
      }
    };
    // ---------------- Stage I, fast path (training / scoring rows without dense statistics):
    // deviation form in fp32 (front.cu / route_rt.cu): P_e = sum_t (w_t / S_t) y_te with
    // y = e^(z - max) - 1 and S_t = E + sum_e y_te ranks like the pooled scores; the set is accepted
    // when a certified bound separates it, else this row (the whole warp) takes the fp64 path below
    uint32_t taken = 0;  // bit j: expert lane + 32 j is shared
    bool exact = true;
    if (PLAIN && a.chunk_dmass == nullptr && ks > 0) {
      float P[EPL];
#pragma unroll
      for (int j = 0; j < EPL; ++j) P[j] = 0.f;
      float perr = 0.f;
      auto fast_task = [&](int t, const float (&zv)[EPL]) {
        uint32_t mk = 0, nk = 0xffffffffu;
#pragma unroll
        for (int j = 0; j < EPL; ++j) {
          const int e = lane + 32 * j;
          if (e < E) {
            if (!isfinite(zv[j])) bad = 1;
            mk = max(mk, fkey(zv[j]));
            nk = min(nk, fkey(zv[j]));
          }
        }
        const float mx = fkey_inv(__reduce_max_sync(0xffffffffu, mk));
        const float mn = fkey_inv(__reduce_min_sync(0xffffffffu, nk));
        float y[EPL], ys = 0.f;
#pragma unroll
        for (int j = 0; j < EPL; ++j) {
          const int e = lane + 32 * j;
          y[j] = e < E ? rt_expm1_neg(zv[j] - mx) : 0.f;
          ys += y[j];
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) ys += __shfl_xor_sync(0xffffffffu, ys, o);
        const float ssum = (float)E + ys;
        const float q = (float)a.tw[t] / ssum;
#pragma unroll
        for (int j = 0; j < EPL; ++j) P[j] = fmaf(q, y[j], P[j]);
        // |error| of q y_tj <= q |y|max (eps_y + rho_t + 3u) (rho_t: S's EPL + 5 roundings and the y
        // errors, relative to S); the accumulation over the tasks adds T u
        const float rho = ((EPL + 5) * 0x1p-24f + kRtEpsY) * (-ys) / ssum + 0x1p-24f;
        perr += q * (-rt_expm1_neg(mn - mx)) * (kRtEpsY + rho + (3 + T) * 0x1p-24f);
      };
      if (TP > 0) {
#pragma unroll
        for (int t = 0; t < (TP > 0 ? TP : 1); ++t)
          if (t < T) fast_task(t, zpre[t]);
      } else {
        for (int t = 0; t < T; ++t) {
          float zv[EPL];
          load_task(t, zv);
          fast_task(t, zv);
        }
      }
      uint32_t pk[EPL];
#pragma unroll
      for (int j = 0; j < EPL; ++j) {
        const uint32_t u = __float_as_uint(P[j]);
        pk[j] = (u & 0x80000000u) ? ~u : (u | 0x80000000u);     // order-preserving (P may be negative)
      }
      for (int i = 0; i < ks; ++i) {
        const int bi = warp_argmax_key32<EPL>(pk, taken, lane, E);
        if ((bi & 31) == lane) taken |= 1u << (bi >> 5);
      }
      const float e_abs = 1.5f * perr + 0x1p-100f;
      float lo = INFINITY, hi = -INFINITY;
#pragma unroll
      for (int j = 0; j < EPL; ++j) {
        const int e = lane + 32 * j;
        if (e < E) {
          if ((taken >> j) & 1u) lo = fminf(lo, P[j] - e_abs);
          else hi = fmaxf(hi, P[j] + e_abs);
        }
      }
      const float lo_all = fkey_inv(__reduce_min_sync(0xffffffffu, fkey(lo)));
      const float hi_all = fkey_inv(__reduce_max_sync(0xffffffffu, fkey(hi)));
      exact = !(lo_all > hi_all);
      if (exact) taken = 0;
    }
    // ---------------- Stage I (fp64): pooled = sum_t w_t softmax(z_t)   (routing.py:256-260)
    double pooled[EPL];
#pragma unroll
    for (int j = 0; j < EPL; ++j) pooled[j] = 0.0;
    auto stage1_task = [&](int t, const float (&zv)[EPL]) {
      double p[EPL];
      if (probs_in == nullptr) {
        uint32_t mk = 0;
#pragma unroll
        for (int j = 0; j < EPL; ++j) {
          const int e = lane + 32 * j;
          if (e < E) {
            if (!isfinite(zv[j])) bad = 1;
            mk = max(mk, fkey(zv[j]));
          }
        }
        const double mx = (double)fkey_inv(__reduce_max_sync(0xffffffffu, mk));
        double sum = 0.0;
#pragma unroll
        for (int j = 0; j < EPL; ++j) {
          const int e = lane + 32 * j;
          p[j] = e < E ? exp((double)zv[j] - mx) : 0.0;
          sum += p[j];
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
        const double inv_sum = 1.0 / sum;
#pragma unroll
        for (int j = 0; j < EPL; ++j) p[j] *= inv_sum;
      } else {
        const double* pr = probs_in + ((long)t * a.B + b) * E;
#pragma unroll
        for (int j = 0; j < EPL; ++j) {
          const int e = lane + 32 * j;
          p[j] = e < E ? pr[e] : 0.0;
          if (e < E && !isfinite(zv[j])) bad = 1;
        }
      }
      const double wt = a.tw[t];
#pragma unroll
      for (int j = 0; j < EPL; ++j) {
        pooled[j] += wt * p[j];
        c_dmass[j] += p[j];
      }
      if (probs_out != nullptr) {
        double* po = probs_out + ((long)t * a.B + b) * E;
#pragma unroll
        for (int j = 0; j < EPL; ++j) {
          const int e = lane + 32 * j;
          if (e < E) po[e] = p[j];
        }
      }
    };
    if (exact) {
      if (TP > 0) {
        // T <= TP: fully unrolled task loop, logits indexed statically from registers
#pragma unroll
        for (int t = 0; t < (TP > 0 ? TP : 1); ++t)
          if (t < T) stage1_task(t, zpre[t]);
      } else {
        for (int t = 0; t < T; ++t) {
          float zv[EPL];
          load_task(t, zv);
          stage1_task(t, zv);
        }
      }
    }
    // shared set S: top-K_s of pooled, (score desc, index asc)   (routing.py:261, :184-187)
    if (!exact) {
      // decided by the fast path
    } else if (frozen) {
      const int v = lane < ks ? a.shared[(long)b * ks + lane] : -1;
      for (int i = 0; i < ks; ++i) {
        const int bi = __shfl_sync(0xffffffffu, v, i);
        if ((bi & 31) == lane) taken |= 1u << (bi >> 5);
      }
    } else if (ks > 0) {
      uint64_t pk[EPL];
#pragma unroll
      for (int j = 0; j < EPL; ++j) pk[j] = dkey(pooled[j]);
      for (int i = 0; i < ks; ++i) {
        const int bi = warp_argmax_key64<EPL>(pk, taken, lane, E);
        if ((bi & 31) == lane) taken |= 1u << (bi >> 5);
      }
    }
    {
      int pos[EPL];
      sorted_positions<EPL>(taken, lane, pos);
      __syncwarp();
#pragma unroll
      for (int j = 0; j < EPL; ++j)
        if ((taken >> j) & 1u) a.shared[(long)b * ks + pos[j]] = lane + 32 * j;
    }

    // ---------------- Stage II per task: top-K_a of z_t with S excluded (routing.py:263-268)
    uint32_t in_union = taken;
    auto stage2_task = [&](int t, const float (&zv)[EPL]) {
      uint32_t picked = 0;
      const long ot = ((long)t * a.B + b);
      if (frozen) {
        const int v = lane < ka ? a.adaptive[ot * ka + lane] : -1;
        for (int i = 0; i < ka; ++i) {
          const int bi = __shfl_sync(0xffffffffu, v, i);
          if ((bi & 31) == lane) picked |= 1u << (bi >> 5);
        }
      } else if (ka > 0) {
        uint32_t zk[EPL];
#pragma unroll
        for (int j = 0; j < EPL; ++j) zk[j] = fkey(zv[j]);
        for (int i = 0; i < ka; ++i) {
          const int bi = warp_argmax_key32<EPL>(zk, taken | picked, lane, E);
          if ((bi & 31) == lane) picked |= 1u << (bi >> 5);
        }
      }
      in_union |= picked;
      const uint32_t act = taken | picked;
      int apos[EPL], kpos[EPL];
      sorted_positions<EPL>(picked, lane, apos);
      sorted_positions<EPL>(act, lane, kpos);
      // renormalised weights: softmax of z over the active set (routing.py:203-211)
      uint32_t mk = 0;
#pragma unroll
      for (int j = 0; j < EPL; ++j)
        if ((act >> j) & 1u) mk = max(mk, fkey(zv[j]));
      const float mx = fkey_inv(__reduce_max_sync(0xffffffffu, mk));
      float ex[EPL], sum = 0.f;
#pragma unroll
      for (int j = 0; j < EPL; ++j) {
        ex[j] = ((act >> j) & 1u) ? expf(zv[j] - mx) : 0.f;
        sum += ex[j];
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
      const float inv = 1.f / sum;
      __syncwarp();
#pragma unroll
      for (int j = 0; j < EPL; ++j) {
        const int e = lane + 32 * j;
        if ((picked >> j) & 1u) a.adaptive[ot * ka + apos[j]] = e;
        if ((act >> j) & 1u) {
          const float w = ex[j] / sum;
          a.active[ot * K + kpos[j]] = e;
          a.wsel[ot * K + kpos[j]] = w;
          c_act[j] += 1;
          c_mass[j] += (double)w;
        }
      }
      (void)inv;
    };
    if (TP > 0) {
#pragma unroll
      for (int t = 0; t < (TP > 0 ? TP : 1); ++t)
        if (t < T) stage2_task(t, zpre[t]);
    } else {
      for (int t = 0; t < T; ++t) {
        float zv[EPL];
        load_task(t, zv);
        stage2_task(t, zv);
      }
    }
    // union bitmask words and size (routing.py:272)
    int usz = 0;
#pragma unroll
    for (int j = 0; j < EPL; ++j) {
      if (j >= EW) break;
      uint32_t bit = 0;
#pragma unroll
      for (int jj = 0; jj < EPL; ++jj)
        if (jj == j) bit = (in_union >> jj) & 1u;
      const uint32_t word = __ballot_sync(0xffffffffu, bit != 0);
      usz += __popc(word);
      if (lane == 0) a.umask[(long)b * EW + j] = word;
    }
    if (lane == 0) a.usize[b] = usz;
#pragma unroll
    for (int j = 0; j < EPL; ++j) c_union[j] += (in_union >> j) & 1u;
  }
  bad = __any_sync(0xffffffffu, bad);
  if (bad && lane == 0) atomicOr(a.flag, 1);
#pragma unroll
  for (int j = 0; j < EPL; ++j) {
    const int e = lane + 32 * j;
    if (e < E) {
      s_union[warp * E + e] = c_union[j];
      s_act[warp * E + e] = c_act[j];
      s_mass[warp * E + e] = c_mass[j];
      s_dmass[warp * E + e] = c_dmass[j];
    }
  }
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
    const long o = (long)blockIdx.x * E + e;
    a.chunk_union[o] = cu;
    a.chunk_active[o] = ca;
    a.chunk_mass[o] = m;
    if (a.chunk_dmass != nullptr) a.chunk_dmass[o] = dm;
  }
}


// ============================================================================ task-grouped router
// route_tg_kernel<T, E, KS, KA>: the same decisions as route_kernel for the training / scoring
// path (not frozen, no probs in/out) with a different lane map: the warp's lanes are T groups of
// L = 32/T, lane (t, q) owns task t's logits of experts [q*EPT, (q+1)*EPT), EPT = E/L.  Every
// per-task reduction (softmax max / sum, Stage-II top-K_a, the active-set softmax) is then a
// log2(L)-level shuffle done for all T tasks at once, where the expert-per-lane map needs a
// 5-level warp reduction per task.  Stage-I pooling is a fixed-order reduce-scatter over the task
// bits, leaving lane (t, q) with the pooled scores of experts q*EPT + t*R + i, R = EPT/T.
// Tie rules as routing.py:184-187 (score desc, index asc); Stage I in fp64.
template <int T, int E, int KS, int KA>
#ifndef SMES_TG_MINB
#define SMES_TG_MINB 8      // 32 warps per SM: occupancy beats the few spills (tools/route_time.py)
#endif
__global__ void __launch_bounds__(RT_WARPS * 32, SMES_TG_MINB) route_tg_kernel(const RouteArgs a) {
  pdl_wait();
  constexpr int L = 32 / T, EPT = E / L, R = EPT / T, K = KS + KA, EW = (E + 31) / 32;
  static_assert(32 % T == 0 && E % L == 0 && EPT % T == 0 && E <= 64, "route_tg shape");
  using mask_t = unsigned long long;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int t = lane / L, q = lane % L;
  const int e0 = q * EPT;                     // first owned expert (Stage II / softmax view)
  const int p0 = e0 + t * R;                  // first owned pooled expert (after reduce-scatter)
  extern __shared__ __align__(16) uint8_t sm[];
  int32_t* s_union = reinterpret_cast<int32_t*>(sm);
  int32_t* s_act = s_union + RT_WARPS * E;
  double* s_mass = reinterpret_cast<double*>(s_act + RT_WARPS * E + (E & 1) * RT_WARPS);
  double* s_dmass = s_mass + RT_WARPS * E;
  // per-(task, expert) running partials of this warp's rows, one owner lane each (shared memory
  // keeps them out of the register file: 4 x EPT accumulators spilled at 128 registers)
  double* w_mass = s_dmass + RT_WARPS * E + (size_t)warp * 2 * T * E;     // [T][E]
  double* w_dmass = w_mass + T * E;                                         // [T][E]
  int32_t* w_act = reinterpret_cast<int32_t*>(s_dmass + RT_WARPS * E + (size_t)RT_WARPS * 2 * T * E) +
                   (size_t)warp * (T + 1) * E;                              // [T][E] + union [E]
  int32_t* w_union = w_act + T * E;
#pragma unroll
  for (int j = 0; j < EPT; ++j) {
    w_mass[t * E + e0 + j] = 0.0;
    w_dmass[t * E + e0 + j] = 0.0;
    w_act[t * E + e0 + j] = 0;
    if (t == 0) w_union[e0 + j] = 0;
  }
  const double wt = a.tw[t];
  const int chunk_rows = RT_WARPS * a.rows_per_warp;
  const int row0 = blockIdx.x * chunk_rows + warp * a.rows_per_warp;
  int bad = 0;
  for (int r = 0; r < a.rows_per_warp; ++r) {
    const int b = row0 + r;
    if (b >= a.B) break;
    float z[EPT];
    {
      const float* zr = a.z + (long)t * a.st + (long)b * a.sb + e0;
      if constexpr (EPT % 4 == 0) {
#pragma unroll
        for (int j = 0; j < EPT; j += 4) {
          const float4 v = __ldg(reinterpret_cast<const float4*>(zr + j));
          z[j] = v.x; z[j + 1] = v.y; z[j + 2] = v.z; z[j + 3] = v.w;
        }
      } else {
#pragma unroll
        for (int j = 0; j < EPT; ++j) z[j] = __ldg(zr + j);
      }
    }
    // ---------------- Stage I (fp64): dense softmax per task, pooled = sum_t w_t p_t
    uint32_t mk = 0;
#pragma unroll
    for (int j = 0; j < EPT; ++j) {
      if (!isfinite(z[j])) bad = 1;
      mk = max(mk, fkey(z[j]));
    }
#pragma unroll
    for (int o = 1; o < L; o <<= 1) mk = max(mk, __shfl_xor_sync(0xffffffffu, mk, o));
    const double mx = (double)fkey_inv(mk);
    double v[EPT], sum = 0.0;
#pragma unroll
    for (int j = 0; j < EPT; ++j) { v[j] = exp((double)z[j] - mx); sum += v[j]; }
#pragma unroll
    for (int o = 1; o < L; o <<= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    const double inv = 1.0 / sum;
#pragma unroll
    for (int j = 0; j < EPT; ++j) {
      const double pj = v[j] * inv;
      w_dmass[t * E + e0 + j] += pj;
      v[j] = wt * pj;
    }
    // reduce-scatter over the task bits (highest first): lane keeps the half its bit selects
#pragma unroll
    for (int s = 0, len = EPT; len > R; ++s, len >>= 1) {
      const int o = (T >> (s + 1)) * L;
      const bool upper = (lane & o) != 0;
      const int half = len >> 1;
#pragma unroll
      for (int i = 0; i < EPT / 2; ++i) {
        if (i < half) {
          const double send = upper ? v[i] : v[i + half];
          const double keep = upper ? v[i + half] : v[i];
          v[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
        }
      }
    }
    // shared set: top-K_s of pooled, (score desc, index asc)   (routing.py:261)
    mask_t smask = 0;
    {
      uint64_t pk[R];
#pragma unroll
      for (int i = 0; i < R; ++i) pk[i] = dkey(v[i]);
#pragma unroll
      for (int k = 0; k < KS; ++k) {
        uint64_t bk = 0;
        int bi = 0x7fffffff;
#pragma unroll
        for (int i = 0; i < R; ++i)
          if (!((smask >> (p0 + i)) & 1ull) && pk[i] > bk) { bk = pk[i]; bi = p0 + i; }
        const uint32_t hi = (uint32_t)(bk >> 32), lo = (uint32_t)bk;
        const uint32_t mh = __reduce_max_sync(0xffffffffu, hi);
        const uint32_t ml = __reduce_max_sync(0xffffffffu, hi == mh ? lo : 0u);
        const int win = __reduce_min_sync(0xffffffffu, (hi == mh && lo == ml) ? bi : 0x7fffffff);
        smask |= 1ull << win;
      }
    }
    // Stage II: top-K_a of z_t with the shared set excluded, within the task's L lanes
    uint32_t tk[KA];
    int ti[KA];
#pragma unroll
    for (int k = 0; k < KA; ++k) { tk[k] = 0; ti[k] = 0x7fffffff; }
#pragma unroll
    for (int j = 0; j < EPT; ++j) {
      if ((smask >> (e0 + j)) & 1ull) continue;
      uint32_t ck = fkey(z[j]);
      int ci = e0 + j;
#pragma unroll
      for (int k = 0; k < KA; ++k) {            // insertion into the descending list
        if (ck > tk[k] || (ck == tk[k] && ci < ti[k])) {
          const uint32_t xk = tk[k]; const int xi = ti[k];
          tk[k] = ck; ti[k] = ci; ck = xk; ci = xi;
        }
      }
    }
#pragma unroll
    for (int o = 1; o < L; o <<= 1) {           // merge the partner's list
      uint32_t ok[KA];
      int oi[KA];
#pragma unroll
      for (int k = 0; k < KA; ++k) {
        ok[k] = __shfl_xor_sync(0xffffffffu, tk[k], o);
        oi[k] = __shfl_xor_sync(0xffffffffu, ti[k], o);
      }
#pragma unroll
      for (int m = 0; m < KA; ++m) {
        uint32_t ck = ok[m];
        int ci = oi[m];
#pragma unroll
        for (int k = 0; k < KA; ++k) {
          if (ck > tk[k] || (ck == tk[k] && ci < ti[k])) {
            const uint32_t xk = tk[k]; const int xi = ti[k];
            tk[k] = ck; ti[k] = ci; ck = xk; ci = xi;
          }
        }
      }
    }
    mask_t amask = 0;
#pragma unroll
    for (int k = 0; k < KA; ++k) amask |= 1ull << ti[k];
    const mask_t act = smask | amask;
    // renormalised weights: softmax of z over the active set (routing.py:203-211)
    uint32_t ak = 0;
#pragma unroll
    for (int j = 0; j < EPT; ++j)
      if ((act >> (e0 + j)) & 1ull) ak = max(ak, fkey(z[j]));
#pragma unroll
    for (int o = 1; o < L; o <<= 1) ak = max(ak, __shfl_xor_sync(0xffffffffu, ak, o));
    const float amx = fkey_inv(ak);
    float ex[EPT], asum = 0.f;
#pragma unroll
    for (int j = 0; j < EPT; ++j) {
      ex[j] = ((act >> (e0 + j)) & 1ull) ? expf(z[j] - amx) : 0.f;
      asum += ex[j];
    }
#pragma unroll
    for (int o = 1; o < L; o <<= 1) asum += __shfl_xor_sync(0xffffffffu, asum, o);
    const long ot = (long)t * a.B + b;
#pragma unroll
    for (int j = 0; j < EPT; ++j) {
      const int e = e0 + j;
      const mask_t below = (1ull << e) - 1ull;
      if ((act >> e) & 1ull) {
        const float w = ex[j] / asum;
        const int pos = __popcll(act & below);
        a.active[ot * K + pos] = e;
        a.wsel[ot * K + pos] = w;
        w_act[t * E + e] += 1;
        w_mass[t * E + e] += (double)w;
      }
      if ((amask >> e) & 1ull) a.adaptive[ot * KA + __popcll(amask & below)] = e;
      if (t == 0 && ((smask >> e) & 1ull)) a.shared[(long)b * KS + __popcll(smask & below)] = e;
    }
    // union over tasks (routing.py:272)
    mask_t un = amask;
#pragma unroll
    for (int o = L; o < 32; o <<= 1) un |= __shfl_xor_sync(0xffffffffu, un, o);
    un |= smask;
    if (lane == 0) {
#pragma unroll
      for (int w = 0; w < EW; ++w) a.umask[(long)b * EW + w] = (uint32_t)(un >> (32 * w));
      a.usize[b] = __popcll(un);
    }
    if (t == 0) {
#pragma unroll
      for (int j = 0; j < EPT; ++j) w_union[e0 + j] += (int)((un >> (e0 + j)) & 1ull);
    }
  }
  bad = __any_sync(0xffffffffu, bad);
  if (bad && lane == 0) atomicOr(a.flag, 1);
  // per-(task, expert) partials -> per-expert in task order (fixed order)
  __syncwarp();
  for (int e = lane; e < E; e += 32) {
    int ca = 0;
    double m = 0.0, dm = 0.0;
    for (int tt = 0; tt < T; ++tt) {
      ca += w_act[tt * E + e];
      m += w_mass[tt * E + e];
      dm += w_dmass[tt * E + e];
    }
    s_union[warp * E + e] = w_union[e];
    s_act[warp * E + e] = ca;
    s_mass[warp * E + e] = m;
    s_dmass[warp * E + e] = dm;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < E; e += blockDim.x) {
    int cu = 0, ca = 0;
    double m = 0.0, dm = 0.0;
    for (int w = 0; w < RT_WARPS; ++w) {
      cu += s_union[w * E + e];
      ca += s_act[w * E + e];
      m += s_mass[w * E + e];
      dm += s_dmass[w * E + e];
    }
    const long o = (long)blockIdx.x * E + e;
    a.chunk_union[o] = cu;
    a.chunk_active[o] = ca;
    a.chunk_mass[o] = m;
    if (a.chunk_dmass != nullptr) a.chunk_dmass[o] = dm;
  }
}

}  // namespace smes

using namespace smes;

extern "C" {

int smes_route_rows_per_warp(int B) {
  int target = B / (148 * SMES_RPW_DIV * RT_WARPS);
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
  // training / scoring mode without dense-mass statistics: the (row, task) router (route_rt.cu)
  if (!frozen && probs_in == nullptr && probs_out == nullptr && chunk_dmass == nullptr &&
      smes_route_rt_supported(T, E, k_shared, k_adaptive) && (stride_t % 4) == 0 && (stride_b % 4) == 0 &&
      (reinterpret_cast<uintptr_t>(z) % 16) == 0)
    return smes_route_rt(z, stride_t, stride_b, task_weights, T, B, E, k_shared, k_adaptive, rows_per_warp, shared,
                         adaptive, active, wsel, umask, usize, chunk_union, chunk_active, chunk_mass, chunk_dmass,
                         flag, stream);
  RouteArgs a{z, stride_t, stride_b, probs_in, task_weights, T, B, E, k_shared, k_adaptive, rows_per_warp,
              shared, adaptive, active, wsel, umask, usize, chunk_union, chunk_active, chunk_mass, chunk_dmass,
              probs_out, flag, frozen};
  const int C = smes_route_num_chunks(B, rows_per_warp);
  const size_t smem = (size_t)RT_WARPS * (E + 1) * 24 + 64;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const int epl = (E + 31) / 32;
  const bool plain = !frozen && probs_in == nullptr && probs_out == nullptr;
  const bool b42 = k_shared == 4 && k_adaptive == 2;
#define RT_LAUNCH_K(N, TPV, KS, KA, PL)                                                           \
  {                                                                                               \
    if (smem > 48 * 1024)                                                                         \
      cudaFuncSetAttribute(route_kernel<N, TPV, KS, KA, PL>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                           (int)smem);                                                            \
    smes_launch(route_kernel<N, TPV, KS, KA, PL>, C, RT_WARPS * 32, smem, st, a);                         \
  }
#define RT_LAUNCH_T(N, TPV)                                                                       \
  {                                                                                               \
    if (plain && b42) RT_LAUNCH_K(N, TPV, 4, 2, true)                                             \
    else RT_LAUNCH_K(N, TPV, 0, 0, false)                                                         \
  }
#define RT_LAUNCH(N)                                                                              \
  if (epl <= N) {                                                                                 \
    if (T * N <= 8 && T <= 8 / N) RT_LAUNCH_T(N, (8 / N > 0 ? 8 / N : 1))                         \
    else if (T * N <= 32 && T <= 32 / N) RT_LAUNCH_T(N, (32 / N > 0 ? 32 / N : 1))               \
    else RT_LAUNCH_T(N, 0)                                                                        \
  } else
  // task-grouped kernel: + per-warp (task, expert) partials (2 doubles + 1 int) and union counts
  const size_t smem_tg = smem + (size_t)RT_WARPS * ((size_t)T * E * 20 + E * 4) + 64;
#define RT_TG(TT, EE)                                                                             \
  if (plain && b42 && T == TT && E == EE) {                                                        \
    if (smem_tg > 48 * 1024)                                                                      \
      cudaFuncSetAttribute(route_tg_kernel<TT, EE, 4, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_tg); \
    smes_launch(route_tg_kernel<TT, EE, 4, 2>, C, RT_WARPS * 32, smem_tg, st, a);                            \
  } else
  RT_TG(8, 32) RT_TG(4, 32)
  RT_LAUNCH(1) RT_LAUNCH(2) RT_LAUNCH(4) RT_LAUNCH(8) RT_LAUNCH(16) RT_LAUNCH(32) {}
#undef RT_TG
#undef RT_LAUNCH
#undef RT_LAUNCH_T
#undef RT_LAUNCH_K
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_error(SMES_ERR_CUDA, "route_batch launch: %s", cudaGetErrorString(e));
  return SMES_OK;
}

}  // extern "C"
