// K1 (logits in HBM) -- progressive router, one thread per (instance row, task).
//
// route_batch (taskmoe/routing.py:235-281) for the configurations whose logits do not fit the
// fused TMEM front (T*E > 256: c3/c4 T=16, E=64), training / scoring mode (not frozen, no dense
// probabilities in or out, no dense-mass statistics).  A group of G = next_pow2(T) lanes owns one
// row; lane t owns task t's E logits in registers:
//
//   Stage I  fp32 exponentials of z_t - max_t (ex2.approx), the task's softmax sum, and the
//            pooled contributions w_t p_te, reduce-scattered over the group (lane l ends with the
//            pooled scores of experts [l E/G, (l+1) E/G)); shared = top-K_s by group arg-max
//            (score desc, index asc, routing.py:256-261, :184-187).  A certified bound on the
//            fp32 error accepts the set when every selected expert's lower bound exceeds every
//            other expert's upper bound; otherwise the group recomputes Stage I entirely in fp64
//            (exp, sums, pooling), so the selections equal an fp64 evaluation.
//   Stage II exact fp32 compare of z_t with the shared set excluded (routing.py:263-268), the
//            active set sorted ascending (:270-271), weights = softmax of z_t over it (:203-211).
//   Chunk statistics (the plan's chunks of 4 * rows_per_warp rows, one per CTA): union and
//            active counts as shared-memory integer atomics (order-free, exact), sparse mass in
//            per-thread shared-memory slots reduced in a fixed order (deterministic).
//
// The expert-per-lane route_kernel (router.cu) needed ~7.5 k warp instructions per c3 row; this
// layout ~0.8 k.
#include "ptx.cuh"
#include "smes_capi.h"

namespace smes {
namespace rt {

constexpr int kThreads = 128;

struct Args {
  const float* z;          // element (t, b, e) at z[t*st + b*sb + e]
  long st, sb;
  const double* tw;        // (T,)
  int T, B, rows_per_cta;
  int32_t* shared;         // (B, KS)
  int32_t* adaptive;       // (T, B, KA)
  int32_t* active;         // (T, B, K)
  float* wsel;             // (T, B, K)
  uint32_t* umask;         // (B, EW)
  int32_t* usize;          // (B,)
  int32_t* chunk_union;    // (C, E)
  int32_t* chunk_active;
  double* chunk_mass;
  double* chunk_dmass;     // zeroed (no dense-mass reading in this mode)
  int32_t* flag;
  int32_t* n_exact;        // optional diagnostic: rows through the fp64 recompute
};

__device__ __forceinline__ float fast_exp(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x * 1.4426950408889634f));
  return y;
}

template <int N>
__device__ __forceinline__ float tree_max(const float (&z)[N]) {
  float m[N / 2];
#pragma unroll
  for (int j = 0; j < N / 2; ++j) m[j] = fmaxf(z[j], z[j + N / 2]);
#pragma unroll
  for (int s = N / 4; s > 0; s >>= 1)
#pragma unroll
    for (int j = 0; j < s; ++j) m[j] = fmaxf(m[j], m[j + s]);
  return m[0];
}
template <int N>
__device__ __forceinline__ float tree_min(const float (&z)[N]) {
  float m[N / 2];
#pragma unroll
  for (int j = 0; j < N / 2; ++j) m[j] = fminf(z[j], z[j + N / 2]);
#pragma unroll
  for (int s = N / 4; s > 0; s >>= 1)
#pragma unroll
    for (int j = 0; j < s; ++j) m[j] = fminf(m[j], m[j + s]);
  return m[0];
}
template <int N, typename V>
__device__ __forceinline__ V tree_sum(const V (&z)[N]) {
  V m[N / 2];
#pragma unroll
  for (int j = 0; j < N / 2; ++j) m[j] = z[j] + z[j + N / 2];
#pragma unroll
  for (int s = N / 4; s > 0; s >>= 1)
#pragma unroll
    for (int j = 0; j < s; ++j) m[j] = m[j] + m[j + s];
  return m[0];
}

// Reduce-scatter of V values over a group of G lanes (V % G == 0): afterwards x[0 .. V/G) of lane
// l hold the group sums of values [l V/G, (l+1) V/G).  Fixed butterfly order (deterministic).
template <int V, int G, typename T>
__device__ __forceinline__ void reduce_scatter(T (&x)[V], unsigned gm, int gl) {
#pragma unroll
  for (int s = 0; (G >> (s + 1)) > 0; ++s) {
    const int o = G >> (s + 1);
    const int half = (V >> s) / 2;
    const bool up = (gl & o) != 0;
#pragma unroll
    for (int i = 0; i < half; ++i) {
      const T send = up ? x[i] : x[half + i];
      const T keep = up ? x[half + i] : x[i];
      x[i] = keep + __shfl_xor_sync(gm, send, o);
    }
  }
}

// (key desc, index asc) arg-max over a group of G lanes
template <int G, typename K>
__device__ __forceinline__ void group_argmax(K& key, int& idx, unsigned gm) {
#pragma unroll
  for (int o = G / 2; o > 0; o >>= 1) {
    const K k2 = __shfl_xor_sync(gm, key, o);
    const int i2 = __shfl_xor_sync(gm, idx, o);
    const bool take = (k2 > key) | ((k2 == key) & (i2 < idx));
    key = take ? k2 : key;
    idx = take ? i2 : idx;
  }
}

template <int G>
__device__ __forceinline__ float group_max(float v, unsigned gm) {
#pragma unroll
  for (int o = G / 2; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(gm, v, o));
  return v;
}
template <int G>
__device__ __forceinline__ double group_min_d(double v, unsigned gm) {
#pragma unroll
  for (int o = G / 2; o > 0; o >>= 1) v = fmin(v, __shfl_xor_sync(gm, v, o));
  return v;
}
template <int G>
__device__ __forceinline__ double group_max_d(double v, unsigned gm) {
#pragma unroll
  for (int o = G / 2; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(gm, v, o));
  return v;
}
template <int G>
__device__ __forceinline__ unsigned long long group_or(unsigned long long v, unsigned gm) {
#pragma unroll
  for (int o = G / 2; o > 0; o >>= 1) v |= __shfl_xor_sync(gm, v, o);
  return v;
}

// top-K_s of this group's owned pooled scores (PER per lane, experts [gl PER, ...)), ties to the
// lowest index; keys are the IEEE bit patterns of the non-negative scores
template <int PER, int G, int KS, typename K>
__device__ __forceinline__ unsigned long long select_shared_keys(const K (&keys)[PER], unsigned gm, int gl) {
  unsigned long long smask = 0ull;
  uint32_t taken = 0;
#pragma unroll
  for (int k = 0; k < KS; ++k) {
    K key = 0;
    int idx = 0x7fffffff;
#pragma unroll
    for (int i = 0; i < PER; ++i) {
      const bool take = !((taken >> i) & 1u) && (idx == 0x7fffffff || keys[i] > key);
      key = take ? keys[i] : key;
      idx = take ? gl * PER + i : idx;
    }
    group_argmax<G, K>(key, idx, gm);
    smask |= 1ull << idx;
    if (idx / PER == gl) taken |= 1u << (idx - gl * PER);
  }
  return smask;
}
template <int PER, int G, int KS, typename P, typename K>
__device__ __forceinline__ unsigned long long select_shared(const P (&v)[PER], unsigned gm, int gl) {
  return select_shared_keys<PER, G, KS, K>(v, gm, gl);
}

// order-preserving u32 key of a float (any sign); +-0 map apart, but equal-valued candidates are
// never certified (their bounds overlap), so the tie rule is the exact path's
__device__ __forceinline__ uint32_t okey(float f) {
  const uint32_t u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

// e^x - 1 for x <= 0 with relative accuracy: |x| < 1/4 a degree-8 Taylor polynomial (truncation
// 4e-11, ~3 ulp of rounding), else ex2.approx(x log2 e) - 1 ((2 + 1.173 |x|) ulp of e^x, <= 8.2 ulp
// of |y| for x <= -1/4).  kEpsY bounds both with the argument rounding, with margin.
constexpr float kEpsY = 16.f * 0x1p-23f;
__device__ __forceinline__ float expm1_neg(float x) {
  float p = fmaf(x, 1.f / 40320.f, 1.f / 5040.f);
  p = fmaf(x, p, 1.f / 720.f);
  p = fmaf(x, p, 1.f / 120.f);
  p = fmaf(x, p, 1.f / 24.f);
  p = fmaf(x, p, 1.f / 6.f);
  p = fmaf(x, p, 0.5f);
  p = fmaf(x, p, 1.f);
  p *= x;
  const float e = fast_exp(x) - 1.f;
  return x > -0.25f ? p : e;
}

template <int E, int G, int KS, int KA>
__global__ void __launch_bounds__(kThreads) route_rt_kernel(const Args a) {
  pdl_wait();
  constexpr int K = KS + KA;
  constexpr int PER = E / G;                       // pooled scores owned per lane
  constexpr int NG = kThreads / G;                 // row groups per CTA
  constexpr int LOG2E = E == 16 ? 4 : E == 32 ? 5 : 6;
  constexpr int LOG2G = G == 4 ? 2 : G == 8 ? 3 : G == 16 ? 4 : 5;
  static_assert(G <= E && E % G == 0 && G <= 32, "group layout");
  extern __shared__ __align__(16) uint8_t sm[];
  float* s_mass = reinterpret_cast<float*>(sm);                    // [kThreads][E + 1]
  float* s_row = s_mass + kThreads * (E + 1);                      // [kThreads][E] Stage-II logit rows
  int32_t* s_act = reinterpret_cast<int32_t*>(s_row + kThreads * E);   // [E]
  int32_t* s_uni = s_act + E;                                      // [E]

  const int tid = threadIdx.x, lane = tid & 31;
  const int gl = lane & (G - 1);                   // task of this lane
  const int grp = tid / G;
  const unsigned gm = G == 32 ? 0xffffffffu : (((1u << G) - 1u) << (lane & ~(G - 1)));
  const int T = a.T;
  const bool has_t = gl < T;
  for (int i = tid; i < kThreads * (E + 1); i += kThreads) s_mass[i] = 0.f;
  for (int i = tid; i < E; i += kThreads) { s_act[i] = 0; s_uni[i] = 0; }
  __syncthreads();
  const int r0 = blockIdx.x * a.rows_per_cta;
  const int r1 = min(r0 + a.rows_per_cta, a.B);
  const double twt = has_t ? a.tw[gl] : 0.0;
  float* my_mass = s_mass + tid * (E + 1);
  float* my_row = s_row + tid * E;
  constexpr int SW = (E / 4 < 8 ? E / 4 : 8) - 1;    // 16-byte chunk swizzle of the per-thread row
  const int swz = tid & SW;
  int bad = 0, n_exact = 0;
  for (int b = r0 + grp; b < r1; b += NG) {
    const float* zr = a.z + (long)gl * a.st + (long)b * a.sb;
    // ---------------- Stage I, fast path: pooled_e = sum_t w_t/S_t + P_e with
    //   y_te = exp(z_te - max_t) - 1 (relative accuracy even when |y| is tiny), S_t = E + sum_e y_te,
    //   P_e = sum_t (w_t / S_t) y_te.  The first term is the same for every expert, so the shared
    //   set is the top-K_s of P.  At reference init |y| ~ 1e-3, so P's absolute error is ~1e-3 of
    //   the pooled scores' (a plain fp32 softmax cannot separate the ~1e-7 gaps of E = 64).
    float c[E];
    float mx = -INFINITY, amax = 0.f;
    if (has_t) {
#pragma unroll
      for (int j = 0; j < E; j += 4) {
        const float4 v = __ldg(reinterpret_cast<const float4*>(zr + j));
        c[j] = v.x; c[j + 1] = v.y; c[j + 2] = v.z; c[j + 3] = v.w;
      }
      mx = tree_max<E>(c);
      const float mn = tree_min<E>(c);
#pragma unroll
      for (int j = 0; j < E; ++j) c[j] = expm1_neg(c[j] - mx);
      const float ysum = tree_sum<E, float>(c);       // <= 0
      const float ssum = (float)E + ysum;
      bad |= !(isfinite(mx) & isfinite(mn) & isfinite(ssum));
      const float q = (float)twt / ssum;
#pragma unroll
      for (int j = 0; j < E; ++j) c[j] *= q;
      // |error| of every q y_tj <= q |y|max (eps_y + rho_t + (3 + log2 G) u):  eps_y the expm1 bound,
      // rho_t the relative error of S_t (its log2 E roundings and the y errors, relative to S)
      const float rho = (LOG2E * 0x1p-24f + kEpsY) * (-ysum) / ssum + 0x1p-24f;
      amax = q * (-expm1_neg(mn - mx)) * (kEpsY + rho + (3 + LOG2G) * 0x1p-24f);
    } else {
#pragma unroll
      for (int j = 0; j < E; ++j) c[j] = 0.f;
    }
    reduce_scatter<E, G, float>(c, gm, gl);        // c[0 .. PER): P of experts [gl PER, ...)
    unsigned long long smask = 0ull;
    if constexpr (KS > 0) {
      float err = amax;
#pragma unroll
      for (int o = G / 2; o > 0; o >>= 1) err += __shfl_xor_sync(gm, err, o);
      uint32_t pk[PER];
#pragma unroll
      for (int i = 0; i < PER; ++i) pk[i] = okey(c[i]);
      smask = select_shared<PER, G, KS, uint32_t, uint32_t>(pk, gm, gl);
      // certification (x 1.5 margin, + an absolute floor for flushed exps)
      const double e_abs = 1.5 * (double)err + 0x1p-100;
      double lo = INFINITY, hi = -INFINITY;
#pragma unroll
      for (int i = 0; i < PER; ++i) {
        const double p = (double)c[i];
        const bool sel = (smask >> (gl * PER + i)) & 1ull;
        lo = sel ? fmin(lo, p - e_abs) : lo;
        hi = sel ? hi : fmax(hi, p + e_abs);
      }
      lo = group_min_d<G>(lo, gm);
      hi = group_max_d<G>(hi, gm);
      if (!(lo > hi)) {
        // ---------------- Stage I, exact path (fp64), the whole group
        ++n_exact;
        double s = 0.0;
        if (has_t) {
          for (int j = 0; j < E; ++j) s += exp((double)__ldg(zr + j) - (double)mx);
        }
        const double qd = has_t ? twt / s : 0.0;
        double pd[PER];
#pragma unroll
        for (int i = 0; i < PER; ++i) pd[i] = 0.0;
        // E / G rounds of a G-wide reduce-scatter: round i gives lane l expert i G + l ... reduce
        // each round's G contributions, then keep this lane's owned experts
#pragma unroll
        for (int rr = 0; rr < PER; ++rr) {
          double v[G];
#pragma unroll
          for (int u = 0; u < G; ++u) {
            const int j = u * PER + rr;             // expert owned (after the scatter) by lane u, slot rr
            v[u] = has_t ? qd * exp((double)__ldg(zr + j) - (double)mx) : 0.0;
          }
          reduce_scatter<G, G, double>(v, gm, gl);
          pd[rr] = v[0];
        }
        unsigned long long dk[PER];
#pragma unroll
        for (int i = 0; i < PER; ++i) dk[i] = (unsigned long long)__double_as_longlong(pd[i]);   // pooled >= 0
        smask = select_shared_keys<PER, G, KS, unsigned long long>(dk, gm, gl);
      }
      if (gl == 0) {
        unsigned long long m = smask;
#pragma unroll
        for (int k = 0; k < KS; ++k) {
          a.shared[(long)b * KS + k] = __ffsll((long long)m) - 1;
          m &= m - 1;
        }
      }
    }
    // ---------------- Stage II: this lane's task
    unsigned long long act = smask;
    if (has_t) {
      float z[E];
#pragma unroll
      for (int j = 0; j < E; j += 4) {
        const float4 v = __ldg(reinterpret_cast<const float4*>(zr + j));
        z[j] = v.x; z[j + 1] = v.y; z[j + 2] = v.z; z[j + 3] = v.w;
        *reinterpret_cast<float4*>(my_row + (((j >> 2) ^ swz) << 2)) = v;
      }
      float tz[KA > 0 ? KA : 1];
      int ti[KA > 0 ? KA : 1];
#pragma unroll
      for (int k = 0; k < KA; ++k) { tz[k] = -INFINITY; ti[k] = 0x7fffffff; }
#pragma unroll
      for (int j = 0; j < E; ++j) {
        float cz = ((smask >> j) & 1ull) ? -INFINITY : z[j];
        int ci = j;
#pragma unroll
        for (int k = 0; k < KA; ++k) {              // descending (value, then index ascending) list
          const bool sw = (cz > tz[k]) | ((cz == tz[k]) & (ci < ti[k]));
          const float xz = tz[k];
          const int xi = ti[k];
          tz[k] = sw ? cz : xz;
          ti[k] = sw ? ci : xi;
          cz = sw ? xz : cz;
          ci = sw ? xi : ci;
        }
      }
      unsigned long long amask = 0ull;
#pragma unroll
      for (int k = 0; k < KA; ++k) amask |= 1ull << ti[k];
      act = smask | amask;
      // the row maximum is active (shared, or the first adaptive pick) when K_a >= 1
      float amx = mx;
      if constexpr (KA == 0) {
        amx = -INFINITY;
#pragma unroll
        for (int j = 0; j < E; ++j) amx = ((act >> j) & 1ull) ? fmaxf(amx, z[j]) : amx;
      }
      int idx[K];
      float ev[K];
      {
        unsigned long long m = act;
#pragma unroll
        for (int k = 0; k < K; ++k) {
          const int j = __ffsll((long long)m) - 1;
          m &= m - 1;
          idx[k] = j;
          ev[k] = my_row[(((j >> 2) ^ swz) << 2) | (j & 3)];
        }
      }
      float asum = 0.f;
#pragma unroll
      for (int k = 0; k < K; ++k) {
        ev[k] = fast_exp(ev[k] - amx);
        asum += ev[k];
      }
      const float ainv = 1.f / asum;
      const long ot = (long)gl * a.B + b;
#pragma unroll
      for (int k = 0; k < K; ++k) {
        ev[k] *= ainv;
        a.active[ot * K + k] = idx[k];
        a.wsel[ot * K + k] = ev[k];
        atomicAdd(&s_act[idx[k]], 1);
        my_mass[idx[k]] += ev[k];
      }
      if constexpr (KA > 0) {
        unsigned long long m = amask;
#pragma unroll
        for (int k = 0; k < KA; ++k) {
          a.adaptive[ot * KA + k] = __ffsll((long long)m) - 1;
          m &= m - 1;
        }
      }
    }
    // union (routing.py:272): OR over the group's tasks
    const unsigned long long un = group_or<G>(act, gm);
#pragma unroll
    for (int i = 0; i < PER; ++i)
      if ((un >> (gl * PER + i)) & 1ull) atomicAdd(&s_uni[gl * PER + i], 1);
    if (gl == 0) {
      constexpr int EW = (E + 31) / 32;
#pragma unroll
      for (int w = 0; w < EW; ++w) a.umask[(long)b * EW + w] = (uint32_t)(un >> (32 * w));
      a.usize[b] = __popcll((long long)un);
    }
  }
  __syncthreads();
  // chunk partials (execution.py:109-113, balance.py:65-68): mass in a fixed order over the slots
  for (int e = tid; e < E; e += kThreads) {
    double m = 0.0;
    for (int i = 0; i < kThreads; ++i) m += (double)s_mass[i * (E + 1) + e];
    const long o = (long)blockIdx.x * E + e;
    a.chunk_union[o] = s_uni[e];
    a.chunk_active[o] = s_act[e];
    a.chunk_mass[o] = m;
    if (a.chunk_dmass != nullptr) a.chunk_dmass[o] = 0.0;
  }
  bad = __any_sync(0xffffffffu, bad);
  if (bad && lane == 0) atomicOr(a.flag, 1);
  if (a.n_exact != nullptr) {
    // n_exact counts rows once per lane of the group: one lane reports
    int v = gl == 0 ? n_exact : 0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0 && v) atomicAdd(a.n_exact, v);
  }
}

}  // namespace rt

static int32_t* g_rt_counter = nullptr;

template <int E, int G>
static int rt_launch_g(const rt::Args& a, int C, int ks, cudaStream_t st) {
  const size_t smem = (size_t)rt::kThreads * (E + 1) * 4 + (size_t)rt::kThreads * E * 4 + 2 * E * 4;
  auto go = [&](auto kern) {
    static bool attr = false;   // per instantiation (the lambda is instantiated per kernel type)
    if (!attr) {
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      attr = true;
    }
    smes_launch(kern, C, rt::kThreads, smem, st, a);
    return 0;
  };
  if (ks == 4) return go(rt::route_rt_kernel<E, G, 4, 2>);
  return go(rt::route_rt_kernel<E, G, 2, 1>);
}

template <int E>
static int rt_launch(const rt::Args& a, int C, int G, int ks, cudaStream_t st) {
  if constexpr (E >= 32) {
    if (G == 32) return rt_launch_g<E, 32>(a, C, ks, st);
  }
  if constexpr (E >= 16) {
    if (G == 16) return rt_launch_g<E, 16>(a, C, ks, st);
  }
  if (G == 8) return rt_launch_g<E, 8>(a, C, ks, st);
  return rt_launch_g<E, 4>(a, C, ks, st);
}

}  // namespace smes

using namespace smes;

extern "C" {

void smes_route_count_exact(int32_t* dev_counter) { g_rt_counter = dev_counter; }

// eligibility of the (row, task) router: training / scoring mode, no dense mass
int smes_route_rt_supported(int T, int E, int k_shared, int k_adaptive) {
  const bool k_ok = (k_shared == 4 && k_adaptive == 2) || (k_shared == 2 && k_adaptive == 1);
  return k_ok && (E == 16 || E == 32 || E == 64) && T >= 1 && T <= 32 && T <= E;
}

int smes_route_rt(const float* z, long st, long sb, const double* tw, int T, int B, int E, int k_shared,
                  int k_adaptive, int rows_per_warp, int32_t* shared, int32_t* adaptive, int32_t* active,
                  float* wsel, uint32_t* umask, int32_t* usize, int32_t* chunk_union, int32_t* chunk_active,
                  double* chunk_mass, double* chunk_dmass, int32_t* flag, void* stream) {
  if (!smes_route_rt_supported(T, E, k_shared, k_adaptive))
    return set_error(SMES_ERR_SHAPE, "route_rt: unsupported T=%d E=%d budget %d+%d", T, E, k_shared, k_adaptive);
  if ((st % 4) || (sb % 4) || (reinterpret_cast<uintptr_t>(z) % 16))
    return set_error(SMES_ERR_SHAPE, "route_rt: logits must be 16-byte aligned rows");
  int G = 4;
  while (G < T) G *= 2;
  const int rows_per_cta = 4 * rows_per_warp;                 // the plan's chunk (router.cu RT_WARPS = 4)
  const int C = (B + rows_per_cta - 1) / rows_per_cta;
  rt::Args a{z, st, sb, tw, T, B, rows_per_cta, shared, adaptive, active, wsel, umask, usize, chunk_union,
             chunk_active, chunk_mass, chunk_dmass, flag, g_rt_counter};
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (E == 16) rt_launch<16>(a, C, G, k_shared, s);
  else if (E == 32) rt_launch<32>(a, C, G, k_shared, s);
  else rt_launch<64>(a, C, G, k_shared, s);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_error(SMES_ERR_CUDA, "route_rt launch: %s", cudaGetErrorString(e));
  return SMES_OK;
}

}  // extern "C"
