// K0+K1 fused: router GEMM on the tensor cores feeding the progressive router
// straight from TMEM (the router logits never round-trip HBM).
//
//   z[b, t*E + e] = h[b] . W_r[t*E + e] + b_r[t*E + e]          (RouterBank.logits, routing.py:101-103)
//   route_batch over z                                            (routing.py:235-281)
//
// A 128-row tile of h (TMA, SW128) times the whole router bank W_r (N = T*E <= 256
// columns, K-major) accumulates in TMEM (tcgen05.mma, fp32); two accumulators let the
// MMA of the next tile run under the routing of this one.  The routing epilogue reads
// the logits from TMEM (epilogue thread i of a lane quarter owns TMEM lane i = row)
// with two threads per row, in two warps that share the lane quarter:
//   Stage I   (split by expert halves) p_t = softmax(z_t) and pooled = sum_t w_t p_t
//             in fp64, as route_kernel: exp, sums and pooling in double, the two
//             half-sums of each task exchanged through shared memory (fixed order);
//             shared = top-K_s of pooled, (score desc, index asc)   (routing.py:256-261).
//   Stage II  (split by tasks, t = half, half + 2, ...) exact fp32 compare of z_t with
//             the shared set excluded (:263-268), weights = softmax of z_t over the
//             active set (:203-211, :273), union bitmask (:272).
//   LoadStats partials per chunk of `sub_rows` rows (the plan's chunk, 4 * rows_per_warp):
//             union counts, active counts, sparse and (DM) dense mass per expert, reduced
//             in row order from shared memory (no atomics, deterministic; balance.py:65-68,
//             execution.py:109-113).
//
// Warp roles (384 threads, 1 CTA/SM): w0 TMA producer, w1 MMA issuer, w2 TMEM allocator,
// w4..w11 routing epilogue (warp w: lane quarter (w - 4) & 3, half (w - 4) >> 2).
#include "ptx.cuh"
#include "smes_capi.h"

namespace smes {

namespace front {

constexpr int BM = 128;
constexpr int BK = 64;
constexpr int kThreads = 384;
constexpr int kEpi = 256;           // 8 epilogue warps

struct Args {
  const float* bias;       // (T*E) router bias
  const double* tw;        // (T,) Stage-I pooling weights
  int T, B, d, sub_rows;
  int32_t* shared;         // (B, KS)
  int32_t* adaptive;       // (T, B, KA)
  int32_t* active;         // (T, B, K)
  float* wsel;             // (T, B, K)
  uint32_t* umask;         // (B, EW)
  int32_t* usize;          // (B,)
  int32_t* chunk_union;    // (C, E), C = ceil(B / sub_rows)
  int32_t* chunk_active;
  double* chunk_mass;
  double* chunk_dmass;     // written only with DM (dense-mass statistics requested)
  int32_t* flag;           // non-finite logits (sticky)
  float* z_out;            // optional (B, T*E) fp32 logits
};

template <int E>
struct Plan {
  static constexpr int kStages = 3;
  static constexpr int kA = BM * BK * 2;          // 16 KB
  static constexpr int kB = 256 * BK * 2;         // 32 KB (N <= 256)
  static constexpr int kOffB = kStages * kA;
  static constexpr int kOffBias = kOffB + kStages * kB;          // T*E floats (<= 1 KB)
  static constexpr int kOffPool = kOffBias + 1024;               // [E][128] fp64 pooled; then [2][E][128] fp32 mass
  static constexpr int kOffDm = kOffPool + E * BM * 8;           // [E][128] fp32 dense mass
  static constexpr int kOffCnt = kOffDm + E * BM * 4;            // [2][E][128] u8 active counts
  static constexpr int kOffSum = kOffCnt + 2 * E * BM;           // [2 parity][2 halves][128] fp64 half sums
  static constexpr int kOffUn = kOffSum + 4 * BM * 8;            // [2 halves][128] u32 union words
  static constexpr int kOffBar = kOffUn + 2 * BM * 4;
  static constexpr int kBytes = kOffBar + 128 + 1024;
  static_assert(E <= 32, "one union word per row");
  static_assert(kBytes <= 232448, "front smem plan exceeds 227 KB");
};

__device__ __forceinline__ uint32_t fkey(float f) {
  const uint32_t u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

__device__ __forceinline__ void bar_named(int id, int count) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}

// one task's E logits (+ bias) of this thread's row (warp-collective: tcgen05.ld)
template <int E>
__device__ __forceinline__ void load_task(uint32_t taddr, const float* sbias, int t, float (&z)[E]) {
  if constexpr (E == 32) {
    uint32_t r[32];
    tmem_ld32(taddr + t * E, r);
    tmem_ld_wait();
#pragma unroll
    for (int j = 0; j < 32; ++j) z[j] = __uint_as_float(r[j]);
  } else {
    static_assert(E == 16, "E must be 16 or 32");
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr + t * E));
    tmem_ld_wait();
#pragma unroll
    for (int j = 0; j < 16; ++j) z[j] = __uint_as_float(r[j]);
  }
#pragma unroll
  for (int j = 0; j < E; j += 4) {
    const float4 b = *reinterpret_cast<const float4*>(sbias + t * E + j);
    z[j] += b.x; z[j + 1] += b.y; z[j + 2] += b.z; z[j + 3] += b.w;
  }
}

template <int E>
__device__ __forceinline__ float tree_max(const float (&z)[E]) {
  float m[E / 2];
#pragma unroll
  for (int j = 0; j < E / 2; ++j) m[j] = fmaxf(z[j], z[j + E / 2]);
#pragma unroll
  for (int s = E / 4; s > 0; s >>= 1)
#pragma unroll
    for (int j = 0; j < s; ++j) m[j] = fmaxf(m[j], m[j + s]);
  return m[0];
}

template <int E, int KS, int KA, bool DM>
__global__ void __launch_bounds__(kThreads, 1)
    route_front_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                       const Args a) {
  using S = Plan<E>;
  constexpr int kStages = S::kStages;
  constexpr int K = KS + KA;
  constexpr int EH = E / 2;
  extern __shared__ __align__(16) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sA = smem;
  uint8_t* sB = smem + S::kOffB;
  float* sbias = reinterpret_cast<float*>(smem + S::kOffBias);
  double* s_pool = reinterpret_cast<double*>(smem + S::kOffPool);
  float* s_mass = reinterpret_cast<float*>(smem + S::kOffPool);     // aliases s_pool after Stage I
  float* s_dm = reinterpret_cast<float*>(smem + S::kOffDm);
  uint8_t* s_cnt = smem + S::kOffCnt;
  double* s_sum = reinterpret_cast<double*>(smem + S::kOffSum);
  uint32_t* s_un = reinterpret_cast<uint32_t*>(smem + S::kOffUn);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + S::kOffBar);
  uint64_t* empty = full + kStages;
  uint64_t* tfull = empty + kStages;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int T = a.T, N = T * E;
  const int ncols = N <= 64 ? 128 : N <= 128 ? 256 : 512;   // two accumulators, power of two
  const int num_tiles = (a.B + BM - 1) / BM;
  const int nkb = (a.d + BK - 1) / BK;

  for (int i = threadIdx.x; i < N; i += blockDim.x) sbias[i] = a.bias[i];
  if (warp == 0 && lane == 0) { tma_prefetch(&tmA); tma_prefetch(&tmB); }
  if (warp == 1 && lane == 0) {
    for (int s = 0; s < kStages; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    for (int s = 0; s < 2; ++s) { mbar_init(&tfull[s], 1); mbar_init(&tempty[s], kEpi); }
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, ncols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      // ================= TMA producer: h tile {64 k, 128 rows}, W_r {64 k, N rows}
      int stage = 0;
      uint32_t phase = 0;
      const uint32_t bytes = S::kA + N * BK * 2;
      for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
        for (int kb = 0; kb < nkb; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          mbar_expect_tx(&full[stage], bytes);
          tma_load_2d(sA + stage * S::kA, &tmA, &full[stage], kb * BK, tile * BM);
          tma_load_2d(sB + stage * S::kB, &tmB, &full[stage], kb * BK, 0);
          if (++stage == kStages) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ================= MMA issuer
      const uint32_t idesc = umma_idesc_bf16(BM, N, 0, 0);
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++it) {
        const int acc = it & 1;
        mbar_wait(&tempty[acc], ((it >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t tmem_d = tmem_base + acc * N;
        for (int kb = 0; kb < nkb; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t a_addr = smem_u32(sA + stage * S::kA);
          const uint32_t b_addr = smem_u32(sB + stage * S::kB);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k)
            tc_mma_f16(tmem_d, umma_desc_sw128(a_addr + k * 32, 16, 1024), umma_desc_sw128(b_addr + k * 32, 16, 1024),
                       idesc, (kb | k) != 0);
          tc_commit(&empty[stage]);
          if (++stage == kStages) { stage = 0; phase ^= 1; }
        }
        tc_commit(&tfull[acc]);
      }
    }
  } else if (warp >= 4) {
    // ================= routing epilogue: two threads per row
    const int q = (warp - 4) & 3;
    const int half = (warp - 4) >> 2;
    const int j0 = half * EH;
    const int r_loc = 32 * q + lane;
    const int pair_bar = 1 + q;             // the two warps of this lane quarter (64 threads)
    const int nsub = BM / a.sub_rows;
    const int C = (a.B + a.sub_rows - 1) / a.sub_rows;
    int it = 0, bad = 0;
    for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++it) {
      const int acc = it & 1;
      const int b = tile * BM + r_loc;
      const bool valid = b < a.B;
      mbar_wait(&tfull[acc], (it >> 1) & 1);
      tc_fence_after();
      const uint32_t taddr = tmem_base + ((uint32_t)(32 * q) << 16) + acc * N;

      // ---------------- Stage I (fp64): this half's experts of every task
      {
        double pp[EH];
        float dm[EH];
#pragma unroll
        for (int j = 0; j < EH; ++j) { pp[j] = 0.0; dm[j] = 0.f; }
        for (int t = 0; t < T; ++t) {
          float z[E];
          load_task<E>(taddr, sbias, t, z);
          const double m = (double)tree_max<E>(z);
          float zh[EH];                       // this half's logits (compile-time register indices)
#pragma unroll
          for (int j = 0; j < EH; ++j) {
            zh[j] = half ? z[EH + j] : z[j];
            bad |= !isfinite(zh[j]);
          }
          if (a.z_out != nullptr && valid) {
            float4* zo = reinterpret_cast<float4*>(a.z_out + (size_t)b * N + t * E + j0);
#pragma unroll
            for (int j = 0; j < EH; j += 4) zo[j / 4] = make_float4(zh[j], zh[j + 1], zh[j + 2], zh[j + 3]);
          }
          double ev[EH], s = 0.0;
#pragma unroll
          for (int j = 0; j < EH; ++j) { ev[j] = exp((double)zh[j] - m); s += ev[j]; }
          double* slot = s_sum + (t & 1) * 2 * BM;
          slot[half * BM + r_loc] = s;
          bar_named(pair_bar, 64);
          const double inv = 1.0 / (slot[r_loc] + slot[BM + r_loc]);     // low half + high half
          const double wt = a.tw[t];
#pragma unroll
          for (int j = 0; j < EH; ++j) {
            const double p = ev[j] * inv;
            pp[j] = fma(wt, p, pp[j]);
            if (DM) dm[j] += (float)p;
          }
        }
#pragma unroll
        for (int j = 0; j < EH; ++j) {
          s_pool[(j0 + j) * BM + r_loc] = pp[j];
          if (DM) s_dm[(j0 + j) * BM + r_loc] = valid ? dm[j] : 0.f;
        }
      }
      bar_named(pair_bar, 64);
      // shared set: top-K_s of pooled, (score desc, index asc); pooled >= 0, so the fp64 bit
      // patterns order like unsigned integers
      uint32_t smask = 0;
      if constexpr (KS > 0) {
        unsigned long long pk[E];
#pragma unroll
        for (int j = 0; j < E; ++j) pk[j] = (unsigned long long)__double_as_longlong(s_pool[j * BM + r_loc]);
#pragma unroll
        for (int k = 0; k < KS; ++k) {
          unsigned long long best = 0ull;
          int bi = -1;
#pragma unroll
          for (int j = 0; j < E; ++j) {
            const bool take = !((smask >> j) & 1u) && (bi < 0 || pk[j] > best);
            best = take ? pk[j] : best;
            bi = take ? j : bi;
          }
          smask |= 1u << bi;
        }
        if (half == 0 && valid) {
          uint32_t m = smask;
#pragma unroll
          for (int k = 0; k < KS; ++k) {
            a.shared[(size_t)b * KS + k] = __ffs(m) - 1;
            m &= m - 1;
          }
        }
      }
      bar_named(pair_bar, 64);          // s_pool reads done: the region becomes the mass partials

      // ---------------- Stage II: tasks half, half + 2, ...
      float mrow[E];
      uint32_t crow[E];
#pragma unroll
      for (int j = 0; j < E; ++j) { mrow[j] = 0.f; crow[j] = 0u; }
      uint32_t un = smask;
      for (int t = half; t < T; t += 2) {
        float z[E];
        load_task<E>(taddr, sbias, t, z);
        uint32_t tk[KA > 0 ? KA : 1];
        int ti[KA > 0 ? KA : 1];
#pragma unroll
        for (int k = 0; k < KA; ++k) { tk[k] = 0u; ti[k] = 0x7fffffff; }
#pragma unroll
        for (int j = 0; j < E; ++j) {
          // candidates outside the shared set: excluded keys are 0, below every real key (a
          // key-0 entry can only fill a slot that a real candidate displaces later, K <= E)
          uint32_t ck = ((smask >> j) & 1u) ? 0u : fkey(z[j]);
          int ci = j;
#pragma unroll
          for (int k = 0; k < KA; ++k) {      // descending (key, then index ascending) list
            const bool sw = ck > tk[k] || (ck == tk[k] && ci < ti[k]);
            const uint32_t xk = tk[k];
            const int xi = ti[k];
            tk[k] = sw ? ck : xk;
            ti[k] = sw ? ci : xi;
            ck = sw ? xk : ck;
            ci = sw ? xi : ci;
          }
        }
        uint32_t amask = 0;
#pragma unroll
        for (int k = 0; k < KA; ++k) amask |= 1u << ti[k];
        const uint32_t act = smask | amask;
        un |= amask;
        float amx = -INFINITY;
#pragma unroll
        for (int j = 0; j < E; ++j) amx = ((act >> j) & 1u) ? fmaxf(amx, z[j]) : amx;
        float asum = 0.f;
#pragma unroll
        for (int j = 0; j < E; ++j) {
          z[j] = ((act >> j) & 1u) ? __expf(z[j] - amx) : 0.f;
          asum += z[j];
        }
        const float ainv = 1.f / asum;
        const size_t ot = (size_t)t * a.B + b;
        int32_t* act_out = a.active + ot * K;
        float* w_out = a.wsel + ot * K;
        int32_t* ad_out = a.adaptive + ot * (KA > 0 ? KA : 1);
#pragma unroll
        for (int j = 0; j < E; ++j) {
          const uint32_t bit = (act >> j) & 1u;
          const float w = z[j] * ainv;
          const int pos = __popc(act & ((1u << j) - 1u));
          if (valid && bit) { act_out[pos] = j; w_out[pos] = w; }
          if (KA > 0 && valid && ((amask >> j) & 1u)) ad_out[__popc(amask & ((1u << j) - 1u))] = j;
          mrow[j] += w;
          crow[j] += bit;
        }
      }
      // the accumulator is consumed: the MMA may start the tile after next in it
      tc_fence_before();
      mbar_arrive(&tempty[acc]);
#pragma unroll
      for (int j = 0; j < E; ++j) {
        s_mass[(half * E + j) * BM + r_loc] = valid ? mrow[j] : 0.f;
        s_cnt[(half * E + j) * BM + r_loc] = valid ? (uint8_t)crow[j] : (uint8_t)0;
      }
      s_un[half * BM + r_loc] = valid ? un : 0u;
      bar_named(5, kEpi);
      if (half == 0 && valid) {
        const uint32_t u = un | s_un[BM + r_loc];
        a.umask[b] = u;
        a.usize[b] = __popc(u);
      }
      // ---------------- per-chunk statistics in row order (deterministic)
      const int tid = threadIdx.x - 128;
      for (int pr = tid; pr < nsub * E; pr += kEpi) {
        const int sc = pr / E, e = pr - sc * E;
        const int c = tile * nsub + sc;
        if (c >= C) continue;
        int cu = 0, ca = 0;
        double m = 0.0, dmv = 0.0;
        for (int r = sc * a.sub_rows; r < (sc + 1) * a.sub_rows; ++r) {
          cu += ((s_un[r] | s_un[BM + r]) >> e) & 1u;
          ca += s_cnt[e * BM + r] + s_cnt[(E + e) * BM + r];
          m += (double)s_mass[e * BM + r];
          m += (double)s_mass[(E + e) * BM + r];
          if (DM) dmv += (double)s_dm[e * BM + r];
        }
        const size_t o = (size_t)c * E + e;
        a.chunk_union[o] = cu;
        a.chunk_active[o] = ca;
        a.chunk_mass[o] = m;
        if (DM) a.chunk_dmass[o] = dmv;
      }
      bar_named(5, kEpi);
    }
    bad = __any_sync(0xffffffffu, bad);
    if (bad && lane == 0) atomicOr(a.flag, 1);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_dealloc(tmem_base, ncols);
}

}  // namespace front

// ---------------------------------------------------------------- host side
typedef CUresult (*EncodeTiledFnF)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static int front_map(CUtensorMap* m, const void* ptr, uint64_t inner, uint64_t rows, uint64_t ld_elems,
                     uint32_t box_rows) {
  static EncodeTiledFnF fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFnF>(p);
  }
  if (!fn) return set_error(SMES_ERR_CUDA, "cuTensorMapEncodeTiled unavailable (no CUDA driver?)");
  cuuint64_t d[2] = {inner, rows}, s[1] = {ld_elems * 2};
  cuuint32_t b[2] = {64, box_rows}, e[2] = {1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), d, s, b, e,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return set_error(SMES_ERR_CUDA, "cuTensorMapEncodeTiled failed (code %d)", (int)r);
  return SMES_OK;
}

template <int E, int KS, int KA, bool DM>
static int front_launch(const CUtensorMap& ta, const CUtensorMap& tb, const front::Args& a, int grid,
                        cudaStream_t st) {
  auto kern = front::route_front_kernel<E, KS, KA, DM>;
  constexpr int bytes = front::Plan<E>::kBytes;
  static bool attr = false;
  if (!attr) {
    cudaError_t ea = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (ea != cudaSuccess) return set_error(SMES_ERR_CUDA, "route_front smem attribute: %s", cudaGetErrorString(ea));
    attr = true;
  }
  kern<<<grid, front::kThreads, bytes, st>>>(ta, tb, a);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_error(SMES_ERR_CUDA, "route_front launch: %s", cudaGetErrorString(e));
  return SMES_OK;
}

template <int E>
static int front_dispatch(const CUtensorMap& ta, const CUtensorMap& tb, const front::Args& a, int grid, int ks,
                          bool dm, cudaStream_t st) {
  if (ks == 4)
    return dm ? front_launch<E, 4, 2, true>(ta, tb, a, grid, st) : front_launch<E, 4, 2, false>(ta, tb, a, grid, st);
  return dm ? front_launch<E, 2, 1, true>(ta, tb, a, grid, st) : front_launch<E, 2, 1, false>(ta, tb, a, grid, st);
}

}  // namespace smes

using namespace smes;

extern "C" {

int smes_route_front_supported(int T, int E, int d, int k_shared, int k_adaptive) {
  const bool e_ok = E == 16 || E == 32;
  const bool k_ok = (k_shared == 4 && k_adaptive == 2) || (k_shared == 2 && k_adaptive == 1);
  return e_ok && k_ok && T >= 2 && T * E <= 256 && (T * E) % 16 == 0 && d >= 64 && d % 64 == 0 &&
         k_shared + k_adaptive <= E;
}

int smes_route_front(const void* h, long ldh, const void* w_r, const float* b_r, const double* task_weights, int T,
                     int B, int E, int d, int k_shared, int k_adaptive, int sub_rows, int32_t* shared,
                     int32_t* adaptive, int32_t* active, float* wsel, uint32_t* umask, int32_t* usize,
                     int32_t* chunk_union, int32_t* chunk_active, double* chunk_mass, double* chunk_dmass,
                     int32_t* flag, float* z_out, void* stream) {
  if (B < 1) return set_error(SMES_ERR_SHAPE, "route_front: empty batch");
  if (!smes_route_front_supported(T, E, d, k_shared, k_adaptive))
    return set_error(SMES_ERR_SHAPE, "route_front: unsupported shape T=%d E=%d d=%d budget %d+%d", T, E, d, k_shared,
                     k_adaptive);
  if (sub_rows < 1 || sub_rows > 128 || 128 % sub_rows)
    return set_error(SMES_ERR_SHAPE, "route_front: chunk rows %d must divide 128", sub_rows);
  if ((ldh * 2) % 16) return set_error(SMES_ERR_SHAPE, "route_front: h stride must be 16-byte aligned");
  CUtensorMap ta, tb;
  int rc;
  if ((rc = front_map(&ta, h, (uint64_t)d, (uint64_t)B, (uint64_t)ldh, 128))) return rc;
  if ((rc = front_map(&tb, w_r, (uint64_t)d, (uint64_t)(T * E), (uint64_t)d, (uint32_t)(T * E)))) return rc;
  front::Args a{b_r, task_weights, T, B, d, sub_rows, shared, adaptive, active, wsel, umask, usize,
                chunk_union, chunk_active, chunk_mass, chunk_dmass, flag, z_out};
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int tiles = (B + 127) / 128;
  const int grid = tiles < sms ? tiles : sms;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const bool dm = chunk_dmass != nullptr;
  if (E == 16) return front_dispatch<16>(ta, tb, a, grid, k_shared, dm, st);
  return front_dispatch<32>(ta, tb, a, grid, k_shared, dm, st);
}

}  // extern "C"
