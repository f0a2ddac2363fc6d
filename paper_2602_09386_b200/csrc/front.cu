// K0+K1 fused: router GEMM on the tensor cores feeding the progressive router
// straight from TMEM (the router logits never round-trip HBM).
//
//   z[b, t*E + e] = h[b] . W_r[t*E + e] + b_r[t*E + e]          (RouterBank.logits, routing.py:101-103)
//   route_batch over z                                            (routing.py:235-281)
//
// A tile of h rows (TMA, SW128; 128 MMA rows, `rpc` <= 128 of them routed by this CTA so the
// grid covers every SM) times the whole router bank W_r (N = T*E <= 256 columns, K-major)
// accumulates in TMEM (tcgen05.mma, fp32); two accumulators let the MMA of the next tile run
// under the routing of this one.  Epilogue thread (g, lane) of lane quarter q owns row
// 32q + lane (its TMEM lane) and the tasks t = g, g + TPR, ...:
//
//   Stage I  pooled[e] = sum_t w_t softmax(z_t)[e] and shared = top-K_s(pooled), ties to the
//            lowest index (routing.py:256-261).  Reference-init routers give pooled gaps down to
//            1e-10, so the SET must come out as an fp64 evaluation would give it.
//            Fast path: exp in fp32 (__expf), softmax sums and pooling in fp64, and a rigorous
//            per-expert bound on the fp32 exp error (documented __expf bound: (2 + 1.173|x|)
//            ulp, plus the argument rounding; inflated 1.5x).  The set is accepted when every
//            selected expert's lower bound exceeds every unselected expert's upper bound.
//            Rows that fail (near-ties: ~5 % at reference init, ~0 at trained scale) are
//            staged to shared memory and recomputed entirely in fp64 by whole warps (lane =
//            expert), then their set replaces the fast one.  Selections stay index-exact.
//   Stage II (same tasks) exact fp32 compare of z_t with the shared set excluded (:263-268),
//            weights = softmax of z_t over the active set (:203-211, :273), union (:272).
//   LoadStats partials per chunk of `sub_rows` rows (the plan's chunk, 4 * rows_per_warp):
//            union counts, active counts (bit-sliced counters), sparse and (DM) dense mass per
//            expert, reduced in a fixed row order (no atomics; balance.py:65-68,
//            execution.py:109-113).
//
// Warp roles (384 threads, 1 CTA/SM): w0 TMA producer, w1 MMA issuer, w2 TMEM allocator,
// w4..w11 routing epilogue (warp w: lane quarter (w - 4) & 3, task thread g = (w - 4) >> 2).
#include "ptx.cuh"
#include "smes_capi.h"

namespace smes {

namespace front {

constexpr int BM = 128;
constexpr int BK = 64;
constexpr int TPR = 2;                       // task threads per row
constexpr int kThreads = 128 + 128 * TPR;
constexpr int kEpi = 128 * TPR;
constexpr int kNPlanes = 4;                  // bit-sliced active counters (up to 15 tasks per thread)

struct Args {
  const float* bias;       // (T*E) router bias
  const double* tw;        // (T,) Stage-I pooling weights
  int T, B, d, sub_rows, rpc;
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
  int32_t* n_exact;        // optional: rows whose shared set needed the fp64 recompute (summed)
};

template <int E, bool DM>
struct Plan {
  static constexpr int EQ = E / TPR;
  // the router GEMM is issued in N chunks of (up to) 64 columns, each committed on its own
  // barrier, so Stage I of the first tasks runs while the MMAs of the later tasks stream W_r
#ifndef SMES_FRONT_WSTAGES
#define SMES_FRONT_WSTAGES 6
#endif
  static constexpr int kWStages = DM ? 3 : SMES_FRONT_WSTAGES;   // (DM: the dense-mass array needs the space)
  static constexpr int kH = BM * BK * 2;          // 16 KB per k-block of h (d <= 256: 4 blocks)
  static constexpr int kW = 64 * BK * 2;          // 8 KB per (chunk, k-block) of W_r
  static constexpr int kOffW = 4 * kH;
  static constexpr int kOffBias = kOffW + kWStages * kW;         // T*E floats (<= 1 KB)
  static constexpr int kOffTw = kOffBias + 1024;                 // T doubles (<= 16)
  static constexpr int kOffM = kOffTw + 128;                     // [16][128] fp32 task maxima
  // R1 (64 KB), reused phase by phase: the Stage-I exchange of pooled partials [TPR][EQ][128]
  // fp64 + exp error bounds [TPR][128] fp32; the fp64 recompute's staged logits; in Stage II
  // the per-thread logit rows [kEpi][E] and the sparse-mass partials [TPR][E][128] (at 32 KB)
  static constexpr int kR1 = 32 * 1024 + TPR * BM * (E + 1) * 4;
  static constexpr int kOffR1 = kOffM + 16 * BM * 4;
  static constexpr int kOffCand = kOffR1 + kR1;                  // [TPR][4][128] u64 keys + u8 indices
  // per-row arrays the chunk statistics read across experts: row stride E + 1 (E/4 + 1) words, so
  // both the per-row writers (lane = row) and the readers (lane = expert) are bank-conflict free
  static constexpr int kOffDm = kOffCand + TPR * 4 * BM * 9 + 64;   // [TPR][128][E + 1] fp32 dense mass
  static constexpr int kOffCnt = kOffDm + (DM ? TPR * BM * (E + 1) * 4 : 0);   // [TPR][128][E/4 + 1] u8 x 4
  static constexpr int kOffLoHi = kOffCnt + TPR * BM * (E / 4 + 1) * 4;       // [TPR][2][128] fp64
  static constexpr int kOffUn = kOffLoHi + TPR * 2 * BM * 8;             // [TPR][128] u32 union words
  static constexpr int kOffSlot = kOffUn + TPR * BM * 4;                 // [128] slot, [CAPMAX] set, counter
  static constexpr int kOffBar = kOffSlot + (BM + 96 + 4) * 4;
  static constexpr int kBytes = kOffBar + 512 + 1024;
  static_assert(E <= 32, "one union word per row");
  static_assert(TPR * EQ * BM * 12 <= kR1, "exchange fits R1");
  static_assert(kEpi * E * 4 <= 32 * 1024, "Stage-II logit rows fit the first 32 KB of R1");
  static_assert(kBytes <= 232448, "front smem plan exceeds 227 KB");
};

// e^x as ex2.approx.ftz(x log2 e): the CUDA __expf algorithm (max error (2 + 1.173 |x|) ulp for
// normal results), without its subnormal fix-up (results below 2^-126 flush to 0)
__device__ __forceinline__ float fast_exp(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x * 1.4426950408889634f));
  return y;
}

// e^x - 1 for x <= 0 with relative accuracy (route_rt.cu): degree-8 Taylor for |x| < 1/4, else
// fast_exp(x) - 1; kEpsY bounds the relative error with the argument rounding, with margin
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
template <int E> constexpr int kLog2E = E == 16 ? 4 : 5;
__device__ __forceinline__ uint32_t okey(float f) {   // order-preserving key of a float of any sign
  const uint32_t u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
template <int E>
__device__ __forceinline__ float tree_sum(const float (&z)[E]) {
  float m[E / 2];
#pragma unroll
  for (int j = 0; j < E / 2; ++j) m[j] = z[j] + z[j + E / 2];
#pragma unroll
  for (int s = E / 4; s > 0; s >>= 1)
#pragma unroll
    for (int j = 0; j < s; ++j) m[j] = m[j] + m[j + s];
  return m[0];
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
template <int E>
__device__ __forceinline__ float tree_min(const float (&z)[E]) {
  float m[E / 2];
#pragma unroll
  for (int j = 0; j < E / 2; ++j) m[j] = fminf(z[j], z[j + E / 2]);
#pragma unroll
  for (int s = E / 4; s > 0; s >>= 1)
#pragma unroll
    for (int j = 0; j < s; ++j) m[j] = fminf(m[j], m[j + s]);
  return m[0];
}

// (key desc, index asc) arg-max over a group of G lanes (G = E <= 32, aligned), 64-bit keys
template <int G>
__device__ __forceinline__ void group_argmax(unsigned long long& key, int& idx) {
#pragma unroll
  for (int o = G / 2; o > 0; o >>= 1) {
    const unsigned long long k2 = __shfl_xor_sync(0xffffffffu, key, o);
    const int i2 = __shfl_xor_sync(0xffffffffu, idx, o);
    const bool take = (k2 > key) | ((k2 == key) & (i2 < idx));
    key = take ? k2 : key;
    idx = take ? i2 : idx;
  }
}

template <int E, int KS, int KA, bool DM>
__global__ void __launch_bounds__(kThreads, 1)
    route_front_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                       const Args a) {
  pdl_wait();
  using S = Plan<E, DM>;
  constexpr int K = KS + KA;
  constexpr int EQ = S::EQ;
  static_assert(TPR == 2, "the Stage-I exchange pairs two task threads per row");
  extern __shared__ __align__(16) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sH = smem;
  uint8_t* sW = smem + S::kOffW;
  float* sbias = reinterpret_cast<float*>(smem + S::kOffBias);
  double* stw = reinterpret_cast<double*>(smem + S::kOffTw);
  float* s_m = reinterpret_cast<float*>(smem + S::kOffM);
  uint8_t* r1 = smem + S::kOffR1;
  double* x_pp = reinterpret_cast<double*>(r1);                          // [TPR][EQ][BM]
  float* x_pe = reinterpret_cast<float*>(r1 + TPR * EQ * BM * 8);        // [TPR][BM] exp error bounds
  float* s_stage = reinterpret_cast<float*>(r1);                         // [CAP][T][E]
  float* s_scr = reinterpret_cast<float*>(r1);                           // [kEpi][E] (Stage II)
  float* s_mass = reinterpret_cast<float*>(r1 + 32 * 1024);              // [TPR][BM][E + 1]
  unsigned long long* s_ckey = reinterpret_cast<unsigned long long*>(smem + S::kOffCand);
  uint8_t* s_cidx = smem + S::kOffCand + TPR * 4 * BM * 8;
  float* s_dm = reinterpret_cast<float*>(smem + S::kOffDm);
  uint32_t* s_cnt = reinterpret_cast<uint32_t*>(smem + S::kOffCnt);
  double* s_lohi = reinterpret_cast<double*>(smem + S::kOffLoHi);
  uint32_t* s_un = reinterpret_cast<uint32_t*>(smem + S::kOffUn);
  int* s_slot = reinterpret_cast<int*>(smem + S::kOffSlot);              // [BM]
  uint32_t* s_fix = reinterpret_cast<uint32_t*>(s_slot + BM);            // [<= 96]
  int* s_nf = s_slot + BM + 96;
  uint64_t* wfull = reinterpret_cast<uint64_t*>(smem + S::kOffBar);
  uint64_t* wempty = wfull + S::kWStages;
  uint64_t* hfull = wempty + S::kWStages;
  uint64_t* hempty = hfull + 1;
  uint64_t* tfull = hempty + 1;          // [2 accumulators][16 chunks]
  uint64_t* tempty = tfull + 32;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int T = a.T, N = T * E;
  const int ncols = N <= 64 ? 128 : N <= 128 ? 256 : 512;   // two accumulators, power of two
  const int rpc = a.rpc;
  const int num_tiles = (a.B + rpc - 1) / rpc;
  const int nkb = (a.d + BK - 1) / BK;
  // columns per chunk: <= 64 (the W_r ring slot), a multiple of E (whole tasks per chunk)
  const int NC = N % 64 == 0 ? 64 : N % 32 == 0 ? 32 : 16;
  const int nch = N / NC;
  const int cap = min(96, S::kR1 / (N * 4));                 // rows per fp64 recompute round

  for (int i = threadIdx.x; i < N; i += blockDim.x) sbias[i] = a.bias[i];
  for (int i = threadIdx.x; i < T; i += blockDim.x) stw[i] = a.tw[i];
  if (threadIdx.x == 0) *s_nf = 0;
  if (warp == 0 && lane == 0) { tma_prefetch(&tmA); tma_prefetch(&tmB); }
  if (warp == 1 && lane == 0) {
    for (int s = 0; s < S::kWStages; ++s) { mbar_init(&wfull[s], 1); mbar_init(&wempty[s], 1); }
    mbar_init(hfull, 1);
    mbar_init(hempty, 1);
    for (int s = 0; s < 32; ++s) mbar_init(&tfull[s], 1);
    for (int s = 0; s < 2; ++s) mbar_init(&tempty[s], kEpi);
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, ncols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      // ================= TMA producer: the tile's h (resident, all k-blocks), then W_r per chunk
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++it) {
        mbar_wait(hempty, (it & 1) ^ 1);
        mbar_expect_tx(hfull, nkb * S::kH);
        for (int kb = 0; kb < nkb; ++kb) tma_load_2d(sH + kb * S::kH, &tmA, hfull, kb * BK, tile * rpc);
        for (int c = 0; c < nch; ++c) {
          for (int kb = 0; kb < nkb; ++kb) {
            mbar_wait(&wempty[stage], phase ^ 1);
            mbar_expect_tx(&wfull[stage], NC * BK * 2);
            tma_load_2d(sW + stage * S::kW, &tmB, &wfull[stage], kb * BK, c * NC);
            if (++stage == S::kWStages) { stage = 0; phase ^= 1; }
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ================= MMA issuer: one commit per chunk
      const uint32_t idesc = umma_idesc_bf16(BM, NC, 0, 0);
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++it) {
        const int acc = it & 1;
        mbar_wait(&tempty[acc], ((it >> 1) & 1) ^ 1);
        mbar_wait(hfull, it & 1);
        tc_fence_after();
        for (int c = 0; c < nch; ++c) {
          const uint32_t tmem_d = tmem_base + acc * N + c * NC;
          for (int kb = 0; kb < nkb; ++kb) {
            mbar_wait(&wfull[stage], phase);
            tc_fence_after();
            const uint32_t h_addr = smem_u32(sH + kb * S::kH);
            const uint32_t w_addr = smem_u32(sW + stage * S::kW);
#pragma unroll
            for (int k = 0; k < BK / 16; ++k)
              tc_mma_f16(tmem_d, umma_desc_sw128(h_addr + k * 32, 16, 1024), umma_desc_sw128(w_addr + k * 32, 16, 1024),
                         idesc, (kb | k) != 0);
            tc_commit(&wempty[stage]);
            if (++stage == S::kWStages) { stage = 0; phase ^= 1; }
          }
          tc_commit(&tfull[acc * 16 + c]);
        }
        tc_commit(hempty);                 // every MMA of this tile has read h
      }
    }
  } else if (warp >= 4) {
    // ================= routing epilogue
    const int q = (warp - 4) & 3;
    const int g = (warp - 4) >> 2;
    const int r_loc = 32 * q + lane;
    const int quad_bar = 1 + q;              // the TPR warps of this lane quarter
    const int tid = threadIdx.x - 128;
    const int C = (a.B + a.sub_rows - 1) / a.sub_rows;
    const int nsub = rpc / a.sub_rows;
    int it = 0, bad = 0, n_exact = 0;
    for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++it) {
      const int acc = it & 1;
      const int b = tile * rpc + r_loc;
      const bool valid = r_loc < rpc && b < a.B;
      const uint32_t taddr = tmem_base + ((uint32_t)(32 * q) << 16) + acc * N;
      const uint32_t tpar = (it >> 1) & 1;
#ifdef SMES_FRONT_GEMM_ONLY
      for (int c = 0; c < nch; ++c) mbar_wait(&tfull[acc * 16 + c], tpar);
      tc_fence_before();
      mbar_arrive(&tempty[acc]);
      continue;
#endif
      int waited = 0;
      auto wait_task = [&](int t) {          // the MMA chunks up to task t's are committed
        const int ct = (t * E) / NC;
        while (waited <= ct) {
          mbar_wait(&tfull[acc * 16 + waited], tpar);
          ++waited;
        }
        tc_fence_after();
      };

      // ---------------- Stage I, fast path: this thread's tasks, every expert
      uint32_t smask = 0;
      bool exact_needed = false;
      if constexpr (KS > 0 || DM) {
        // pooled_e = sum_t w_t / S_t + P_e with y_te = exp(z_te - max_t) - 1, S_t = E + sum_e y_te and
        // P_e = sum_t (w_t / S_t) y_te: the first term is common to every expert, so the shared set
        // is the top-K_s of P, which fp32 holds to ~1e-3 of the pooled scores' rounding error at
        // reference init (|y| ~ 1e-3; route_rt.cu has the bound)
        float pp[E];
        float perr = 0.f;          // absolute error bound of this thread's partial P (every expert)
#pragma unroll
        for (int j = 0; j < E; ++j) pp[j] = 0.f;
        bool first = true;
        for (int t = g; t < T; t += TPR) {
          wait_task(t);
          float z[E];
          load_task<E>(taddr, sbias, t, z);
          const float mx = tree_max<E>(z), mn = tree_min<E>(z);
          s_m[t * BM + r_loc] = mx;
          if (a.z_out != nullptr && valid) {
            float4* zo = reinterpret_cast<float4*>(a.z_out + (size_t)b * N + t * E);
#pragma unroll
            for (int j = 0; j < E; j += 4) zo[j / 4] = make_float4(z[j], z[j + 1], z[j + 2], z[j + 3]);
          }
#pragma unroll
          for (int j = 0; j < E; ++j) z[j] = expm1_neg(z[j] - mx);
          const float ysum = tree_sum<E>(z);
          const float ssum = (float)E + ysum;
          bad |= !(isfinite(mx) & isfinite(mn) & isfinite(ssum));
          const float q = (float)stw[t] / ssum;
#pragma unroll
          for (int j = 0; j < E; ++j) pp[j] = fmaf(q, z[j], pp[j]);
          // |error| of q y_tj <= q |y|max (eps_y + rho_t + 3u), rho_t the relative error of S_t;
          // the fp32 accumulation over this thread's tasks and the partner's adds (T/TPR + 1) u
          const float rho = (kLog2E<E> * 0x1p-24f + kEpsY) * (-ysum) / ssum + 0x1p-24f;
          perr += q * (-expm1_neg(mn - mx)) * (kEpsY + rho + (3 + T / TPR + 2) * 0x1p-24f);
          if constexpr (DM) {
            const float qf = 1.f / ssum;
#pragma unroll
            for (int j = 0; j < E; ++j) {
              float* dp = s_dm + (g * BM + r_loc) * (E + 1) + j;
              *dp = first ? qf * (1.f + z[j]) : fmaf(qf, 1.f + z[j], *dp);
            }
          }
          first = false;
        }
        if constexpr (DM) {
          if (first || !valid) {
#pragma unroll
            for (int j = 0; j < E; ++j) s_dm[(g * BM + r_loc) * (E + 1) + j] = 0.f;
          }
        }
        if constexpr (KS > 0) {
          // exchange: thread g owns experts [g EQ, (g + 1) EQ); pooled = own partial + partner's
          // (fp64 addition commutes, so both threads would get the same value)
          const int oh = 1 - g;
          float* x_pf = reinterpret_cast<float*>(x_pp);                     // [TPR][EQ][BM] fp32 partials
#pragma unroll
          for (int j = 0; j < EQ; ++j) x_pf[(oh * EQ + j) * BM + r_loc] = g == 0 ? pp[EQ + j] : pp[j];
          x_pe[g * BM + r_loc] = perr;
          bar_named(quad_bar, 32 * TPR);
          float pq[EQ];
#pragma unroll
          for (int j = 0; j < EQ; ++j) pq[j] = (g == 0 ? pp[j] : pp[EQ + j]) + x_pf[(g * EQ + j) * BM + r_loc];
          // x 1.5 margin, + an absolute floor for flushed exps
          const double e_abs = 1.5 * ((double)x_pe[r_loc] + (double)x_pe[BM + r_loc]) + 0x1p-100;
          const int j0 = g * EQ;
          // shared set: top-K_s of pooled, (score desc, index asc).  pooled >= 0, so the fp64 bit
          // patterns order like unsigned integers.  Each thread sorts its half, the lists merge
          // through shared memory.
          unsigned long long pk[EQ];
#pragma unroll
          for (int j = 0; j < EQ; ++j) pk[j] = okey(pq[j]);     // P may be negative: order-preserving key
          uint32_t taken = 0;
#pragma unroll
          for (int k = 0; k < KS; ++k) {
            unsigned long long best = 0ull;
            int bi = -1;
#pragma unroll
            for (int j = 0; j < EQ; ++j) {
              const bool take = !((taken >> j) & 1u) & ((bi < 0) | (pk[j] > best));
              best = take ? pk[j] : best;
              bi = take ? j : bi;
            }
            if (k < EQ) taken |= 1u << bi;
            s_ckey[(g * KS + k) * BM + r_loc] = k < EQ ? best : 0ull;
            s_cidx[(g * KS + k) * BM + r_loc] = k < EQ ? (uint8_t)(j0 + bi) : (uint8_t)255;
          }
          bar_named(quad_bar, 32 * TPR);
          int head[TPR];
#pragma unroll
          for (int h = 0; h < TPR; ++h) head[h] = 0;
#pragma unroll
          for (int k = 0; k < KS; ++k) {
            unsigned long long best = 0ull;
            int bidx = 255, bg = 0;
#pragma unroll
            for (int h = 0; h < TPR; ++h) {
              const bool ok = head[h] < KS;
              const int slot = (h * KS + (ok ? head[h] : 0)) * BM + r_loc;
              const unsigned long long key = s_ckey[slot];
              const int idx = s_cidx[slot];
              const bool take = ok & (idx != 255) & ((bidx == 255) | (key > best) | ((key == best) & (idx < bidx)));
              best = take ? key : best;
              bidx = take ? idx : bidx;
              bg = take ? h : bg;
            }
            smask |= 1u << bidx;
#pragma unroll
            for (int h = 0; h < TPR; ++h) head[h] += (h == bg);
          }
          // certify the set: min over selected of (pooled - err) > max over the rest of (pooled + err)
          double lo = INFINITY, hi = -INFINITY;
#pragma unroll
          for (int j = 0; j < EQ; ++j) {
            const bool sel = (smask >> (j0 + j)) & 1u;
            lo = sel ? fmin(lo, (double)pq[j] - e_abs) : lo;
            hi = sel ? hi : fmax(hi, (double)pq[j] + e_abs);
          }
          s_lohi[(g * 2) * BM + r_loc] = lo;
          s_lohi[(g * 2 + 1) * BM + r_loc] = hi;
          bar_named(quad_bar, 32 * TPR);
          const double lo_all = fmin(s_lohi[0 * BM + r_loc], s_lohi[2 * BM + r_loc]);
          const double hi_all = fmax(s_lohi[1 * BM + r_loc], s_lohi[3 * BM + r_loc]);
          exact_needed = valid && !(lo_all > hi_all);
        }
      }

      // ---------------- Stage I, exact path: rows the fast path could not certify, in fp64
      if constexpr (KS > 0) {
        if (g == 0) s_slot[r_loc] = exact_needed ? atomicAdd(s_nf, 1) : -1;
        bar_named(5, kEpi);
        const int nf = *s_nf;
        const int slot = s_slot[r_loc];
#ifdef SMES_FRONT_NO_EXACT
        if (nf < 0)
#endif
        for (int base = 0; base < nf; base += cap) {
          const bool mine = slot >= base && slot < base + cap;
          if (__any_sync(0xffffffffu, mine)) {        // warp-uniform TMEM loads
            for (int t = g; t < T; t += TPR) {
              float z[E];
              load_task<E>(taddr, sbias, t, z);
              if (mine) {
                float4* dst = reinterpret_cast<float4*>(s_stage + ((size_t)(slot - base) * T + t) * E);
#pragma unroll
                for (int j = 0; j < E; j += 4) dst[j / 4] = make_float4(z[j], z[j + 1], z[j + 2], z[j + 3]);
              }
            }
          }
          bar_named(5, kEpi);
          // whole warps: lane = expert (E = 16: two rows per warp)
          constexpr int RPW = 32 / E;
          const int nrows = min(cap, nf - base);
          const int wi = warp - 4;
          const int e = lane % E;
          for (int r0 = wi * RPW; r0 < nrows; r0 += (kEpi / 32) * RPW) {
            const int sr = r0 + lane / E;
            const bool act = sr < nrows;
            double pooled = 0.0;
            // four tasks at a time: their shuffle / exp chains are independent (latency overlap)
            for (int t0 = 0; t0 < T; t0 += 4) {
              float zz[4], m[4];
#pragma unroll
              for (int u = 0; u < 4; ++u) {
                zz[u] = (act && t0 + u < T) ? s_stage[((size_t)sr * T + t0 + u) * E + e] : 0.f;
                m[u] = zz[u];
              }
#pragma unroll
              for (int o = E / 2; o > 0; o >>= 1)
#pragma unroll
                for (int u = 0; u < 4; ++u) m[u] = fmaxf(m[u], __shfl_xor_sync(0xffffffffu, m[u], o));
              double ev[4], sm[4];
#pragma unroll
              for (int u = 0; u < 4; ++u) { ev[u] = exp((double)zz[u] - (double)m[u]); sm[u] = ev[u]; }
#pragma unroll
              for (int o = E / 2; o > 0; o >>= 1)
#pragma unroll
                for (int u = 0; u < 4; ++u) sm[u] += __shfl_xor_sync(0xffffffffu, sm[u], o);
#pragma unroll
              for (int u = 0; u < 4; ++u)
                if (t0 + u < T) pooled = fma(stw[t0 + u], ev[u] / sm[u], pooled);
            }
            uint32_t set = 0;
            // pooled >= 0: its bit pattern orders as an unsigned key.  A taken expert drops to key 0
            // with index +inf, so it loses every later round (also to a live expert with pooled 0)
            unsigned long long mykey = (unsigned long long)__double_as_longlong(pooled);
            int myidx = e;
#pragma unroll
            for (int k = 0; k < KS; ++k) {
              unsigned long long key = mykey;
              int idx = myidx;
              group_argmax<E>(key, idx);
              set |= 1u << idx;
              if (idx == e) { mykey = 0ull; myidx = 0x7fffffff; }
            }
            if (act && e == 0) s_fix[sr] = set;
          }
          bar_named(5, kEpi);
          if (mine) smask = s_fix[slot - base];
        }
        if (g == 0 && valid) {
          n_exact += slot >= 0;
          uint32_t m = smask;
#pragma unroll
          for (int k = 0; k < KS; ++k) {
            a.shared[(size_t)b * KS + k] = __ffs(m) - 1;
            m &= m - 1;
          }
        }
      }

      // ---------------- Stage II: tasks g, g + TPR, ...
      uint32_t cnt[kNPlanes];           // bit-sliced per-expert active counters
#pragma unroll
      for (int p = 0; p < kNPlanes; ++p) cnt[p] = 0u;
#pragma unroll
      for (int j = 0; j < E; ++j) s_mass[(g * BM + r_loc) * (E + 1) + j] = 0.f;
      constexpr int SW = E / 4 - 1;     // 16-byte chunk swizzle of the per-thread logit row
      float* my_row = s_scr + tid * E;
      uint32_t un = smask;
#ifdef SMES_FRONT_NO_STAGE2
      if (T < 0)
#endif
      for (int t = g; t < T; t += TPR) {
        if constexpr (KS == 0 && !DM) wait_task(t);
        float z[E];
        load_task<E>(taddr, sbias, t, z);
        if constexpr (KS == 0 && !DM) {     // no Stage I: the finiteness check (routing.py:246-247) is here
#pragma unroll
          for (int j = 0; j < E; ++j) bad |= !isfinite(z[j]);
        }
        float tz[KA > 0 ? KA : 1];
        int ti[KA > 0 ? KA : 1];
#pragma unroll
        for (int k = 0; k < KA; ++k) { tz[k] = -INFINITY; ti[k] = 0x7fffffff; }
#pragma unroll
        for (int j = 0; j < E; ++j) {
          // candidates outside the shared set (excluded ones enter as -inf and can only fill a slot
          // that a finite candidate displaces later, K <= E); float compares: -0 == +0 ties by index
          float cz = ((smask >> j) & 1u) ? -INFINITY : z[j];
          int ci = j;
#pragma unroll
          for (int k = 0; k < KA; ++k) {      // descending (value, then index ascending) list
            const bool sw = (cz > tz[k]) | ((cz == tz[k]) & (ci < ti[k]));   // bitwise: no branches
            const float xz = tz[k];
            const int xi = ti[k];
            tz[k] = sw ? cz : xz;
            ti[k] = sw ? ci : xi;
            cz = sw ? xz : cz;
            ci = sw ? xi : ci;
          }
        }
        uint32_t amask = 0;
#pragma unroll
        for (int k = 0; k < KA; ++k) amask |= 1u << ti[k];
        const uint32_t act = smask | amask;
        un |= amask;
        {   // bit-sliced add of the active set to the per-expert counters
          uint32_t c = act;
#pragma unroll
          for (int p = 0; p < kNPlanes; ++p) { const uint32_t nc = cnt[p] & c; cnt[p] ^= c; c = nc; }
        }
        // max over the active set: with K_a >= 1 the row maximum is always active (shared, or the
        // first adaptive pick), so it is the task maximum of Stage I
        float amx;
        if constexpr (KA > 0 && (KS > 0 || DM)) {
          amx = s_m[t * BM + r_loc];
        } else {
          amx = -INFINITY;
#pragma unroll
          for (int j = 0; j < E; ++j) amx = ((act >> j) & 1u) ? fmaxf(amx, z[j]) : amx;
        }
        // the K active logits, ascending expert index, through this thread's shared-memory row
#pragma unroll
        for (int c = 0; c < E / 4; ++c)
          *reinterpret_cast<float4*>(my_row + ((c ^ (tid & SW)) << 2)) =
              make_float4(z[4 * c], z[4 * c + 1], z[4 * c + 2], z[4 * c + 3]);
        int idx[K];
        float ev[K];
        {
          uint32_t m = act;
#pragma unroll
          for (int k = 0; k < K; ++k) {
            const int j = __ffs(m) - 1;
            m &= m - 1;
            idx[k] = j;
            ev[k] = my_row[((((j >> 2) ^ (tid & SW))) << 2) | (j & 3)];
          }
        }
        float asum = 0.f;
#pragma unroll
        for (int k = 0; k < K; ++k) {
          ev[k] = fast_exp(ev[k] - amx);
          asum += ev[k];
        }
        const float ainv = 1.f / asum;
#pragma unroll
        for (int k = 0; k < K; ++k) ev[k] *= ainv;
        const size_t ot = (size_t)t * a.B + b;
        if (valid) {
          int32_t* act_out = a.active + ot * K;
          float* w_out = a.wsel + ot * K;
          if constexpr (K % 2 == 0) {       // 8-byte aligned rows
#pragma unroll
            for (int k = 0; k < K; k += 2) {
              *reinterpret_cast<int2*>(act_out + k) = make_int2(idx[k], idx[k + 1]);
              *reinterpret_cast<float2*>(w_out + k) = make_float2(ev[k], ev[k + 1]);
            }
          } else {
#pragma unroll
            for (int k = 0; k < K; ++k) { act_out[k] = idx[k]; w_out[k] = ev[k]; }
          }
          if constexpr (KA > 0) {
            int32_t* ad_out = a.adaptive + ot * KA;
            uint32_t m = amask;
#pragma unroll
            for (int k = 0; k < KA; ++k) { ad_out[k] = __ffs(m) - 1; m &= m - 1; }
          }
        }
#pragma unroll
        for (int k = 0; k < K; ++k) s_mass[(g * BM + r_loc) * (E + 1) + idx[k]] += ev[k];
      }
      // the accumulator is consumed: the MMA may start the tile after next in it
      tc_fence_before();
      mbar_arrive(&tempty[acc]);
      // bit planes -> four u8 counts per word (expert 4w + i in byte i): x * 0x204081 spreads the
      // four bits of a nibble to bit 0 of four bytes without carries
#pragma unroll
      for (int w = 0; w < E / 4; ++w) {
        uint32_t packed = 0u;
#pragma unroll
        for (int p = 0; p < kNPlanes; ++p) packed |= ((((cnt[p] >> (4 * w)) & 15u) * 0x204081u) & 0x01010101u) << p;
        s_cnt[(g * BM + r_loc) * (E / 4 + 1) + w] = valid ? packed : 0u;
      }
      s_un[g * BM + r_loc] = valid ? un : 0u;
      if (!valid) {
#pragma unroll
        for (int j = 0; j < E; ++j) s_mass[(g * BM + r_loc) * (E + 1) + j] = 0.f;
        if (DM) {
#pragma unroll
          for (int j = 0; j < E; ++j) s_dm[(g * BM + r_loc) * (E + 1) + j] = 0.f;
        }
      }
      bar_named(5, kEpi);
      if (g == 0 && valid) {
        uint32_t u = 0;
#pragma unroll
        for (int h = 0; h < TPR; ++h) u |= s_un[h * BM + r_loc];
        a.umask[b] = u;
        a.usize[b] = __popc(u);
      }
      // ---------------- per-chunk statistics in row order (deterministic)
#ifdef SMES_FRONT_NO_STATS
      if (nsub < 0)
#endif
      for (int pr = tid; pr < nsub * E; pr += kEpi) {
        const int sc = pr / E, e = pr - sc * E;
        const int c = (tile * rpc) / a.sub_rows + sc;
        if (c >= C) continue;
        int cu = 0, ca = 0;
        double m = 0.0, dmv = 0.0;
        for (int r = sc * a.sub_rows; r < (sc + 1) * a.sub_rows; ++r) {
          uint32_t ur = 0;
#pragma unroll
          for (int h = 0; h < TPR; ++h) {
            ur |= s_un[h * BM + r];
            ca += (s_cnt[(h * BM + r) * (E / 4 + 1) + (e >> 2)] >> (8 * (e & 3))) & 0xffu;
            m += (double)s_mass[(h * BM + r) * (E + 1) + e];
            if (DM) dmv += (double)s_dm[(h * BM + r) * (E + 1) + e];
          }
          cu += (ur >> e) & 1u;
        }
        const size_t o = (size_t)c * E + e;
        a.chunk_union[o] = cu;
        a.chunk_active[o] = ca;
        a.chunk_mass[o] = m;
        if (DM) a.chunk_dmass[o] = dmv;
      }
      if (tid == 0) *s_nf = 0;          // every read of the counter happened before the last barrier
      bar_named(5, kEpi);
    }
    bad = __any_sync(0xffffffffu, bad);
    if (bad && lane == 0) atomicOr(a.flag, 1);
    if (a.n_exact != nullptr) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) n_exact += __shfl_xor_sync(0xffffffffu, n_exact, o);
      if (lane == 0 && n_exact) atomicAdd(a.n_exact, n_exact);
    }
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

static int32_t* g_front_counter = nullptr;   // diagnostic: rows routed through the fp64 recompute

template <int E, int KS, int KA, bool DM>
static int front_launch(const CUtensorMap& ta, const CUtensorMap& tb, const front::Args& a, int grid,
                        cudaStream_t st) {
  auto kern = front::route_front_kernel<E, KS, KA, DM>;
  constexpr int bytes = front::Plan<E, DM>::kBytes;
  static bool attr = false;
  if (!attr) {
    cudaError_t ea = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (ea != cudaSuccess) return set_error(SMES_ERR_CUDA, "route_front smem attribute: %s", cudaGetErrorString(ea));
    attr = true;
  }
  smes_launch(kern, grid, front::kThreads, bytes, st, ta, tb, a);
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

void smes_route_front_count_exact(int32_t* dev_counter) { g_front_counter = dev_counter; }

int smes_route_front_supported(int T, int E, int d, int k_shared, int k_adaptive) {
  const bool e_ok = E == 16 || E == 32;
  const bool k_ok = (k_shared == 4 && k_adaptive == 2) || (k_shared == 2 && k_adaptive == 1);
  return e_ok && k_ok && T >= 2 && T <= 16 && T * E <= 256 && (T * E) % 16 == 0 && d >= 64 && d <= 256 &&
         d % 64 == 0 && k_shared + k_adaptive <= E;
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
  const int nc = (T * E) % 64 == 0 ? 64 : (T * E) % 32 == 0 ? 32 : 16;      // W_r chunk rows (see kernel)
  if ((rc = front_map(&tb, w_r, (uint64_t)d, (uint64_t)(T * E), (uint64_t)d, (uint32_t)nc))) return rc;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  // rows per CTA: a multiple of the statistics chunk, <= 128, small enough that the grid covers
  // every SM (c2: 112 rows x 147 CTAs instead of 128 x 128)
  int rpc = (B + sms - 1) / sms;
  rpc = (rpc + sub_rows - 1) / sub_rows * sub_rows;
  if (rpc > 128) rpc = 128;
  const int tiles = (B + rpc - 1) / rpc;
  const int grid = tiles < sms ? tiles : sms;
  front::Args a{b_r, task_weights, T, B, d, sub_rows, rpc, shared, adaptive, active, wsel, umask, usize,
                chunk_union, chunk_active, chunk_mass, chunk_dmass, flag, z_out, g_front_counter};
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const bool dm = chunk_dmass != nullptr;
  if (E == 16) return front_dispatch<16>(ta, tb, a, grid, k_shared, dm, st);
  return front_dispatch<32>(ta, tb, a, grid, k_shared, dm, st);
}

}  // extern "C"
