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
// with four threads per row, in the four warps that share a lane quarter:
//   Stage I   (split by expert quarters) p_t = softmax(z_t) and pooled = sum_t w_t p_t
//             in fp64, as route_kernel: exp, sums and pooling in double, the quarter
//             sums of each task exchanged through shared memory (fixed order); every
//             thread keeps its quarter's top-K_s, and the four sorted lists are merged
//             into shared = top-K_s of pooled, (score desc, index asc)  (routing.py:256-261).
//   Stage II  (split by tasks, t = g, g + 4, ...) exact fp32 compare of z_t with the
//             shared set excluded (:263-268), weights = softmax of z_t over the active
//             set (:203-211, :273), union bitmask (:272).
//   LoadStats partials per chunk of `sub_rows` rows (the plan's chunk, 4 * rows_per_warp):
//             union counts, active counts, sparse and (DM) dense mass per expert.  Each
//             thread leaves dense per-row partials in shared memory; a fixed-order reduce
//             over rows and threads produces the chunk sums (no atomics, deterministic;
//             balance.py:65-68, execution.py:109-113).
//
// Warp roles (640 threads, 1 CTA/SM): w0 TMA producer, w1 MMA issuer, w2 TMEM allocator,
// w4..w19 routing epilogue (warp w: lane quarter (w - 4) & 3, row thread g = (w - 4) >> 2).
#include "ptx.cuh"
#include "smes_capi.h"

namespace smes {

namespace front {

constexpr int BM = 128;
constexpr int BK = 64;
// TPR threads per row (2 or 4): 4 non-epilogue warps + 4 * TPR epilogue warps
template <int TPR> constexpr int kThreads = 128 + 128 * TPR;
template <int TPR> constexpr int kEpi = 128 * TPR;

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

template <int E, int TPR>
struct Plan {
  // the router GEMM is issued in N chunks of (up to) 64 columns, each committed on its own
  // barrier, so Stage I of the first tasks runs while the MMAs of the later tasks stream W_r
  static constexpr int kWStages = 4;
  static constexpr int kH = BM * BK * 2;          // 16 KB per k-block of h (d <= 256: 4 blocks)
  static constexpr int kW = 64 * BK * 2;          // 8 KB per (chunk, k-block) of W_r
  static constexpr int kOffW = 4 * kH;
  static constexpr int kOffBias = kOffW + kWStages * kW;         // T*E floats (<= 1 KB)
  static constexpr int kOffTw = kOffBias + 1024;                 // T doubles (<= 32)
  static constexpr int kOffM = kOffTw + 256;                     // [T][128] fp32 task maxima (T <= 16)
  // [TPR threads][E][128] fp32 per-row sparse-mass partials (Stage II); before that, the
  // per-thread top-K_s candidates [TPR][4][128] fp64 keys + [TPR][4][128] u8 indices (Stage I)
  static constexpr int kOffMass = kOffM + 16 * BM * 4;
  static constexpr int kOffDm = kOffMass + TPR * E * BM * 4;     // [E][128] fp32 dense mass
  static constexpr int kOffCnt = kOffDm + E * BM * 4;            // [TPR][E/4][128] u32, 4 packed u8 counts
  static constexpr int kOffSum = kOffCnt + TPR * E * BM;         // [2 parity][TPR][128] fp64 partial sums
  static constexpr int kOffUn = kOffSum + 2 * TPR * BM * 8;      // [TPR][128] u32 union words
  static constexpr int kOffBar = kOffUn + TPR * BM * 4;
  static constexpr int kBytes = kOffBar + 512 + 1024;
  static_assert(E <= 32, "one union word per row");
  static_assert(TPR * 4 * BM * 9 <= TPR * E * BM * 4, "candidate lists fit the mass region");
  static_assert(kBytes <= 232448, "front smem plan exceeds 227 KB");
};

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

// columns [c, c + N) of this thread's TMEM lane (warp-collective), N in {4, 8, 16}
template <int N>
__device__ __forceinline__ void tmem_ldn(uint32_t taddr, float (&v)[N]) {
  uint32_t r[N];
  if constexpr (N == 8) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(taddr));
  } else if constexpr (N == 16) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
  } else {
    static_assert(N == 4, "row-slice width");
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(taddr));
  }
#pragma unroll
  for (int j = 0; j < N; ++j) v[j] = __uint_as_float(r[j]);
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

template <int E, int KS, int KA, bool DM, int TPR>
__global__ void __launch_bounds__(kThreads<TPR>, 1)
    route_front_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                       const Args a) {
  using S = Plan<E, TPR>;
  constexpr int K = KS + KA;
  extern __shared__ __align__(16) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sH = smem;
  uint8_t* sW = smem + S::kOffW;
  float* sbias = reinterpret_cast<float*>(smem + S::kOffBias);
  double* stw = reinterpret_cast<double*>(smem + S::kOffTw);
  float* s_m = reinterpret_cast<float*>(smem + S::kOffM);
  float* s_mass = reinterpret_cast<float*>(smem + S::kOffMass);
  unsigned long long* s_ckey = reinterpret_cast<unsigned long long*>(smem + S::kOffMass);   // Stage I only
  uint8_t* s_cidx = smem + S::kOffMass + TPR * 4 * BM * 8;
  float* s_dm = reinterpret_cast<float*>(smem + S::kOffDm);
  uint32_t* s_cnt = reinterpret_cast<uint32_t*>(smem + S::kOffCnt);
  double* s_sum = reinterpret_cast<double*>(smem + S::kOffSum);
  uint32_t* s_un = reinterpret_cast<uint32_t*>(smem + S::kOffUn);
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
  const int num_tiles = (a.B + BM - 1) / BM;
  const int nkb = (a.d + BK - 1) / BK;
  // columns per chunk: <= 64 (the W_r ring slot), a multiple of E (whole tasks per chunk)
  const int NC = N % 64 == 0 ? 64 : N % 32 == 0 ? 32 : 16;
  const int nch = N / NC;

  for (int i = threadIdx.x; i < N; i += blockDim.x) sbias[i] = a.bias[i];
  for (int i = threadIdx.x; i < T; i += blockDim.x) stw[i] = a.tw[i];
  if (warp == 0 && lane == 0) { tma_prefetch(&tmA); tma_prefetch(&tmB); }
  if (warp == 1 && lane == 0) {
    for (int s = 0; s < S::kWStages; ++s) { mbar_init(&wfull[s], 1); mbar_init(&wempty[s], 1); }
    mbar_init(hfull, 1);
    mbar_init(hempty, 1);
    for (int s = 0; s < 32; ++s) mbar_init(&tfull[s], 1);
    for (int s = 0; s < 2; ++s) mbar_init(&tempty[s], kEpi<TPR>);
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
        for (int kb = 0; kb < nkb; ++kb) tma_load_2d(sH + kb * S::kH, &tmA, hfull, kb * BK, tile * BM);
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
    // ================= routing epilogue: four threads per row
    constexpr int EQ = E / TPR;              // Stage-I experts per thread
    const int q = (warp - 4) & 3;
    const int g = (warp - 4) >> 2;
    const int j0 = g * EQ;
    const int r_loc = 32 * q + lane;
    const int quad_bar = 1 + q;              // the TPR warps of this lane quarter
    const int nsub = BM / a.sub_rows;
    const int C = (a.B + a.sub_rows - 1) / a.sub_rows;
    int it = 0, bad = 0;
    for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++it) {
      const int acc = it & 1;
      const int b = tile * BM + r_loc;
      const bool valid = b < a.B;
      const uint32_t taddr = tmem_base + ((uint32_t)(32 * q) << 16) + acc * N;
#ifdef SMES_FRONT_GEMM_ONLY
      for (int c = 0; c < nch; ++c) mbar_wait(&tfull[acc * 16 + c], (it >> 1) & 1);
      tc_fence_before();
      mbar_arrive(&tempty[acc]);
      continue;
#endif

      // ---------------- Stage I (fp64): this thread's quarter of the experts of every task
      double pp[EQ];
      {
        float dm[EQ];
#pragma unroll
        for (int j = 0; j < EQ; ++j) { pp[j] = 0.0; dm[j] = 0.f; }
        int chunk = 0, next_chunk_task = 0;
        for (int t = 0; t < T; ++t) {
          if (t == next_chunk_task) {        // first task of a chunk: wait for its MMAs
            mbar_wait(&tfull[acc * 16 + chunk], (it >> 1) & 1);
            tc_fence_after();
            ++chunk;
            next_chunk_task += NC / E;
          }
          float zq[EQ];                       // this quarter's logits
          tmem_ldn<EQ>(taddr + t * E + j0, zq);
          float z[E];
          load_task<E>(taddr, sbias, t, z);   // (waits for both loads)
          const float mf = tree_max<E>(z);
          if (g == t % TPR) s_m[t * BM + r_loc] = mf;
          const double m = (double)mf;
#pragma unroll
          for (int j = 0; j < EQ; ++j) {
            zq[j] += sbias[t * E + j0 + j];
            bad |= !isfinite(zq[j]);
          }
          if (a.z_out != nullptr && valid) {
            float4* zo = reinterpret_cast<float4*>(a.z_out + (size_t)b * N + t * E + j0);
#pragma unroll
            for (int j = 0; j < EQ; j += 4) zo[j / 4] = make_float4(zq[j], zq[j + 1], zq[j + 2], zq[j + 3]);
          }
          double ev[EQ], s = 0.0;
#pragma unroll
          for (int j = 0; j < EQ; ++j) { ev[j] = exp((double)zq[j] - m); s += ev[j]; }
          double* slot = s_sum + (t & 1) * TPR * BM;
          slot[g * BM + r_loc] = s;
          bar_named(quad_bar, 32 * TPR);
          double stot = slot[r_loc];
#pragma unroll
          for (int h = 1; h < TPR; ++h) stot += slot[h * BM + r_loc];     // fixed order
          const double inv = 1.0 / stot;
          const double wt = stw[t];
#pragma unroll
          for (int j = 0; j < EQ; ++j) {
            const double p = ev[j] * inv;
            pp[j] = fma(wt, p, pp[j]);
            if (DM) dm[j] += (float)p;
          }
        }
        if (DM) {
#pragma unroll
          for (int j = 0; j < EQ; ++j) s_dm[(j0 + j) * BM + r_loc] = valid ? dm[j] : 0.f;
        }
      }
      // shared set: top-K_s of pooled, (score desc, index asc).  pooled >= 0, so the fp64 bit
      // patterns order like unsigned integers.  Each thread sorts its quarter, the four lists
      // are merged through shared memory.
      uint32_t smask = 0;
      if constexpr (KS > 0) {
        unsigned long long pk[EQ];
#pragma unroll
        for (int j = 0; j < EQ; ++j) pk[j] = (unsigned long long)__double_as_longlong(pp[j]);
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
            // (key desc, index asc); exhausted lists and empty slots (index 255) never win
            const bool take = ok & (idx != 255) & ((bidx == 255) | (key > best) | ((key == best) & (idx < bidx)));
            best = take ? key : best;
            bidx = take ? idx : bidx;
            bg = take ? h : bg;
          }
          smask |= 1u << bidx;
#pragma unroll
          for (int h = 0; h < TPR; ++h) head[h] += (h == bg);
        }
        if (g == 0 && valid) {
          uint32_t m = smask;
#pragma unroll
          for (int k = 0; k < KS; ++k) {
            a.shared[(size_t)b * KS + k] = __ffs(m) - 1;
            m &= m - 1;
          }
        }
      }
      bar_named(quad_bar, 32 * TPR);    // candidate reads done: the region becomes the mass partials

      // ---------------- Stage II: tasks g, g + 4, ...
      uint32_t cnt_p[E / 4];            // active counts, four u8 per word
#pragma unroll
      for (int j = 0; j < E / 4; ++j) cnt_p[j] = 0u;
      uint32_t un = smask;
      bool first = true;
      for (int t = g; t < T; t += TPR) {
        float z[E];
        load_task<E>(taddr, sbias, t, z);
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
        // max over the active set: with K_a >= 1 the row maximum is always active (shared, or the
        // first adaptive pick), so it is the task maximum of Stage I
        float amx;
        if constexpr (KA > 0) {
          amx = s_m[t * BM + r_loc];
        } else {
          amx = -INFINITY;
#pragma unroll
          for (int j = 0; j < E; ++j) amx = ((act >> j) & 1u) ? fmaxf(amx, z[j]) : amx;
        }
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
        int pos = 0, apos = 0;
#pragma unroll
        for (int j = 0; j < E; ++j) {
          const uint32_t bit = (act >> j) & 1u;
          const float w = z[j] * ainv;
          if (valid && bit) { act_out[pos] = j; w_out[pos] = w; }
          pos += bit;
          if (KA > 0) {
            const uint32_t abit = (amask >> j) & 1u;
            if (valid && abit) ad_out[apos] = j;
            apos += abit;
          }
          cnt_p[j >> 2] += bit << (8 * (j & 3));
          float* mp = s_mass + (g * E + j) * BM + r_loc;
          *mp = first ? w : *mp + w;
        }
        first = false;
      }
      if (first) {                      // no task for this thread (T < TPR)
#pragma unroll
        for (int j = 0; j < E; ++j) s_mass[(g * E + j) * BM + r_loc] = 0.f;
      }
      // the accumulator is consumed: the MMA may start the tile after next in it
      tc_fence_before();
      mbar_arrive(&tempty[acc]);
#pragma unroll
      for (int j = 0; j < E / 4; ++j) s_cnt[(g * (E / 4) + j) * BM + r_loc] = valid ? cnt_p[j] : 0u;
      s_un[g * BM + r_loc] = valid ? un : 0u;
      if (!valid) {
#pragma unroll
        for (int j = 0; j < E; ++j) s_mass[(g * E + j) * BM + r_loc] = 0.f;
        if (DM && g == 0) {
#pragma unroll
          for (int j = 0; j < E; ++j) s_dm[j * BM + r_loc] = 0.f;
        }
      }
      bar_named(5, kEpi<TPR>);
      if (g == 0 && valid) {
        uint32_t u = 0;
#pragma unroll
        for (int h = 0; h < TPR; ++h) u |= s_un[h * BM + r_loc];
        a.umask[b] = u;
        a.usize[b] = __popc(u);
      }
      // ---------------- per-chunk statistics in row order (deterministic)
      const int tid = threadIdx.x - 128;
      for (int pr = tid; pr < nsub * E; pr += kEpi<TPR>) {
        const int sc = pr / E, e = pr - sc * E;
        const int c = tile * nsub + sc;
        if (c >= C) continue;
        int cu = 0, ca = 0;
        double m = 0.0, dmv = 0.0;
        const int sh = 8 * (e & 3), wj = e >> 2;
        for (int r = sc * a.sub_rows; r < (sc + 1) * a.sub_rows; ++r) {
          uint32_t ur = 0;
#pragma unroll
          for (int h = 0; h < TPR; ++h) ur |= s_un[h * BM + r];
          cu += (ur >> e) & 1u;
#pragma unroll
          for (int h = 0; h < TPR; ++h) {
            ca += (s_cnt[(h * (E / 4) + wj) * BM + r] >> sh) & 0xffu;
            m += (double)s_mass[(h * E + e) * BM + r];
          }
          if (DM) dmv += (double)s_dm[e * BM + r];
        }
        const size_t o = (size_t)c * E + e;
        a.chunk_union[o] = cu;
        a.chunk_active[o] = ca;
        a.chunk_mass[o] = m;
        if (DM) a.chunk_dmass[o] = dmv;
      }
      bar_named(5, kEpi<TPR>);
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

#ifndef SMES_FRONT_TPR
#define SMES_FRONT_TPR 2
#endif

template <int E, int KS, int KA, bool DM>
static int front_launch(const CUtensorMap& ta, const CUtensorMap& tb, const front::Args& a, int grid,
                        cudaStream_t st) {
  constexpr int TPR = SMES_FRONT_TPR;
  auto kern = front::route_front_kernel<E, KS, KA, DM, TPR>;
  constexpr int bytes = front::Plan<E, TPR>::kBytes;
  static bool attr = false;
  if (!attr) {
    cudaError_t ea = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (ea != cudaSuccess) return set_error(SMES_ERR_CUDA, "route_front smem attribute: %s", cudaGetErrorString(ea));
    attr = true;
  }
  kern<<<grid, front::kThreads<TPR>, bytes, st>>>(ta, tb, a);
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
