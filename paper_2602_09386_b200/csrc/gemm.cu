// Grouped expert GEMM on sm_100a: TMA -> smem (SW128) -> tcgen05.mma (TMEM
// fp32 accumulators, double-buffered) -> tcgen05.ld epilogue -> smem -> TMA store.
//
// Replaces the reference's per-expert segment loop `grouped_gemm`
// (taskmoe/execution.py:126-158) and the expert part of `backward`
// (taskmoe/training.py:180-191).  One persistent, warp-specialised kernel
// template covers the three contractions of the SMES expert stack:
//
//   RAGGED_M, B K-major  (fwd):   C[m, n]  = act(sum_k A[m, k] W_g[n, k] + b_g[n])   rows m in group g
//   RAGGED_M, B MN-major (dgrad): C[m, n]  = mask(sum_k A[m, k] W_g[k, n])
//   RAGGED_K            (wgrad): C_g[i, j] = sum_{m in g} P[m, i] Q[m, j]            (fp32 out)
//
// Packed rows are grouped expert-major and every group is padded to a multiple
// of 128 rows (pad rows are zero in the operands), so an M-tile never straddles
// two experts and the wgrad reduction runs in whole 64-row K-blocks.  Group
// offsets live on the device: no host sync, CUDA-graph capturable.
//
// Warp roles (256 threads, 1 CTA/SM): w0 TMA producer, w1 MMA issuer,
// w2 TMEM allocator, w4..w7 epilogue (warp q%4 owns TMEM lanes 32q..32q+31).
#include <cstdlib>
#include "ptx.cuh"
#include "smes_capi.h"

namespace smes {

constexpr int BM = 128;
constexpr int BK = 64;
constexpr int kThreads = 384;   // 4 non-epilogue warps + 8 epilogue warps (2 per TMEM lane quarter)
constexpr int kEpiWarps = 8;

enum { MODE_RAGGED_M = 0, MODE_RAGGED_K = 1 };
// lanes of the producer warp issuing gathered rows (TMA gather4) in the ragged-K kernel
#ifndef SMES_GATHER_LANES
#define SMES_GATHER_LANES 8
#endif
constexpr int kGatherLanes = SMES_GATHER_LANES;

struct GemmArgs {
  const int* seg;             // (G+1) padded group offsets in rows (multiples of BM)
  int G;                      // groups
  int N;                      // ragged-M: output cols;   ragged-K: J
  int K;                      // ragged-M: reduction dim; ragged-K: unused
  int I;                      // ragged-K: output rows per group
  const float* bias;          // ragged-M fwd: (G, N) or null
  int act;                    // 0 identity, 1 relu
  uint32_t* bits_out;         // relu bitmask out: [(N/32)][bits_ld] words, or null
  const uint32_t* bits_in;    // relu bitmask applied to the output (dgrad), or null
  int bits_ld;
  float* db_out;              // ragged-K: per-group column sums of P via Q's ones column (G, I), or null
  int a_period;               // ragged-K: P rows are read modulo this period (a shared P for every group), or 0
  int x3;                     // ragged-M fp32 mode: K of one bf16 plane (A, W = three planes hi|mid|lo), or 0
  int ksplit;                 // ragged-K: K split into this many contiguous parts (partials at group s G + g), or 0
  const int* gather;          // ragged-K: Q row r is source row gather[r] (tmB maps the source, box {64, 1};
                              // -1 reads zeros), or null
};

// fp32-accurate products from bf16 planes: x = x0 + x1 + x2 with x_i = bf16(x - x_0 - .. - x_{i-1})
// (8 significant bits each, 24 in all).  The six leading cross terms a_i b_j (i + j <= 2) are summed
// as one GEMM over a virtual K of 6 planes, smallest terms first; the dropped terms are below
// 2^-24 relative.  Virtual plane s reads A plane (kX3A >> 4s) & 15 and W plane (kX3B >> 4s) & 15.
constexpr uint32_t kX3A = 0x001012u;   // a2 a1 a0 a1 a0 a0
constexpr uint32_t kX3B = 0x010210u;   // b0 b1 b2 b0 b1 b0

// Shared-memory plan.  ragged-M tiles are epilogue(store)-paced at the c2 shapes, so every
// epilogue warp double-buffers its 4 KB TMA-store staging chunk (ncu r1: the single-buffer
// bulk wait was the top stall); ragged-K (wgrad) runs long K loops and stores once per tile.
// ragged-K with BN = 256: 4 k-block stages, the epilogue's TMA-store staging aliased onto the
// first stage slots (a long K loop stores once per tile; the producer starts the next tile only
// after the staging reads completed).  fc1 wgrad at c2: 95 -> 85 us.
#ifndef SMES_RK256_STAGES
#define SMES_RK256_STAGES 4
#endif
template <int BN, int MODE>
struct Smem {
  static constexpr int kStages = MODE == MODE_RAGGED_K ? (BN == 256 ? SMES_RK256_STAGES : BN == 128 ? 5 : 6)
                                                       : (BN == 256 ? 3 : BN == 128 ? 4 : 6);
  static constexpr bool kStgAlias = MODE == MODE_RAGGED_K && BN == 256 && SMES_RK256_STAGES > 3;
  static constexpr int kAccStages = MODE == MODE_RAGGED_K ? 1 : 2;
  static constexpr int kStgBufs = MODE == MODE_RAGGED_K ? 1 : 2;
  static constexpr int kA = BM * BK * 2;                         // 16 KB
  static constexpr int kB = (BN < 64 && MODE == MODE_RAGGED_K ? 64 : BN) * BK * 2;   // MN-major boxes are 64 wide
  static constexpr int kStg = 32 * 128;                          // 4 KB per staging buffer
  static constexpr int kOffB = kStages * kA;
  static constexpr int kOffOnes = kOffB + kStages * kB;                       // ragged-K: 64x64 bf16 ones tile
  static constexpr int kOffStg = kStgAlias ? 0 : kOffOnes + (MODE == MODE_RAGGED_K ? 8192 : 0);
  static constexpr int kOffBias = (kStgAlias ? kOffOnes + 8192 : kOffStg + kEpiWarps * kStgBufs * kStg);
  static constexpr int kOffBar = kOffBias + kEpiWarps * 256;
  static constexpr int kOffSeg = kOffBar + 256;
  static constexpr int kOffIdx = (kOffSeg + 257 * 4 + 12 + 15) / 16 * 16;   // ragged-K gather: 8 x 64 row indices
  static constexpr int kBytes = kOffIdx + (MODE == MODE_RAGGED_K ? 2048 : 0) + 1024;   // + alignment slack
  static constexpr int kTmemCols = 2 * BN;
  static_assert(kBytes <= 232448, "shared memory plan exceeds 227 KB");
};

__device__ __forceinline__ int find_group(const int* seg_s, int G, int row) {
  // largest g with seg[g] <= row  (segments are padded, so row lies inside a non-empty one)
  int lo = 0, hi = G - 1;
  while (lo < hi) {
    int mid = (lo + hi + 1) >> 1;
    if (seg_s[mid] <= row) lo = mid; else hi = mid - 1;
  }
  return lo;
}

template <int BN, int MODE, bool B_MN, bool F32>
__global__ void __launch_bounds__(kThreads, 1)
    grouped_gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                        const __grid_constant__ CUtensorMap tmC, const GemmArgs args) {
  pdl_wait();
  using S = Smem<BN, MODE>;
  constexpr int kStages = S::kStages;
  constexpr int kAcc = S::kAccStages;
  constexpr int CPC = F32 ? 32 : 64;                 // output columns per 128-byte staged row chunk
  constexpr int NCH = BN / CPC > 0 ? BN / CPC : 1;   // chunks per tile
  constexpr int MYCH = (NCH + 1) / 2;                // chunks per epilogue warp (column parity split)
  constexpr int NBBOX = BN / 64 > 0 ? BN / 64 : 1;   // 64-wide MN-major B boxes per stage
  extern __shared__ __align__(16) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);   // stays in the shared window
  uint8_t* sA = smem;
  uint8_t* sB = smem + S::kOffB;
  uint8_t* sOnes = smem + S::kOffOnes;
  uint8_t* sStg = smem + S::kOffStg;       // (re-pointed below for the aliased ragged-K layout)
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + S::kOffBar);
  uint64_t* empty = full + kStages;
  uint64_t* tfull = empty + kStages;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  int* seg_s = reinterpret_cast<int*>(smem + S::kOffSeg);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const bool fused_bias = MODE == MODE_RAGGED_K && args.db_out != nullptr;

  for (int i = threadIdx.x; i <= args.G; i += blockDim.x) seg_s[i] = args.seg[i];
  if (MODE == MODE_RAGGED_K) {
    // ones tile as an MN-major SW128 B operand: B'[k][n] = (n == 0) for 64 k-rows x 64 n-cols
    uint32_t* o32 = reinterpret_cast<uint32_t*>(sOnes);
    for (int i = threadIdx.x; i < 8192 / 4; i += blockDim.x) o32[i] = 0u;
    __syncthreads();
    if (threadIdx.x < 64) {
      const int k = threadIdx.x;   // element n = 0 of row k sits in 16B chunk (0 ^ (k & 7))
      reinterpret_cast<__nv_bfloat16*>(sOnes + k * 128 + (k & 7) * 16)[0] = __float2bfloat16_rn(1.f);
    }
    fence_proxy_async_smem();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmA);
    tma_prefetch(&tmB);
    tma_prefetch(&tmC);
  }
  if (warp == 1 && lane == 0) {
    for (int s = 0; s < kStages; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    for (int s = 0; s < 2; ++s) { mbar_init(&tfull[s], 1); mbar_init(&tempty[s], kEpiWarps * 32); }
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, S::kTmemCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  // ---- tile space
  int num_tiles, n_tiles = 0, i_tiles = 0, j_tiles = 0;
  if (MODE == MODE_RAGGED_M) {
    n_tiles = (args.N + BN - 1) / BN;
    num_tiles = (seg_s[args.G] / BM) * n_tiles;
  } else {
    i_tiles = (args.I + BM - 1) / BM;
    j_tiles = (args.N + BN - 1) / BN;
    num_tiles = args.G * i_tiles * j_tiles * (args.ksplit > 1 ? args.ksplit : 1);
  }
  // ring depth and store staging of the ragged-K BN = 256 layout (see Smem)
  const bool one_tile = num_tiles <= (int)gridDim.x;
  const int nst = (S::kStgAlias && !one_tile) ? kStages - 1 : kStages;
  if (S::kStgAlias) sStg = one_tile ? smem : smem + S::kOffB + (kStages - 1) * S::kB;
  // decode: (group, row0 of A / i0, n0 / j0, k-block range); go = output group (split-K partial slot)
  const int ks = args.ksplit > 1 ? args.ksplit : 1;
  auto decode = [&](int tile, int& g, int& r0, int& c0, int& kb0, int& nkb, int& go) {
    if (MODE == MODE_RAGGED_M) {
      int mt = tile / n_tiles;
      r0 = mt * BM;
      c0 = (tile - mt * n_tiles) * BN;
      g = find_group(seg_s, args.G, r0);
      kb0 = 0;
      nkb = (args.K + BK - 1) / BK;
      go = g;
    } else {
      const int per = i_tiles * j_tiles;
      const int gs = tile / per;
      g = gs / ks;
      const int sp = gs - g * ks;
      const int r = tile - gs * per;
      r0 = (r / j_tiles) * BM;
      c0 = (r % j_tiles) * BN;
      const int tot = (seg_s[g + 1] - seg_s[g]) / BK;
      const int chunk = (tot + ks - 1) / ks;
      kb0 = seg_s[g] / BK + sp * chunk;
      nkb = max(0, min(chunk, tot - sp * chunk));
      go = sp * args.G + g;
    }
  };

  if (warp == 0) {
    if (MODE == MODE_RAGGED_K && args.gather != nullptr && lane < kGatherLanes) {
      // ================= TMA producer, gathered Q: each k-block's 64 rows straight from the source
      // rows (TMA gather4, 4 rows per op), issued by kGatherLanes lanes together (one issuing
      // thread managed ~1 op / 75 cycles).  Each lane copies its own row indices to shared memory
      // (LDGSTS) 4 k-blocks ahead of their use, through an 8-slot ring.
      constexpr unsigned kMask = (1u << kGatherLanes) - 1u;
      int* sIdx = reinterpret_cast<int*>(smem + S::kOffIdx);
      int stage = 0;
      uint32_t phase = 0;
      for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
        int g, r0, c0, kb0, nkb, go;
        decode(tile, g, r0, c0, kb0, nkb, go);
        auto pf = [&](int kb) {
          if (kb < nkb) {
            const int* src = args.gather + (long)(kb0 + kb) * BK;
#pragma unroll
            for (int q = lane; q < BK / 4; q += kGatherLanes) cp_async16(sIdx + (kb & 7) * BK + 4 * q, src + 4 * q);
          }
          cp_async_commit();
        };
#pragma unroll
        for (int p = 0; p < 4; ++p) pf(p);
        for (int kb = 0; kb < nkb; ++kb) {
          pf(kb + 4);
          cp_async_wait<4>();
          uint8_t* a = sA + stage * S::kA;
          uint8_t* b = sB + stage * S::kB;
          const int k0 = (kb0 + kb) * BK;
          if (lane == 0) {
            mbar_wait(&empty[stage], phase ^ 1);
            mbar_expect_tx(&full[stage], S::kA + S::kB);
#pragma unroll
            for (int j = 0; j < BM / 64; ++j)
              tma_load_2d(a + j * 8192, &tmA, &full[stage], r0 + 64 * j, args.a_period ? k0 % args.a_period : k0);
          }
          __syncwarp(kMask);
          const int4* ix = reinterpret_cast<const int4*>(sIdx + (kb & 7) * BK);
#pragma unroll
          for (int q = lane; q < BK / 4; q += kGatherLanes) {
            const int4 r = ix[q];
#pragma unroll
            for (int j = 0; j < NBBOX; ++j)
              tma_gather4(b + j * 8192 + q * 512, &tmB, &full[stage], c0 + 64 * j, r.x, r.y, r.z, r.w);
          }
          if (++stage == nst) { stage = 0; phase ^= 1; }
        }
      }
      cp_async_wait<0>();
    } else if (lane == 0) {
      // ================= TMA producer
      int stage = 0;
      uint32_t phase = 0;
      for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
        int g, r0, c0, kb0, nkb, go;
        decode(tile, g, r0, c0, kb0, nkb, go);
        for (int kb = 0; kb < nkb; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          mbar_expect_tx(&full[stage], S::kA + S::kB);
          uint8_t* a = sA + stage * S::kA;
          uint8_t* b = sB + stage * S::kB;
          const int k0 = (kb0 + kb) * BK;
          if (MODE == MODE_RAGGED_M) {
            int ka = k0, kw = k0;
            if (args.x3) {           // virtual plane -> (A plane, W plane)
              const int sp = k0 / args.x3, kin = k0 - sp * args.x3;
              ka = (int)((kX3A >> (4 * sp)) & 15u) * args.x3 + kin;
              kw = (int)((kX3B >> (4 * sp)) & 15u) * args.x3 + kin;
            }
            tma_load_2d(a, &tmA, &full[stage], ka, r0);                       // box {64 k, 128 rows}
            if (!B_MN) {
              tma_load_3d(b, &tmB, &full[stage], kw, c0, g);                  // box {64 k, BN n, 1}
            } else {
#pragma unroll
              for (int j = 0; j < BN / 64; ++j)                               // box {64 n, 64 k, 1}
                tma_load_3d(b + j * 8192, &tmB, &full[stage], c0 + 64 * j, k0, g);
            }
          } else {
#pragma unroll
            for (int j = 0; j < BM / 64; ++j)
              tma_load_2d(a + j * 8192, &tmA, &full[stage], r0 + 64 * j, args.a_period ? k0 % args.a_period : k0);
#pragma unroll
            for (int j = 0; j < NBBOX; ++j) tma_load_2d(b + j * 8192, &tmB, &full[stage], c0 + 64 * j, k0);
          }
          if (++stage == nst) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ================= MMA issuer (single thread)
      constexpr bool A_MN = (MODE == MODE_RAGGED_K);
      constexpr bool BMN = (MODE == MODE_RAGGED_K) || B_MN;
      constexpr uint32_t idesc = umma_idesc_bf16(BM, BN, A_MN ? 1 : 0, BMN ? 1 : 0);
      constexpr uint32_t idesc_bias = umma_idesc_bf16(BM, 16, 1, 1);     // D[:, 0:16] += A * ones-tile
      const uint32_t ones_addr = smem_u32(sOnes);
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++it) {
        int g, r0, c0, kb0, nkb, go;
        decode(tile, g, r0, c0, kb0, nkb, go);
        const int acc = it % kAcc;
        const uint32_t aphase = (it / kAcc) & 1;
        mbar_wait(&tempty[acc], aphase ^ 1);
        tc_fence_after();
        const uint32_t tmem_d = tmem_base + acc * BN;
        const bool with_bias = fused_bias && c0 == 0;    // once per (group, i-tile)
        for (int kb = 0; kb < nkb; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t a_addr = smem_u32(sA + stage * S::kA);
          const uint32_t b_addr = smem_u32(sB + stage * S::kB);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            uint64_t ad = A_MN ? umma_desc_sw128(a_addr + k * 2048, 8192, 1024)
                               : umma_desc_sw128(a_addr + k * 32, 16, 1024);
            uint64_t bd = BMN ? umma_desc_sw128(b_addr + k * 2048, 8192, 1024)
                              : umma_desc_sw128(b_addr + k * 32, 16, 1024);
            tc_mma_f16(tmem_d, ad, bd, idesc, (kb | k) != 0);
            if (with_bias)   // bias grad db[i] = sum_m P[m, i]: same A, constant ones B (cols BN..BN+15)
              tc_mma_f16(tmem_base + BN, ad, umma_desc_sw128(ones_addr + k * 2048, 8192, 1024), idesc_bias,
                         (kb | k) != 0);
          }
          tc_commit(&empty[stage]);        // smem slot free once these MMAs have read it
          if (++stage == nst) { stage = 0; phase ^= 1; }
        }
        tc_commit(&tfull[acc]);            // accumulator ready (also fires for nkb == 0)
      }
    }
  } else if (warp >= 4) {
    // ================= epilogue: TMEM -> regs -> (bias, act, mask) -> smem (SW128) -> TMA store
    // warp w owns TMEM lanes 32*(w%4).. and the column chunks of parity (w-4)/4
    const int q = warp & 3;
    const int par = (warp - 4) >> 2;
    uint8_t* stg0 = sStg + (warp - 4) * S::kStgBufs * S::kStg;
    float* sbias = reinterpret_cast<float*>(smem + S::kOffBias) + (warp - 4) * 64;
    const int ncols = args.N;
    int it = 0, nstore = 0;
    for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++it) {
      int g, r0, c0, kb0, nkb, go;
      decode(tile, g, r0, c0, kb0, nkb, go);
      const int row = r0 + 32 * q + lane;    // this thread's output row (packed row or i)
      // prefetch (before waiting for the MMA): relu bit-mask words and bias values of my chunks
      uint32_t mw[MYCH][2];
      float bv[MYCH][2];
#pragma unroll
      for (int i = 0; i < MYCH; ++i) {
        const int n = c0 + (par + 2 * i) * CPC;
        const bool ok = (par + 2 * i) < NCH && n < ncols;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          mw[i][h] = 0u;
          bv[i][h] = 0.f;
          if (MODE == MODE_RAGGED_M && h * 32 < CPC && ok && n + 32 * h < ncols) {
            if (args.bits_in != nullptr) mw[i][h] = __ldg(&args.bits_in[(size_t)((n >> 5) + h) * args.bits_ld + row]);
            if (args.bias != nullptr && n + 32 * h + lane < ncols)
              bv[i][h] = __ldg(args.bias + (size_t)g * args.N + n + 32 * h + lane);
          }
        }
      }
      const int acc = it % kAcc;
      const uint32_t aphase = (it / kAcc) & 1;
      mbar_wait(&tfull[acc], aphase);
      tc_fence_after();
      const uint32_t tbase = tmem_base + ((uint32_t)(32 * q) << 16) + acc * BN;
      if (fused_bias && c0 == 0 && par == 0) {
        // bias grad: column 0 of the ones-product accumulator at TMEM column BN
        uint32_t t0[32];
        tmem_ld32(tmem_base + ((uint32_t)(32 * q) << 16) + BN, t0);
        tmem_ld_wait();
        if (row < args.I) args.db_out[(size_t)go * args.I + row] = nkb > 0 ? __uint_as_float(t0[0]) : 0.f;
      }
#pragma unroll
      for (int i = 0; i < MYCH; ++i) {
        const int cc = par + 2 * i;
        const int n = c0 + cc * CPC;
        if (cc >= NCH || n >= ncols) break;
        float f[CPC];
        if (nkb > 0) {
#pragma unroll
          for (int h = 0; h < CPC / 32; ++h) {
            uint32_t t[32];
            tmem_ld32(tbase + cc * CPC + 32 * h, t);
            tmem_ld_wait();
#pragma unroll
            for (int j = 0; j < 32; ++j) f[32 * h + j] = __uint_as_float(t[j]);
          }
        } else {
#pragma unroll
          for (int j = 0; j < CPC; ++j) f[j] = 0.f;
        }
        if (MODE == MODE_RAGGED_M) {
          if (args.bias != nullptr) {
            // bias of these CPC columns, broadcast through a warp-private smem slot
            __syncwarp();
#pragma unroll
            for (int h = 0; h < CPC / 32; ++h) sbias[32 * h + lane] = bv[i][h];
            __syncwarp();
#pragma unroll
            for (int j = 0; j < CPC; j += 4) {
              const float4 bb = *reinterpret_cast<const float4*>(sbias + j);
              f[j] += bb.x; f[j + 1] += bb.y; f[j + 2] += bb.z; f[j + 3] += bb.w;
            }
          }
          if (args.act == 1) {
#pragma unroll
            for (int j = 0; j < CPC; ++j) f[j] = f[j] > 0.f ? f[j] : 0.f;
          }
          if (args.bits_out != nullptr) {
#pragma unroll
            for (int h = 0; h < CPC / 32; ++h) {
              if (n + h * 32 < ncols) {
                const uint32_t w = pos_mask32(f + h * 32);
                args.bits_out[(size_t)((n >> 5) + h) * args.bits_ld + row] = w;
              }
            }
          }
          if (args.bits_in != nullptr) {
#pragma unroll
            for (int h = 0; h < CPC / 32; ++h) {
              const uint32_t w = mw[i][h];
#pragma unroll
              for (int j = 0; j < 32; ++j) f[h * 32 + j] = ((w >> j) & 1u) ? f[h * 32 + j] : 0.f;
            }
          }
        }
        // stage into smem (128 B per row, 128B swizzle) and TMA-store a {CPC x 32} box; the
        // staging buffers alternate so this chunk's STS overlaps the previous chunk's store
        uint8_t* stg = stg0 + (nstore % S::kStgBufs) * S::kStg;
        ++nstore;
        if (lane == 0) {
          if (S::kStgBufs == 2) bulk_wait_read<1>(); else bulk_wait_read<0>();
        }
        __syncwarp();
        uint4* rowp = reinterpret_cast<uint4*>(stg + lane * 128);
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          uint4 pk;
          if (F32) {
            pk = make_uint4(__float_as_uint(f[4 * c]), __float_as_uint(f[4 * c + 1]), __float_as_uint(f[4 * c + 2]),
                            __float_as_uint(f[4 * c + 3]));
          } else {
            pk = make_uint4(pack_bf16(f[8 * c], f[8 * c + 1]), pack_bf16(f[8 * c + 2], f[8 * c + 3]),
                            pack_bf16(f[8 * c + 4], f[8 * c + 5]), pack_bf16(f[8 * c + 6], f[8 * c + 7]));
          }
          rowp[c ^ (lane & 7)] = pk;
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          if (MODE == MODE_RAGGED_M) tma_store_2d(&tmC, stg, n, r0 + 32 * q);
          else tma_store_3d(&tmC, stg, n, r0 + 32 * q, go);
          bulk_commit();
        }
      }
      tc_fence_before();
      mbar_arrive(&tempty[acc]);
    }
    if (lane == 0) bulk_wait<0>();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_dealloc(tmem_base, S::kTmemCols);
}

// ============================================================================ CTA pairs
// Ragged-M GEMM on CTA pairs (cta_group::2, cluster of 2): a unit is two 128-row tiles of the SAME
// group (the second one empty when the group has an odd tile count) times a 256-wide N tile.  Each
// CTA loads its own A tile and its 128-column half of the B tile; the leader issues M = 256 MMAs
// that read both CTAs' smem, and every CTA drains its own 128 TMEM lanes.  Per CTA the B stream
// is half of the single-CTA kernel's, so the large banks (c3 / c5 fc1, N >= 1024) are no longer
// bound by the L2 -> SMEM fill rate (torch._grouped_mm ran the c3 fc1 10 % faster than the
// single-CTA kernel).
template <bool B_MN, bool F32>
struct PairSmem {
  static constexpr int BN = 256;
  static constexpr int kStages = 4;
  static constexpr int kA = BM * BK * 2;            // 16 KB: own 128 rows
  static constexpr int kB = (BN / 2) * BK * 2;      // 16 KB: own half of the N tile
  static constexpr int kStg = 32 * 128;
  static constexpr int kOffB = kStages * kA;
  static constexpr int kOffStg = kOffB + kStages * kB;
  static constexpr int kOffBias = kOffStg + kEpiWarps * 2 * kStg;
  static constexpr int kOffBar = kOffBias + kEpiWarps * 256;
  static constexpr int kOffSeg = kOffBar + 256;
  static constexpr int kBytes = kOffSeg + 2 * 258 * 4 + 1024;
  static_assert(kBytes <= 232448, "pair GEMM smem");
};

template <bool B_MN, bool F32>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    grouped_gemm_pair_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                             const __grid_constant__ CUtensorMap tmC, const GemmArgs args) {
  pdl_wait();
  using S = PairSmem<B_MN, F32>;
  constexpr int BN = S::BN;
  constexpr int kStages = S::kStages;
  constexpr int CPC = F32 ? 32 : 64;                 // output columns per 128-byte staged row chunk
  constexpr int NCH = BN / CPC;
  constexpr int MYCH = NCH / 2;
  constexpr uint16_t kPair = 0x3;
  extern __shared__ __align__(16) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sA = smem;
  uint8_t* sB = smem + S::kOffB;
  uint8_t* sStg = smem + S::kOffStg;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + S::kOffBar);
  uint64_t* empty = full + kStages;
  uint64_t* tfull = empty + kStages;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  int* seg_s = reinterpret_cast<int*>(smem + S::kOffSeg);
  int* upref = seg_s + 258;                          // tile-pair units per group, prefix

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  for (int i = threadIdx.x; i <= args.G; i += blockDim.x) seg_s[i] = args.seg[i];
  __syncthreads();
  if (threadIdx.x == 0) {
    int u = 0;
    for (int g = 0; g < args.G; ++g) {
      upref[g] = u;
      u += ((seg_s[g + 1] - seg_s[g]) / BM + 1) / 2;
    }
    upref[args.G] = u;
  }
  if (warp == 0 && lane == 0) { tma_prefetch(&tmA); tma_prefetch(&tmB); tma_prefetch(&tmC); }
  if (warp == 1 && lane == 0) {
    for (int s = 0; s < kStages; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    for (int s = 0; s < 2; ++s) { mbar_init(&tfull[s], 1); mbar_init(&tempty[s], 2 * kEpiWarps); }
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc_2sm(tmem_slot, 2 * BN);
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int n_tiles = (args.N + BN - 1) / BN;
  const int num_units = upref[args.G] * n_tiles;
  const int nkb = (args.K + BK - 1) / BK;
  const int cl = blockIdx.x >> 1, ncl = gridDim.x >> 1;
  // unit -> group, first row of the tile pair, tiles in the pair (1 or 2), n0
  auto decode = [&](int u, int& g, int& rp, int& nt, int& n0) {
    const int pu = u / n_tiles;
    n0 = (u - pu * n_tiles) * BN;
    int lo = 0, hi = args.G - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (upref[mid] <= pu) lo = mid; else hi = mid - 1;
    }
    g = lo;
    const int j = pu - upref[g];
    rp = seg_s[g] + 2 * j * BM;
    nt = min(2, (seg_s[g + 1] - seg_s[g]) / BM - 2 * j);
  };

  if (warp == 0) {
    if (lane == 0) {
      // ================= TMA producer (both CTAs): own A tile, own half of the B tile
      int stage = 0;
      uint32_t phase = 0;
      for (int u = cl; u < num_units; u += ncl) {
        int g, rp, nt, n0;
        decode(u, g, rp, nt, n0);
        const bool valid = (int)rank < nt;
        const int r0 = rp + (int)rank * BM;
        const int nb = n0 + (int)rank * (BN / 2);
        for (int kb = 0; kb < nkb; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          if (rank == 0) mbar_expect_tx(&full[stage], nt * S::kA + 2 * S::kB);
          uint8_t* a = sA + stage * S::kA;
          uint8_t* b = sB + stage * S::kB;
          const int k0 = kb * BK;
          if (valid) tma_load_2d_2sm(a, &tmA, &full[stage], k0, r0);                 // {64 k, 128 rows}
          if (!B_MN) {
            tma_load_3d_2sm(b, &tmB, &full[stage], k0, nb, g);                         // {64 k, 128 n, 1}
          } else {
#pragma unroll
            for (int j = 0; j < 2; ++j) tma_load_3d_2sm(b + j * 8192, &tmB, &full[stage], nb + 64 * j, k0, g);
          }
          if (++stage == kStages) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && rank == 0) {
      // ================= MMA issuer (leader): M = 256 over the pair, N = 256
      constexpr uint32_t idesc = umma_idesc_bf16(2 * BM, BN, 0, B_MN ? 1 : 0);
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int u = cl; u < num_units; u += ncl, ++it) {
        const int acc = it & 1;
        mbar_wait(&tempty[acc], ((it >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t tmem_d = tmem_base + acc * BN;
        for (int kb = 0; kb < nkb; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t a_addr = smem_u32(sA + stage * S::kA);
          const uint32_t b_addr = smem_u32(sB + stage * S::kB);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            const uint64_t ad = umma_desc_sw128(a_addr + k * 32, 16, 1024);
            const uint64_t bd = B_MN ? umma_desc_sw128(b_addr + k * 2048, 8192, 1024)
                                     : umma_desc_sw128(b_addr + k * 32, 16, 1024);
            tc_mma_f16_2sm(tmem_d, ad, bd, idesc, (kb | k) != 0);
          }
          tc_commit_2sm_mc(&empty[stage], kPair);
          if (++stage == kStages) { stage = 0; phase ^= 1; }
        }
        tc_commit_2sm_mc(&tfull[acc], kPair);
      }
    }
  } else if (warp >= 4) {
    // ================= epilogue (both CTAs): own 128 rows; releases the accumulator on the leader
    const int q = warp & 3;
    const int par = (warp - 4) >> 2;
    uint8_t* stg0 = sStg + (warp - 4) * 2 * S::kStg;
    float* sbias = reinterpret_cast<float*>(smem + S::kOffBias) + (warp - 4) * 64;
    const uint32_t lead_tempty0 = mapa_shared(smem_u32(&tempty[0]), 0);
    const uint32_t lead_tempty1 = mapa_shared(smem_u32(&tempty[1]), 0);
    const int ncols = args.N;
    int it = 0, nstore = 0;
    for (int u = cl; u < num_units; u += ncl, ++it) {
      int g, rp, nt, n0;
      decode(u, g, rp, nt, n0);
      const bool valid = (int)rank < nt;
      const int r0 = rp + (int)rank * BM;
      const int row = r0 + 32 * q + lane;
      uint32_t mw[MYCH][2];
      float bv[MYCH][2];
#pragma unroll
      for (int i = 0; i < MYCH; ++i) {
        const int n = n0 + (par + 2 * i) * CPC;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          mw[i][h] = 0u;
          bv[i][h] = 0.f;
          if (valid && h * 32 < CPC && n + 32 * h < ncols) {
            if (args.bits_in != nullptr) mw[i][h] = __ldg(&args.bits_in[(size_t)((n >> 5) + h) * args.bits_ld + row]);
            if (args.bias != nullptr && n + 32 * h + lane < ncols)
              bv[i][h] = __ldg(args.bias + (size_t)g * args.N + n + 32 * h + lane);
          }
        }
      }
      const int acc = it & 1;
      mbar_wait(&tfull[acc], (it >> 1) & 1);
      tc_fence_after();
      const uint32_t tbase = tmem_base + ((uint32_t)(32 * q) << 16) + acc * BN;
#pragma unroll
      for (int i = 0; i < MYCH; ++i) {
        const int cc = par + 2 * i;
        const int n = n0 + cc * CPC;
        if (n >= ncols) break;
        float f[CPC];
#pragma unroll
        for (int h = 0; h < CPC / 32; ++h) {
          uint32_t t[32];
          tmem_ld32(tbase + cc * CPC + 32 * h, t);
          tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < 32; ++j) f[32 * h + j] = __uint_as_float(t[j]);
        }
        if (!valid) continue;            // (warp-uniform: the whole CTA holds the pair's empty tile)
        if (args.bias != nullptr) {
          __syncwarp();
#pragma unroll
          for (int h = 0; h < CPC / 32; ++h) sbias[32 * h + lane] = bv[i][h];
          __syncwarp();
#pragma unroll
          for (int j = 0; j < CPC; j += 4) {
            const float4 bb = *reinterpret_cast<const float4*>(sbias + j);
            f[j] += bb.x; f[j + 1] += bb.y; f[j + 2] += bb.z; f[j + 3] += bb.w;
          }
        }
        if (args.act == 1) {
#pragma unroll
          for (int j = 0; j < CPC; ++j) f[j] = f[j] > 0.f ? f[j] : 0.f;
        }
        if (args.bits_out != nullptr) {
#pragma unroll
          for (int h = 0; h < CPC / 32; ++h) {
            if (n + h * 32 < ncols) args.bits_out[(size_t)((n >> 5) + h) * args.bits_ld + row] = pos_mask32(f + h * 32);
          }
        }
        if (args.bits_in != nullptr) {
#pragma unroll
          for (int h = 0; h < CPC / 32; ++h) {
            const uint32_t w = mw[i][h];
#pragma unroll
            for (int j = 0; j < 32; ++j) f[h * 32 + j] = ((w >> j) & 1u) ? f[h * 32 + j] : 0.f;
          }
        }
        uint8_t* stg = stg0 + (nstore & 1) * S::kStg;
        ++nstore;
        if (lane == 0) bulk_wait_read<1>();
        __syncwarp();
        uint4* rowp = reinterpret_cast<uint4*>(stg + lane * 128);
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          uint4 pk;
          if (F32) {
            pk = make_uint4(__float_as_uint(f[4 * c]), __float_as_uint(f[4 * c + 1]), __float_as_uint(f[4 * c + 2]),
                            __float_as_uint(f[4 * c + 3]));
          } else {
            pk = make_uint4(pack_bf16(f[8 * c], f[8 * c + 1]), pack_bf16(f[8 * c + 2], f[8 * c + 3]),
                            pack_bf16(f[8 * c + 4], f[8 * c + 5]), pack_bf16(f[8 * c + 6], f[8 * c + 7]));
          }
          rowp[c ^ (lane & 7)] = pk;
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          tma_store_2d(&tmC, stg, n, r0 + 32 * q);
          bulk_commit();
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(acc ? lead_tempty1 : lead_tempty0);
    }
    if (lane == 0) bulk_wait<0>();
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  if (warp == 2) tmem_dealloc_2sm(tmem_base, 2 * BN);
}

// Ragged-K (weight gradient) on CTA pairs: C_g[i, j] = sum_{m in g} P[m, i] Q[m, j] with a unit =
// (group, two 128-row i tiles, 256-wide j tile); each CTA loads its own i tile of P (MN-major) and
// its half of the j tile of Q (MN-major), the leader's M = 256 MMAs run the group's whole K range.
// db_g[i] = sum_m P[m, i] (the fused bias gradient) comes from a second N = 16 MMA against a
// constant ones operand (K-major: row n = 0 of the leader's half is all ones), TMEM columns
// BN .. BN + 15, on the unit's first j tile.
struct PairKSmem {
  static constexpr int BN = 256;
  static constexpr int kStages = 5;
  static constexpr int kA = BM * BK * 2;            // 16 KB: own 128 i x 64 k (2 MN-major boxes)
  static constexpr int kB = (BN / 2) * BK * 2;      // 16 KB: own 128 j x 64 k
  static constexpr int kStg = 32 * 128;
  static constexpr int kOffB = kStages * kA;
  static constexpr int kOffOnes = kOffB + kStages * kB;           // 1 KB: 8 n rows x 64 k, K-major SW128
  static constexpr int kOffStg = kOffOnes + 1024;
  static constexpr int kOffBar = kOffStg + kEpiWarps * kStg;
  static constexpr int kOffSeg = kOffBar + 256;
  static constexpr int kBytes = kOffSeg + 258 * 4 + 1024;
  static_assert(kBytes <= 232448, "pair ragged-K smem");
};

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    grouped_gemm_pair_k_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                               const __grid_constant__ CUtensorMap tmC, const GemmArgs args) {
  pdl_wait();
  using S = PairKSmem;
  constexpr int BN = S::BN;
  constexpr int kStages = S::kStages;
  constexpr int CPC = 32;                            // fp32 output: 32 columns per 128-byte row chunk
  constexpr int NCH = BN / CPC;
  constexpr int MYCH = NCH / 2;
  constexpr uint16_t kPair = 0x3;
  extern __shared__ __align__(16) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sA = smem;
  uint8_t* sB = smem + S::kOffB;
  uint8_t* sOnes = smem + S::kOffOnes;
  uint8_t* sStg = smem + S::kOffStg;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + S::kOffBar);
  uint64_t* empty = full + kStages;
  uint64_t* tfull = empty + kStages;
  uint64_t* tempty = tfull + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 1);
  int* seg_s = reinterpret_cast<int*>(smem + S::kOffSeg);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const bool fused_bias = args.db_out != nullptr;
  for (int i = threadIdx.x; i <= args.G; i += blockDim.x) seg_s[i] = args.seg[i];
  {  // ones operand: K-major, 8 n rows of 64 k (one SW128 atom); n = 0 of the leader's half is 1.0
    uint32_t* o32 = reinterpret_cast<uint32_t*>(sOnes);
    const uint32_t one2 = rank == 0 ? 0x3F803F80u : 0u;            // two bf16 1.0
    for (int i = threadIdx.x; i < 256; i += blockDim.x) o32[i] = (i < 32) ? one2 : 0u;   // row 0 = 128 B
    fence_proxy_async_smem();
  }
  if (warp == 0 && lane == 0) { tma_prefetch(&tmA); tma_prefetch(&tmB); tma_prefetch(&tmC); }
  if (warp == 1 && lane == 0) {
    for (int s = 0; s < kStages; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    mbar_init(tfull, 1);
    mbar_init(tempty, 2 * kEpiWarps);
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc_2sm(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int i_tiles = (args.I + BM - 1) / BM;
  const int i_pairs = (i_tiles + 1) / 2;
  const int j_tiles = (args.N + BN - 1) / BN;
  const int per_g = i_pairs * j_tiles;
  const int num_units = args.G * per_g;
  const int cl = blockIdx.x >> 1, ncl = gridDim.x >> 1;
  auto decode = [&](int u, int& g, int& i0, int& ni, int& j0, int& kb0, int& nkb) {
    g = u / per_g;
    const int r = u - g * per_g;
    const int ip = r / j_tiles;
    j0 = (r - ip * j_tiles) * BN;
    i0 = ip * 2 * BM;
    ni = min(2, i_tiles - 2 * ip);
    kb0 = seg_s[g] / BK;
    nkb = (seg_s[g + 1] - seg_s[g]) / BK;
  };

  if (warp == 0) {
    if (lane == 0) {
      // ================= TMA producer (both CTAs)
      int stage = 0;
      uint32_t phase = 0;
      for (int u = cl; u < num_units; u += ncl) {
        int g, i0, ni, j0, kb0, nkb;
        decode(u, g, i0, ni, j0, kb0, nkb);
        const bool valid = (int)rank < ni;
        const int ia = i0 + (int)rank * BM;
        const int jb = j0 + (int)rank * (BN / 2);
        for (int kb = 0; kb < nkb; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          if (rank == 0) mbar_expect_tx(&full[stage], ni * S::kA + 2 * S::kB);
          uint8_t* a = sA + stage * S::kA;
          uint8_t* b = sB + stage * S::kB;
          const int k0 = (kb0 + kb) * BK;
          if (valid) {
#pragma unroll
            for (int j = 0; j < 2; ++j) tma_load_2d_2sm(a + j * 8192, &tmA, &full[stage], ia + 64 * j, k0);
          }
#pragma unroll
          for (int j = 0; j < 2; ++j) tma_load_2d_2sm(b + j * 8192, &tmB, &full[stage], jb + 64 * j, k0);
          if (++stage == kStages) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && rank == 0) {
      // ================= MMA issuer (leader)
      constexpr uint32_t idesc = umma_idesc_bf16(2 * BM, BN, 1, 1);
      constexpr uint32_t idesc_bias = umma_idesc_bf16(2 * BM, 16, 1, 0);
      const uint32_t ones_addr = smem_u32(sOnes);
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int u = cl; u < num_units; u += ncl, ++it) {
        int g, i0, ni, j0, kb0, nkb;
        decode(u, g, i0, ni, j0, kb0, nkb);
        mbar_wait(tempty, (it & 1) ^ 1);
        tc_fence_after();
        const bool with_bias = fused_bias && j0 == 0;
        for (int kb = 0; kb < nkb; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t a_addr = smem_u32(sA + stage * S::kA);
          const uint32_t b_addr = smem_u32(sB + stage * S::kB);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            const uint64_t ad = umma_desc_sw128(a_addr + k * 2048, 8192, 1024);
            tc_mma_f16_2sm(tmem_base, ad, umma_desc_sw128(b_addr + k * 2048, 8192, 1024), idesc, (kb | k) != 0);
            if (with_bias)
              tc_mma_f16_2sm(tmem_base + BN, ad, umma_desc_sw128(ones_addr + k * 32, 16, 1024), idesc_bias,
                             (kb | k) != 0);
          }
          tc_commit_2sm_mc(&empty[stage], kPair);
          if (++stage == kStages) { stage = 0; phase ^= 1; }
        }
        tc_commit_2sm_mc(tfull, kPair);     // (also fires for an empty group: the epilogue writes zeros)
      }
    }
  } else if (warp >= 4) {
    // ================= epilogue (both CTAs): own 128 i rows of C_g (fp32)
    const int q = warp & 3;
    const int par = (warp - 4) >> 2;
    uint8_t* stg = sStg + (warp - 4) * S::kStg;
    const uint32_t lead_tempty = mapa_shared(smem_u32(tempty), 0);
    int it = 0;
    for (int u = cl; u < num_units; u += ncl, ++it) {
      int g, i0, ni, j0, kb0, nkb;
      decode(u, g, i0, ni, j0, kb0, nkb);
      const bool valid = (int)rank < ni;
      const int ia = i0 + (int)rank * BM;
      const int row = ia + 32 * q + lane;       // output row i
      mbar_wait(tfull, it & 1);
      tc_fence_after();
      const uint32_t tbase = tmem_base + ((uint32_t)(32 * q) << 16);
      if (fused_bias && j0 == 0 && par == 0) {
        uint32_t t0[32];
        tmem_ld32(tbase + BN, t0);
        tmem_ld_wait();
        if (valid && row < args.I) args.db_out[(size_t)g * args.I + row] = nkb > 0 ? __uint_as_float(t0[0]) : 0.f;
      }
#pragma unroll
      for (int i = 0; i < MYCH; ++i) {
        const int cc = par + 2 * i;
        const int n = j0 + cc * CPC;
        if (n >= args.N) break;
        uint32_t t[32];
        tmem_ld32(tbase + cc * CPC, t);
        tmem_ld_wait();
        if (!valid) continue;
        if (lane == 0) bulk_wait_read<0>();
        __syncwarp();
        uint4* rowp = reinterpret_cast<uint4*>(stg + lane * 128);
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const uint4 pk = nkb > 0 ? make_uint4(t[4 * c], t[4 * c + 1], t[4 * c + 2], t[4 * c + 3]) : make_uint4(0, 0, 0, 0);
          rowp[c ^ (lane & 7)] = pk;
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          tma_store_3d(&tmC, stg, n, ia + 32 * q, g);
          bulk_commit();
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(lead_tempty);
    }
    if (lane == 0) bulk_wait<0>();
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  if (warp == 2) tmem_dealloc_2sm(tmem_base, 512);
}

// split-K partials of the ragged-K GEMM -> C (and db), summed over the splits in order
__global__ void __launch_bounds__(256) ksplit_reduce_kernel(int S, long n_c, long n_db, const float* __restrict__ part_c,
                                                            const float* __restrict__ part_db, float* __restrict__ C,
                                                            float* __restrict__ db) {
  pdl_wait();
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n_c + n_db; i += (long)gridDim.x * blockDim.x) {
    float v = 0.f;
    if (i < n_c) {
      for (int s = 0; s < S; ++s) v += part_c[(long)s * n_c + i];
      C[i] = v;
    } else {
      const long k = i - n_c;
      for (int s = 0; s < S; ++s) v += part_db[(long)s * n_db + k];
      db[k] = v;
    }
  }
}

// ---------------------------------------------------------------- host side

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn get_encode() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

// rank-2/3 tensor map; dims innermost first; strides (bytes) for dims 1..rank-1
static int make_map(CUtensorMap* m, CUtensorMapDataType dt, int rank, const void* ptr, const uint64_t* dims,
                    const uint64_t* strides_bytes, const uint32_t* box) {
  EncodeTiledFn enc = get_encode();
  if (!enc) return set_error(SMES_ERR_CUDA, "cuTensorMapEncodeTiled unavailable (no CUDA driver?)");
  cuuint64_t d[3], s[2];
  cuuint32_t b[3], e[3] = {1, 1, 1};
  for (int i = 0; i < rank; ++i) { d[i] = dims[i]; b[i] = box[i]; }
  for (int i = 0; i < rank - 1; ++i) s[i] = strides_bytes[i];
  CUresult r = enc(m, dt, rank, const_cast<void*>(ptr), d, s, b, e, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return set_error(SMES_ERR_CUDA, "cuTensorMapEncodeTiled failed (code %d)", (int)r);
  return SMES_OK;
}

static int g_num_sms = 0;
static int num_sms() {
  if (!g_num_sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
    if (g_num_sms <= 0) g_num_sms = 148;
  }
  return g_num_sms;
}

template <int BN, int MODE, bool B_MN, bool F32>
static int launch(const CUtensorMap& a, const CUtensorMap& b, const CUtensorMap& c, const GemmArgs& args,
                  cudaStream_t st) {
  auto kern = grouped_gemm_kernel<BN, MODE, B_MN, F32>;
  using SM = Smem<BN, MODE>;
  static bool attr = false;
  if (!attr) {
    cudaError_t ea = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SM::kBytes);
    if (ea != cudaSuccess)
      return set_error(SMES_ERR_CUDA, "grouped_gemm smem attribute (%d B): %s", SM::kBytes, cudaGetErrorString(ea));
    attr = true;
  }
  smes_launch(kern, num_sms(), kThreads, SM::kBytes, st, a, b, c, args);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_error(SMES_ERR_CUDA, "grouped_gemm launch: %s", cudaGetErrorString(e));
  return SMES_OK;
}

template <bool B_MN, bool F32>
static int launch_pair(const CUtensorMap& a, const CUtensorMap& b, const CUtensorMap& c, const GemmArgs& args,
                       cudaStream_t st) {
  auto kern = grouped_gemm_pair_kernel<B_MN, F32>;
  using SM = PairSmem<B_MN, F32>;
  static bool attr = false;
  if (!attr) {
    cudaError_t ea = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SM::kBytes);
    if (ea != cudaSuccess)
      return set_error(SMES_ERR_CUDA, "grouped_gemm_pair smem attribute (%d B): %s", SM::kBytes, cudaGetErrorString(ea));
    attr = true;
  }
  smes_launch(kern, num_sms() / 2 * 2, kThreads, SM::kBytes, st, a, b, c, args);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_error(SMES_ERR_CUDA, "grouped_gemm_pair launch: %s", cudaGetErrorString(e));
  return SMES_OK;
}

static bool pair_enabled() {
  static const int on = [] {
    const char* v = std::getenv("SMES_GEMM_PAIR");
    return (v == nullptr || v[0] != '0') ? 1 : 0;
  }();
  return on != 0;
}

template <int BN>
static int launch_m(bool b_mn, bool f32, const CUtensorMap& a, const CUtensorMap& b, const CUtensorMap& c,
                    const GemmArgs& args, cudaStream_t st) {
  if (b_mn) return f32 ? launch<BN, MODE_RAGGED_M, true, true>(a, b, c, args, st)
                       : launch<BN, MODE_RAGGED_M, true, false>(a, b, c, args, st);
  return f32 ? launch<BN, MODE_RAGGED_M, false, true>(a, b, c, args, st)
             : launch<BN, MODE_RAGGED_M, false, false>(a, b, c, args, st);
}

}  // namespace smes

using namespace smes;

extern "C" {

int smes_gemm_ragged_m(const void* A, long lda, long rows_cap, const void* W, int G, int N, int K, int b_mn,
                       const int* seg, const float* bias, int act, uint32_t* bits_out, const uint32_t* bits_in,
                       long bits_ld, void* C, long ldc, int out_fp32, long m_limit, void* stream) {
  if (G < 1 || G > 256) return set_error(SMES_ERR_SHAPE, "group count %d outside [1, 256]", G);
  if (N <= 0 || K <= 0 || rows_cap <= 0) return set_error(SMES_ERR_SHAPE, "empty GEMM N=%d K=%d", N, K);
  if ((lda * 2) % 16 || (ldc * (out_fp32 ? 4 : 2)) % 16 || (K * 2) % 16)
    return set_error(SMES_ERR_SHAPE, "GEMM strides must be 16-byte aligned (lda=%ld ldc=%ld K=%d N=%d)", lda, ldc,
                     K, N);
  if ((bits_out || bits_in) && (N % 32))
    return set_error(SMES_ERR_SHAPE, "relu bitmask needs N %% 32 == 0 (N=%d)", N);
  // N <= 32 with fp32 out (head projections, K = T outputs): a narrow BN = 32 tile
  const bool narrow = N <= 32 && out_fp32 && !b_mn;
  CUtensorMap ta, tb, tc;
  int rc;
  {
    uint64_t dims[2] = {(uint64_t)K, (uint64_t)rows_cap}, str[1] = {(uint64_t)lda * 2};
    uint32_t box[2] = {64, 128};
    if ((rc = make_map(&ta, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, A, dims, str, box))) return rc;
  }
  if (!b_mn) {  // W (G, N, K) K-major
    uint64_t dims[3] = {(uint64_t)K, (uint64_t)N, (uint64_t)G};
    uint64_t str[2] = {(uint64_t)K * 2, (uint64_t)N * K * 2};
    uint32_t box[3] = {64, (uint32_t)(narrow ? 32 : N >= 256 ? 256 : 128), 1};
    if ((rc = make_map(&tb, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, W, dims, str, box))) return rc;
  } else {      // W (G, K, N): element (n, k) at W[g][k][n]
    uint64_t dims[3] = {(uint64_t)N, (uint64_t)K, (uint64_t)G};
    uint64_t str[2] = {(uint64_t)N * 2, (uint64_t)N * K * 2};
    uint32_t box[3] = {64, 64, 1};
    if ((rc = make_map(&tb, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, W, dims, str, box))) return rc;
  }
  {
    uint64_t dims[2] = {(uint64_t)N, (uint64_t)m_limit}, str[1] = {(uint64_t)ldc * (out_fp32 ? 4 : 2)};
    uint32_t box[2] = {(uint32_t)(out_fp32 ? 32 : 64), 32};
    if ((rc = make_map(&tc, out_fp32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, C, dims,
                       str, box)))
      return rc;
  }
  GemmArgs args{seg, G, N, K, 0, bias, act, bits_out, bits_in, (int)bits_ld, nullptr, 0, 0};
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (narrow) return launch<32, MODE_RAGGED_M, false, true>(ta, tb, tc, args, st);
  // CTA pairs for the large banks (N a multiple of 256, many rows): half the B stream per CTA
  if (pair_enabled() && N % 256 == 0 && K >= 256 && rows_cap >= 64L * 1024) {
    CUtensorMap tb2;
    if (!b_mn) {  // W (G, N, K) K-major, box {64 k, 128 n, 1}: each CTA its half of the 256-wide tile
      uint64_t dims[3] = {(uint64_t)K, (uint64_t)N, (uint64_t)G};
      uint64_t str[2] = {(uint64_t)K * 2, (uint64_t)N * K * 2};
      uint32_t box[3] = {64, 128, 1};
      if ((rc = make_map(&tb2, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, W, dims, str, box))) return rc;
    } else {
      tb2 = tb;    // MN-major boxes are {64 n, 64 k, 1} already
    }
    if (b_mn) return out_fp32 ? launch_pair<true, true>(ta, tb2, tc, args, st) : launch_pair<true, false>(ta, tb2, tc, args, st);
    return out_fp32 ? launch_pair<false, true>(ta, tb2, tc, args, st) : launch_pair<false, false>(ta, tb2, tc, args, st);
  }
  // K-major B box is {64, 256} for N >= 256: requires BN == 256
  if (N >= 256) return launch_m<256>(b_mn, out_fp32, ta, tb, tc, args, st);
  return launch_m<128>(b_mn, out_fp32, ta, tb, tc, args, st);
}

int smes_gemm_ragged_m_x3(const void* A3, long lda, long rows_cap, const void* W3, int G, int N, int K,
                          const int* seg, const float* bias, int act, float* C, long ldc, long m_limit, void* stream) {
  if (G < 1 || G > 256) return set_error(SMES_ERR_SHAPE, "group count %d outside [1, 256]", G);
  if (N <= 0 || K <= 0 || rows_cap <= 0) return set_error(SMES_ERR_SHAPE, "empty GEMM N=%d K=%d", N, K);
  if (K % BK) return set_error(SMES_ERR_SHAPE, "fp32 (bf16x3) GEMM needs K %% 64 == 0 (K=%d)", K);
  if ((lda * 2) % 16 || (ldc * 4) % 16 || lda < 3L * K)
    return set_error(SMES_ERR_SHAPE, "fp32 GEMM: A stride %ld must hold 3 planes of K=%d, 16-byte aligned", lda, K);
  const bool narrow = N <= 32;
  CUtensorMap ta, tb, tc;
  int rc;
  {
    uint64_t dims[2] = {(uint64_t)3 * K, (uint64_t)rows_cap}, str[1] = {(uint64_t)lda * 2};
    uint32_t box[2] = {64, 128};
    if ((rc = make_map(&ta, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, A3, dims, str, box))) return rc;
  }
  {  // W3 (G, N, 3K): planes along K
    uint64_t dims[3] = {(uint64_t)3 * K, (uint64_t)N, (uint64_t)G};
    uint64_t str[2] = {(uint64_t)3 * K * 2, (uint64_t)N * 3 * K * 2};
    uint32_t box[3] = {64, (uint32_t)(narrow ? 32 : N >= 256 ? 256 : 128), 1};
    if ((rc = make_map(&tb, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, W3, dims, str, box))) return rc;
  }
  {
    uint64_t dims[2] = {(uint64_t)N, (uint64_t)m_limit}, str[1] = {(uint64_t)ldc * 4};
    uint32_t box[2] = {32, 32};
    if ((rc = make_map(&tc, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, C, dims, str, box))) return rc;
  }
  GemmArgs args{seg, G, N, 6 * K, 0, bias, act, nullptr, nullptr, 0, nullptr, 0, K};
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (narrow) return launch<32, MODE_RAGGED_M, false, true>(ta, tb, tc, args, st);
  if (N >= 256) return launch<256, MODE_RAGGED_M, false, true>(ta, tb, tc, args, st);
  return launch<128, MODE_RAGGED_M, false, true>(ta, tb, tc, args, st);
}

static int ragged_k_impl(const void* P, long ldp, long p_rows, const void* Q, long ldq, long rows_cap, int G, int I,
                         int J, const int* seg, float* C, float* db_out, int a_period, const int* gather, long n_src,
                         void* stream) {
  if (G < 1 || G > 256) return set_error(SMES_ERR_SHAPE, "group count %d outside [1, 256]", G);
  if (I <= 0 || J <= 0) return set_error(SMES_ERR_SHAPE, "empty wgrad I=%d J=%d", I, J);
  if ((ldp * 2) % 16 || (ldq * 2) % 16 || (J * 4) % 16)
    return set_error(SMES_ERR_SHAPE, "wgrad strides must be 16-byte aligned");
  CUtensorMap ta, tb, tc;
  int rc;
  {
    if (a_period < 0 || a_period % BK) return set_error(SMES_ERR_SHAPE, "wgrad: P period %d must be a multiple of 64", a_period);
    uint64_t dims[2] = {(uint64_t)I, (uint64_t)(a_period ? p_rows : rows_cap)}, str[1] = {(uint64_t)ldp * 2};
    uint32_t box[2] = {64, 64};
    if ((rc = make_map(&ta, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, P, dims, str, box))) return rc;
  }
  {
    // gathered: Q is the source ((n_src, ldq) rows), one row per box (4 per gather4 op)
    uint64_t dims[2] = {(uint64_t)J, (uint64_t)(gather ? n_src : rows_cap)}, str[1] = {(uint64_t)ldq * 2};
    uint32_t box[2] = {64, gather ? 1u : 64u};
    if ((rc = make_map(&tb, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, Q, dims, str, box))) return rc;
  }
  {
    uint64_t dims[3] = {(uint64_t)J, (uint64_t)I, (uint64_t)G};
    uint64_t str[2] = {(uint64_t)J * 4, (uint64_t)I * J * 4};
    uint32_t box[3] = {32, 32, 1};
    if ((rc = make_map(&tc, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, C, dims, str, box))) return rc;
  }
  GemmArgs args{seg, G, J, 0, I, nullptr, 0, nullptr, nullptr, 0, db_out, a_period, 0, 0, gather};
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  // CTA pairs for the large wgrad banks (I spans >= 2 i tiles, J >= 256, many rows)
  // measured neutral at c3 under the power cap (fc1 wgrad 1.84 / 1.83 ms paired vs 1.89 / 1.79 ms,
  // tools/ab_pairk.sh): off unless SMES_GEMM_PAIR_K=1
  const char* pk_env = std::getenv("SMES_GEMM_PAIR_K");
  const bool pair_k = pk_env != nullptr && pk_env[0] == '1';
  if (pair_enabled() && pair_k && gather == nullptr && a_period == 0 && I >= 2 * BM && J >= 256 &&
      rows_cap >= 64L * 1024) {
    auto kern = grouped_gemm_pair_k_kernel;
    static bool attr = false;
    if (!attr) {
      cudaError_t ea = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, PairKSmem::kBytes);
      if (ea != cudaSuccess) return set_error(SMES_ERR_CUDA, "pair ragged-K smem attribute: %s", cudaGetErrorString(ea));
      attr = true;
    }
    smes_launch(kern, num_sms() / 2 * 2, kThreads, PairKSmem::kBytes, st, ta, tb, tc, args);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return set_error(SMES_ERR_CUDA, "pair ragged-K launch: %s", cudaGetErrorString(e));
    return SMES_OK;
  }
  if (J <= 16) return launch<16, MODE_RAGGED_K, true, true>(ta, tb, tc, args, st);
  // BN = 256 halves the tile count; with a single i-tile (I <= 128: the folded-head wgrad) keep
  // it only while the grid still covers every SM
  const int tiles256 = G * ((I + BM - 1) / BM) * ((J + 255) / 256);
  if (J >= 256 && (I > BM || tiles256 >= num_sms())) return launch<256, MODE_RAGGED_K, true, true>(ta, tb, tc, args, st);
  return launch<128, MODE_RAGGED_K, true, true>(ta, tb, tc, args, st);
}

int smes_gemm_ragged_k_periodic(const void* P, long ldp, long p_rows, const void* Q, long ldq, long rows_cap, int G,
                                int I, int J, const int* seg, float* C, float* db_out, int a_period, void* stream) {
  return ragged_k_impl(P, ldp, p_rows, Q, ldq, rows_cap, G, I, J, seg, C, db_out, a_period, nullptr, 0, stream);
}

int smes_gemm_ragged_k_gather(const void* P, long ldp, const void* src, long ld_src, long n_src, const int32_t* gather,
                              long rows_cap, int G, int I, int J, const int* seg, float* C, float* db_out,
                              void* stream) {
  if (gather == nullptr || n_src < 1) return set_error(SMES_ERR_SHAPE, "ragged_k_gather: empty source");
  if (reinterpret_cast<uintptr_t>(gather) % 16) return set_error(SMES_ERR_SHAPE, "ragged_k_gather: row table must be 16-byte aligned");
  return ragged_k_impl(P, ldp, rows_cap, src, ld_src, rows_cap, G, I, J, seg, C, db_out, 0, gather, n_src, stream);
}

long smes_gemm_ragged_k_split_work(int G, int I, int J, int splits, int with_db) {
  return (long)splits * G * I * J + (with_db ? (long)splits * G * I : 0);
}

int smes_gemm_ragged_k_split(const void* P, long ldp, const void* Q, long ldq, long rows_cap, int G, int I, int J,
                             const int* seg, float* C, float* db_out, int splits, float* work, void* stream) {
  if (splits <= 1) return smes_gemm_ragged_k_periodic(P, ldp, rows_cap, Q, ldq, rows_cap, G, I, J, seg, C, db_out, 0,
                                                      stream);
  if (G < 1 || G * splits > 65535) return set_error(SMES_ERR_SHAPE, "wgrad split: %d groups x %d splits", G, splits);
  if (I <= 0 || J <= 0) return set_error(SMES_ERR_SHAPE, "empty wgrad I=%d J=%d", I, J);
  if ((ldp * 2) % 16 || (ldq * 2) % 16 || (J * 4) % 16) return set_error(SMES_ERR_SHAPE, "wgrad strides must be 16-byte aligned");
  if (work == nullptr) return set_error(SMES_ERR_STATE, "wgrad split: work buffer required");
  CUtensorMap ta, tb, tc;
  int rc;
  {
    uint64_t dims[2] = {(uint64_t)I, (uint64_t)rows_cap}, str[1] = {(uint64_t)ldp * 2};
    uint32_t box[2] = {64, 64};
    if ((rc = make_map(&ta, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, P, dims, str, box))) return rc;
  }
  {
    uint64_t dims[2] = {(uint64_t)J, (uint64_t)rows_cap}, str[1] = {(uint64_t)ldq * 2};
    uint32_t box[2] = {64, 64};
    if ((rc = make_map(&tb, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, Q, dims, str, box))) return rc;
  }
  {  // partials [splits][G][I][J] in the work buffer
    uint64_t dims[3] = {(uint64_t)J, (uint64_t)I, (uint64_t)G * splits};
    uint64_t str[2] = {(uint64_t)J * 4, (uint64_t)I * J * 4};
    uint32_t box[3] = {32, 32, 1};
    if ((rc = make_map(&tc, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, work, dims, str, box))) return rc;
  }
  const long n_c = (long)G * I * J, n_db = db_out ? (long)G * I : 0;
  float* part_db = db_out ? work + (long)splits * n_c : nullptr;
  GemmArgs args{seg, G, J, 0, I, nullptr, 0, nullptr, nullptr, 0, part_db, 0, 0, splits};
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (J <= 16) rc = launch<16, MODE_RAGGED_K, true, true>(ta, tb, tc, args, st);
  else if (J >= 256) rc = launch<256, MODE_RAGGED_K, true, true>(ta, tb, tc, args, st);
  else rc = launch<128, MODE_RAGGED_K, true, true>(ta, tb, tc, args, st);
  if (rc) return rc;
  const long n = n_c + n_db;
  const long want = (n + 255) / 256;
  smes_launch(ksplit_reduce_kernel, (int)(want < 148L * 8 ? want : 148L * 8), 256, 0, st, splits, n_c, n_db, work,
              part_db, C, db_out);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_error(SMES_ERR_CUDA, "wgrad split reduce: %s", cudaGetErrorString(e));
  return SMES_OK;
}

int smes_gemm_ragged_k(const void* P, long ldp, const void* Q, long ldq, long rows_cap, int G, int I, int J,
                       const int* seg, float* C, float* db_out, void* stream) {
  return smes_gemm_ragged_k_periodic(P, ldp, rows_cap, Q, ldq, rows_cap, G, I, J, seg, C, db_out, 0, stream);
}

}  // extern "C"
