// Fused expert-MLP kernels for the training step (BASELINE expert MLP d -> d_ff -> d_out with
// ReLU after fc1 and the identity last pool folded into the task heads, csrc/fold.cu).
//
// Both kernels chain two tcgen05 MMAs per 128-row tile through shared memory: the epilogue
// warps turn the first accumulator (TMEM) into the bf16 A operand of the second MMA, chunk by
// chunk (128 columns of d_ff), so the d_ff-wide intermediate never makes a round trip to HBM
// between the two products.
//
//   mlp_fwd   (fc1 + folded fc2/heads, execution.py:126-158 twice + model.py:202-208):
//       S_c = X W1[c]^T            (K = d, TMA-fed, N = 128)
//       H_c = relu(S_c + b1[c])    -> relu bit-mask, H (kept for the weight gradients), smem
//       P  += H_c G[c]^T           (K = 128, N = 16: the head projections, fp32)
//   mlp_dgrad (training.py:180-192 for the two pools):
//       S_c = C G[c]               (K = T: the rank-T d_packed through the folded heads)
//       dH_c = S_c * mask[c]       -> smem
//       dX += dH_c W1[c]           (K = 128, N = d)
//
// Rows are the padded expert-major packed rows of the execution plan (128-row aligned
// segments, so a tile never straddles two experts); group offsets stay on the device.
//
// Warp roles (384 threads, 1 CTA/SM): w0 TMA producer, w1 MMA issuer (fwd: S only), w2 TMEM
// allocator, w3 (fwd) P-MMA issuer, w4..w11 epilogue (warp w owns TMEM lanes 32*(w%4).. and the 64-column half (w-4)/4 of a chunk).
#include <algorithm>

#include "ptx.cuh"
#include "smes_capi.h"

namespace smes {
namespace mlp {

constexpr int BM = 128;          // rows per tile
constexpr int CH = 128;          // d_ff columns per chunk
constexpr int kThreads = 384;
constexpr int kEpiWarps = 8;
#ifndef SMES_FWD_XS         // ring depths of mlp_fwd (X / W1 k-block slots); 0 = the defaults below
#define SMES_FWD_XS 0
#endif
#ifndef SMES_FWD_WS
#define SMES_FWD_WS 0
#endif
#ifdef SMES_TRACE
// experiment builds only: per-CTA cycles spent in each barrier wait (tools/trace_mlp.py)
__device__ unsigned long long g_trace[148 * 16];
#define TW(k, stmt)                                                      \
  do {                                                                   \
    const long long _t0 = clock64();                                     \
    stmt;                                                                \
    if ((threadIdx.x & 31) == 0) atomicAdd(&g_trace[blockIdx.x * 16 + (k)], (unsigned long long)(clock64() - _t0)); \
  } while (0)
__device__ long long g_ev[4 * 12 * 64];
__device__ __forceinline__ long long gtimer() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define EV(r, i)                                                                       \
  do {                                                                                 \
    if (blockIdx.x < 4 && (i) < 64) g_ev[(blockIdx.x * 12 + (r)) * 64 + (i)] = clock64(); \
  } while (0)
#else
#define TW(k, stmt) stmt
#define EV(r, i)
#endif

struct FwdArgs {
  const int* seg;                // (E+1) padded segment offsets
  int E, d, d_ff, ldp;
  const float* b1;               // (E, d_ff)
  const float* c;                // (E, ldg) folded head bias
  int ldg;
  uint32_t* bits;                // [(d_ff/32)][bits_ld] relu bit-mask of H
  int bits_ld;
  float* P;                      // (rows, ldp) fp32 head projections
  int store_h;                   // write H through tmH
  const int* gather;             // non-null: X row r is source row gather[r] (tmX maps the source,
                                 // box {64, 1}); -1 (pad rows) reads zeros
  const __nv_bfloat16* src;      // pack mode (PACK): warp 2 copies the X rows from
  long ld_src;                   // src[gather[r]] (LDGSTS) and stores the packed tile through tmX
};

struct DgradArgs {
  const int* seg;
  int E, d, d_ff;
  const uint32_t* bits;          // relu mask of H
  int bits_ld;
  int store_dh;                  // also write dH through tmDH (for the separate fc1 weight-gradient GEMM)
};

__device__ __forceinline__ int find_group(const int* seg_s, int G, int row) {
  int lo = 0, hi = G - 1;
  while (lo < hi) {
    int mid = (lo + hi + 1) >> 1;
    if (seg_s[mid] <= row) lo = mid; else hi = mid - 1;
  }
  return lo;
}

// Ring-buffer bookkeeping: slot and parity of the i-th use of an n-slot ring.
__device__ __forceinline__ int slot_of(int i, int n) { return i % n; }
__device__ __forceinline__ uint32_t par_of(int i, int n) { return (uint32_t)((i / n) & 1); }

// Named barrier for the epilogue warps only (id 1, 256 threads).
__device__ __forceinline__ void epi_sync() { asm volatile("bar.sync 1, 256;" ::: "memory"); }

// 32 lanes x 16 columns TMEM load
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}

// ============================================================================ forward
// S accumulators (128 TMEM columns each): three, so the S-MMA of chunk c+2 does not wait for the
// epilogue to drain chunk c (a double buffer left a ~380-cycle bubble per chunk, tools/mma_probe)
constexpr int kSB = 3;
// lanes of warp 0 issuing the gathered X rows (TMA gather4) in mlp_fwd
#ifndef SMES_GATHER_LANES
#define SMES_GATHER_LANES 8
#endif
constexpr int kGatherLanes = SMES_GATHER_LANES;
// H staging tiles in shared memory (the P-MMA operand and the TMA-store source).  Two tiles (the
// epilogue writing chunk c + 1 while the P-MMA / store of chunk c read theirs, W1 ring 6 -> 4)
// measured 123 us against 120 us for one at c2, so one it is (SMES_FWD_HB=2 builds the other)
#ifndef SMES_FWD_HB
#define SMES_FWD_HB 1
#endif
constexpr int kHBMax = SMES_FWD_HB;
template <int DK>     // d / 64
struct FwdSmem {
  // X k-block ring (16 KB slots, spare slots prefetch the next tile), W1 k-block ring (16 KB:
  // 128 n x 64 k, 1.5 chunks deep at d = 256), G chunk ring (4 KB: 2 x {64 f, 16 t})
  static constexpr int kXS = SMES_FWD_XS > 0 ? SMES_FWD_XS : DK <= 2 ? DK + 2 : DK <= 4 ? DK + 1 : DK;
  static constexpr int kHB = DK <= 4 ? kHBMax : 1;       // d = 512: the X ring takes the space
  static constexpr int kWS = SMES_FWD_WS > 0 ? SMES_FWD_WS : DK <= 4 ? (kHB == 2 ? 4 : 6) : 3;
  static constexpr int kGS = 2;
  static constexpr int kOffX = 0;
  static constexpr int kOffW = kOffX + kXS * 16384;
  static constexpr int kOffG = kOffW + kWS * 16384;
  static constexpr int kOffH = kOffG + kGS * 4096;      // kHB x (2 x 16 KB atoms: 128 rows x 64 cols)
  static constexpr int kOffBias = kOffH + kHB * 32768;  // 64 fp32 per epilogue warp
  static constexpr int kOffIdx = kOffBias + kEpiWarps * 256;   // gathered X: 2 x 128 source-row indices
  static constexpr int kOffBar = kOffIdx + 2 * BM * 4;
  static constexpr int kOffSeg = kOffBar + 512;
  static constexpr int kBytes = kOffSeg + 257 * 4 + 1024;
  static_assert(kBytes <= 232448, "mlp_fwd smem");
};

template <int DK, bool PACK>
__global__ void __launch_bounds__(kThreads, 1)
    mlp_fwd_kernel(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmW1,
                   const __grid_constant__ CUtensorMap tmG, const __grid_constant__ CUtensorMap tmH,
                   const FwdArgs a) {
  pdl_wait();
  using S = FwdSmem<DK>;
  extern __shared__ __align__(16) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);   // stays in the shared window
  uint8_t* sX = smem + S::kOffX;
  uint8_t* sW = smem + S::kOffW;
  uint8_t* sG = smem + S::kOffG;
  uint8_t* sH = smem + S::kOffH;
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + S::kOffBar);
  uint64_t* xfull = bar;                    // [kXS]
  uint64_t* xempty = xfull + S::kXS;        // [kXS]
  uint64_t* wfull = xempty + S::kXS;        // [kWS]
  uint64_t* wempty = wfull + S::kWS;        // [kWS]
  uint64_t* gfull = wempty + S::kWS;        // [kGS]
  uint64_t* gempty = gfull + S::kGS;        // [kGS]
  uint64_t* sfull = gempty + S::kGS;        // [kSB]
  uint64_t* sempty = sfull + kSB;           // [kSB]
  uint64_t* hfull = sempty + kSB;           // [S::kHB]
  uint64_t* hempty = hfull + S::kHB;           // [S::kHB]
  uint64_t* pfull = hempty + S::kHB;           // [2]
  uint64_t* pempty = pfull + 2;             // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(pempty + 2);
  int* seg_s = reinterpret_cast<int*>(smem + S::kOffSeg);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int NC = a.d_ff / CH;
  for (int i = threadIdx.x; i <= a.E; i += blockDim.x) seg_s[i] = a.seg[i];
  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmX); tma_prefetch(&tmW1); tma_prefetch(&tmG); tma_prefetch(&tmH);
  }
  if (warp == 1 && lane == 0) {
    for (int i = 0; i < S::kXS; ++i) { mbar_init(&xfull[i], 1); mbar_init(&xempty[i], 1); }
    for (int i = 0; i < S::kWS; ++i) { mbar_init(&wfull[i], 1); mbar_init(&wempty[i], 1); }
    for (int i = 0; i < S::kGS; ++i) { mbar_init(&gfull[i], 1); mbar_init(&gempty[i], 1); }
    for (int i = 0; i < kSB; ++i) { mbar_init(&sfull[i], 1); mbar_init(&sempty[i], kEpiWarps); }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&pfull[i], 1); mbar_init(&pempty[i], kEpiWarps / 2);
    }
    for (int i = 0; i < S::kHB; ++i) { mbar_init(&hfull[i], kEpiWarps); mbar_init(&hempty[i], 1); }
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int num_tiles = seg_s[a.E] / BM;
#ifdef SMES_TRACE
  const long long t_start = clock64();
  if (threadIdx.x == 0) g_trace[blockIdx.x * 16 + 10] = gtimer();
#endif

  // G producer: released by the P-MMA, kept off the W1 stream (warp 2 lane 0; warp 0 lane 1 when
  // warp 2 copies X rows)
  auto produce_g = [&]() {
    int gi = 0;
    for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
      const int e = find_group(seg_s, a.E, tile * BM);
      for (int c = 0; c < NC; ++c, ++gi) {
        const int s = slot_of(gi, S::kGS);
        TW(2, mbar_wait(&gempty[s], par_of(gi, S::kGS) ^ 1));
        mbar_expect_tx(&gfull[s], 4096);
        tma_load_3d(sG + s * 4096, &tmG, &gfull[s], c * CH, 0, e);          // box {64 f, 16 t, 1}
        tma_load_3d(sG + s * 4096 + 2048, &tmG, &gfull[s], c * CH + 64, 0, e);
      }
    }
  };
  if (warp == 0) {
    if (!PACK && lane >= 1 && lane <= kGatherLanes && a.gather != nullptr) {
      // ================= X producer, gathered: the tile's rows straight from the source rows
      // (TMA gather4, 4 rows per op); the packed X is never materialised.  kGatherLanes lanes issue
      // the 32 ops of a k-block together (one issuing thread managed ~1 op / 75 cycles); each lane
      // copies its own row indices of the next tile to shared memory (LDGSTS) a tile ahead.
      constexpr unsigned kMask = ((1u << kGatherLanes) - 1u) << 1;
      const int gl = lane - 1;
      int* sIdx = reinterpret_cast<int*>(smem + S::kOffIdx);
      auto fetch_idx = [&](int tile, int slot) {
        if (tile < num_tiles) {
#pragma unroll
          for (int q = gl; q < BM / 4; q += kGatherLanes)
            cp_async16(sIdx + slot * BM + 4 * q, a.gather + (long)tile * BM + 4 * q);
        }
        cp_async_commit();
      };
      fetch_idx(blockIdx.x, 0);
      int xi = 0, ti = 0;
      for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++ti) {
        fetch_idx(tile + gridDim.x, (ti + 1) & 1);
        cp_async_wait<1>();
        const int4* ix = reinterpret_cast<const int4*>(sIdx + (ti & 1) * BM);
        for (int kb = 0; kb < DK; ++kb, ++xi) {
          const int s = slot_of(xi, S::kXS);
          if (gl == 0) {
            TW(0, mbar_wait(&xempty[s], par_of(xi, S::kXS) ^ 1));
            mbar_expect_tx(&xfull[s], 16384);
          }
          __syncwarp(kMask);
#pragma unroll
          for (int q = gl; q < BM / 4; q += kGatherLanes) {
            const int4 r = ix[q];
            tma_gather4(sX + s * 16384 + q * 512, &tmX, &xfull[s], kb * 64, r.x, r.y, r.z, r.w);
          }
        }
      }
    } else if (lane == 1 && PACK) {
      produce_g();
    } else if (lane == 1) {
      // ================= X producer (lane 1): its own thread, so the next tile's W1 k-blocks do
      // not queue behind X loads that wait for the current tile's last chunk
      int xi = 0;
      for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
        for (int kb = 0; kb < DK; ++kb, ++xi) {
          const int s = slot_of(xi, S::kXS);
          TW(0, mbar_wait(&xempty[s], par_of(xi, S::kXS) ^ 1));
          mbar_expect_tx(&xfull[s], 16384);
          tma_load_2d(sX + s * 16384, &tmX, &xfull[s], kb * 64, tile * BM);   // box {64 k, 128 rows}
        }
      }
    } else if (lane == 0) {
      // ================= W1 producer (lane 0; G: warp 2)
      int wi = 0;
      for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
        const int r0 = tile * BM;
        const int e = find_group(seg_s, a.E, r0);
        for (int c = 0; c < NC; ++c) {
          for (int kb = 0; kb < DK; ++kb, ++wi) {
            const int s = slot_of(wi, S::kWS);
            TW(1, mbar_wait(&wempty[s], par_of(wi, S::kWS) ^ 1));
#ifdef SMES_FWD_EXP_NO_W1      // timing experiment only (wrong results): W1 streamed for the first tile only
            if (tile != (int)blockIdx.x) { mbar_arrive(&wfull[s]); continue; }
#endif
            mbar_expect_tx(&wfull[s], 16384);
            tma_load_3d(sW + s * 16384, &tmW1, &wfull[s], kb * 64, c * CH, e);  // box {64 k, 128 n, 1}
          }
        }
      }
    }
  } else if (warp == 2) {
    if (PACK) {
      // ================= X copy warp (pack mode; the G producer moved to warp 0 lane 1): the tile's rows copied from their source rows
      // src[gather[r]] by LDGSTS (16 B per lane, zero-filled for pad rows), swizzled like a TMA tile;
      // once a k-block's copies land (up to LAG k-blocks later, the tile's last at once) it is fenced to the async proxy, handed to
      // the S-MMA and stored to the packed X (the fc1 weight gradient reads it) -- the plan scatter
      // then only places rows
      constexpr int LAG = 2;
      constexpr int kStoreLag = S::kXS - 1 - LAG > 0 ? S::kXS - 1 - LAG : 0;
      int* sIdx = reinterpret_cast<int*>(smem + S::kOffIdx);
      const int jc = lane & 7, rb = lane >> 3;
      const int per_cta = (num_tiles - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x;
      const int total = per_cta > 0 ? per_cta * DK : 0;
      auto finish = [&](int k) {                   // k-block k of this CTA's sequence has landed
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          const int s = slot_of(k, S::kXS);
          const int tile = (int)blockIdx.x + (k / DK) * (int)gridDim.x, kb = k % DK;
          tma_store_2d(&tmX, sX + s * 16384, kb * 64, tile * BM);
          bulk_commit();
          mbar_arrive(&xfull[s]);
        }
      };
      int done = 0;                                // k-blocks handed over so far
      for (int k = 0; k < total; ++k) {
        const int tile = (int)blockIdx.x + (k / DK) * (int)gridDim.x, kb = k % DK;
        if (kb == 0) {
          __syncwarp();
          const int4 v = __ldg(reinterpret_cast<const int4*>(a.gather + (long)tile * BM) + lane);
          reinterpret_cast<int4*>(sIdx)[lane] = v;
          __syncwarp();
        }
        const int s = slot_of(k, S::kXS);
        if (lane == 0) {
          mbar_wait(&xempty[s], par_of(k, S::kXS) ^ 1);
          bulk_wait_read<kStoreLag>();              // the store of this slot's previous k-block has read it
        }
        __syncwarp();
        uint8_t* dst = sX + s * 16384;
#pragma unroll 8
        for (int i = 0; i < BM / 4; ++i) {
          const int r = rb + 4 * i;
          const int idx = sIdx[r];
          const __nv_bfloat16* g = a.src + (idx >= 0 ? (long)idx * a.ld_src : 0L) + kb * 64 + jc * 8;
          cp_async16_zfill(dst + r * 128 + ((jc ^ (r & 7)) << 4), g, idx >= 0 ? 16 : 0);
        }
        cp_async_commit();
        if (kb == DK - 1) {
          // a tile's k-blocks are all handed over before the next tile's are issued: its slots are
          // released only after this tile's last S-MMA, which needs every k-block of this tile
          cp_async_wait<0>();
          while (done <= k) finish(done++);
        } else if (k - done >= LAG) {
          cp_async_wait<LAG>();
          finish(done++);
        }
      }
      cp_async_wait<0>();
      while (done < total) finish(done++);
      if (lane == 0) bulk_wait<0>();
    } else if (lane == 0) {
      produce_g();
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ================= S-MMA issuer: S_c = X W1[c]^T, never waits on the epilogue's H
      constexpr uint32_t idS = umma_idesc_bf16(BM, CH, 0, 0);
      int xi = 0, wi = 0, si = 0;
      for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
        const int xbase = xi;
        for (int c = 0; c < NC; ++c, ++si) {
          const int sb = slot_of(si, kSB);
          TW(3, mbar_wait(&sempty[sb], par_of(si, kSB) ^ 1));
          EV(0, si);
          tc_fence_after();
          const uint32_t tS = tmem_base + sb * CH;
          for (int kb = 0; kb < DK; ++kb, ++wi) {
            const int xs = slot_of(xbase + kb, S::kXS);
            if (c == 0) TW(4, mbar_wait(&xfull[xs], par_of(xbase + kb, S::kXS)));
            const int ws = slot_of(wi, S::kWS);
            TW(5, mbar_wait(&wfull[ws], par_of(wi, S::kWS)));
            tc_fence_after();
            const uint32_t x_addr = smem_u32(sX + xs * 16384), w_addr = smem_u32(sW + ws * 16384);
#pragma unroll
            for (int k = 0; k < 4; ++k)
              tc_mma_f16(tS, umma_desc_sw128(x_addr + k * 32, 16, 1024), umma_desc_sw128(w_addr + k * 32, 16, 1024),
                         idS, (kb | k) != 0);
            tc_commit(&wempty[ws]);
            if (c == NC - 1) tc_commit(&xempty[xs]);     // X k-block no longer needed by this tile
          }
          tc_commit(&sfull[sb]);
          EV(1, si);
        }
        xi = xbase + DK;
      }
    }
  } else if (warp == 3) {
    if (lane == 0) {
      // ================= P-MMA issuer: P += H_c G[c]^T once the epilogue has staged H_c
      constexpr uint32_t idP = umma_idesc_bf16(BM, 16, 0, 0);
      int gi = 0, hi = 0, it = 0;
      for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++it) {
        const int pb = it & 1;
        const uint32_t tP = tmem_base + kSB * CH + pb * 16;
        for (int c = 0; c < NC; ++c, ++gi, ++hi) {
          const int hb = hi % S::kHB;
          TW(6, mbar_wait(&hfull[hb], (uint32_t)((hi / S::kHB) & 1)));
          const int gs = slot_of(gi, S::kGS);
          TW(7, mbar_wait(&gfull[gs], par_of(gi, S::kGS)));
          EV(6, gi);
          if (c == 0) TW(8, mbar_wait(&pempty[pb], (uint32_t)(((it >> 1) & 1) ^ 1)));
          tc_fence_after();
          const uint32_t h_addr = smem_u32(sH + hb * 32768), g_addr = smem_u32(sG + gs * 4096);
#pragma unroll
          for (int k = 0; k < CH / 16; ++k) {
            const int atom = k >> 2, kk = k & 3;
            tc_mma_f16(tP, umma_desc_sw128(h_addr + atom * 16384 + kk * 32, 16, 1024),
                       umma_desc_sw128(g_addr + atom * 2048 + kk * 32, 16, 1024), idP, (c | k) != 0);
          }
          tc_commit(&hempty[hb]);
          tc_commit(&gempty[gs]);
          EV(7, gi);
        }
        tc_commit(&pfull[pb]);
      }
    }
  } else if (warp >= 4) {
    // ================= epilogue
    const int q = warp & 3;
    const int par = (warp - 4) >> 2;          // 64-column half of the chunk
    float* sbias = reinterpret_cast<float*>(smem + S::kOffBias) + (warp - 4) * 64;
    int si = 0, hi = 0, it = 0;
    // head projections P[row, t] = acc + c[e, t] of a finished tile are read after chunk 1 of the
    // next tile: the tile's last P-MMA queues behind the S-MMAs already issued for that tile, and
    // waiting for it at the tile boundary stalled the epilogue ~2.5 k cycles per tile
    int p_e = -1, p_row = 0, p_it = 0;
    auto store_p = [&]() {
      const int pb = p_it & 1;
      if (warp == 4) TW(11, mbar_wait(&pfull[pb], (uint32_t)((p_it >> 1) & 1))); else mbar_wait(&pfull[pb], (uint32_t)((p_it >> 1) & 1));
      tc_fence_after();
      if (par == 0) {
        uint32_t t0[16];
        tmem_ld16(tmem_base + ((uint32_t)(32 * q) << 16) + kSB * CH + pb * 16, t0);
        tmem_ld_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&pempty[pb]);
        float* prow = a.P + (size_t)p_row * a.ldp;
        const float* ce = a.c + (size_t)p_e * a.ldg;
#pragma unroll
        for (int t = 0; t < 16; t += 4) {
          if (t < a.ldp) {
            float4 v;
            v.x = __uint_as_float(t0[t + 0]) + ce[t + 0];
            v.y = __uint_as_float(t0[t + 1]) + ce[t + 1];
            v.z = __uint_as_float(t0[t + 2]) + ce[t + 2];
            v.w = __uint_as_float(t0[t + 3]) + ce[t + 3];
            *reinterpret_cast<float4*>(prow + t) = v;
          }
        }
      }
      p_e = -1;
    };
    // fc1 bias of the next chunk is fetched one chunk ahead (its L2 latency was on the chain)
    float bv0 = 0.f, bv1 = 0.f;
    if ((int)blockIdx.x < num_tiles) {
      const float* bp = a.b1 + (size_t)find_group(seg_s, a.E, blockIdx.x * BM) * a.d_ff + par * 64 + lane;
      bv0 = __ldg(bp);
      bv1 = __ldg(bp + 32);
    }
    for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++it) {
      const int r0 = tile * BM;
      const int e = find_group(seg_s, a.E, r0);
      const int row = r0 + 32 * q + lane;
      for (int c = 0; c < NC; ++c, ++si) {
        const int n0 = c * CH + par * 64;
        float nb0 = 0.f, nb1 = 0.f;
        {
          const int nt = c + 1 < NC ? tile : tile + (int)gridDim.x, nc = c + 1 < NC ? c + 1 : 0;
          if (nt < num_tiles) {
            const int ne = nc ? e : find_group(seg_s, a.E, nt * BM);
            const float* bp = a.b1 + (size_t)ne * a.d_ff + nc * CH + par * 64 + lane;
            nb0 = __ldg(bp);
            nb1 = __ldg(bp + 32);
          }
        }
        const int sb = slot_of(si, kSB);
        if (warp == 4) TW(9, mbar_wait(&sfull[sb], par_of(si, kSB))); else mbar_wait(&sfull[sb], par_of(si, kSB));
        if (warp == 4 && lane == 0) EV(2, si);
        tc_fence_after();
        // the two 32-column TMEM loads are split: the second is in flight while the first half's
        // bias / ReLU / mask run (the chunk's 64 KB TMEM drain is as long as its S-MMA)
        float f[64];
        const uint32_t ta = tmem_base + ((uint32_t)(32 * q) << 16) + sb * CH + par * 64;
        {
          uint32_t t0[32];
          tmem_ld32(ta, t0);
          tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < 32; ++j) f[j] = __uint_as_float(t0[j]);
        }
        uint32_t t1[32];
        tmem_ld32(ta + 32, t1);
        sbias[lane] = bv0;
        sbias[32 + lane] = bv1;
        __syncwarp();
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          if (hh == 1) {
            tmem_ld_wait();
#pragma unroll
            for (int j = 0; j < 32; ++j) f[32 + j] = __uint_as_float(t1[j]);
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&sempty[sb]);   // accumulator drained into registers
            if (warp == 4 && lane == 0) EV(3, si);
          }
#pragma unroll
          for (int j = 32 * hh; j < 32 * hh + 32; j += 4) {
            const float4 bb = *reinterpret_cast<const float4*>(sbias + j);
            f[j] = fmaxf(f[j] + bb.x, 0.f);
            f[j + 1] = fmaxf(f[j + 1] + bb.y, 0.f);
            f[j + 2] = fmaxf(f[j + 2] + bb.z, 0.f);
            f[j + 3] = fmaxf(f[j + 3] + bb.w, 0.f);
          }
          const uint32_t w = pos_mask32(f + hh * 32);
          if (a.bits != nullptr) a.bits[(size_t)((n0 >> 5) + hh) * a.bits_ld + row] = w;
        }
        if (warp == 4 && lane == 0) EV(8, si);
        if (warp == 4 && lane == 0) EV(9, si);
        if (warp == 4 && lane == 0) EV(9, si);
        // H smem tile hb is free once the P-MMA of the chunk that last used it has read it (and our
        // TMA store of it too; with two tiles the store of the other one may still be reading)
        const int hb = hi % S::kHB;
        uint8_t* sHb = sH + hb * 32768;
        if (warp == 4) TW(10, mbar_wait(&hempty[hb], (uint32_t)(((hi / S::kHB) & 1) ^ 1)));
        else mbar_wait(&hempty[hb], (uint32_t)(((hi / S::kHB) & 1) ^ 1));
        if (warp == 4 && lane == 0) EV(4, si);
        if (lane == 0) {
          if (S::kHB == 2) TW(12, bulk_wait_read<1>()); else TW(12, bulk_wait_read<0>());
        }
        __syncwarp();
        uint8_t* hrow = sHb + par * 16384 + (32 * q + lane) * 128;
#pragma unroll
        for (int cc = 0; cc < 8; ++cc) {
          const uint4 pk = make_uint4(pack_bf16(f[8 * cc], f[8 * cc + 1]), pack_bf16(f[8 * cc + 2], f[8 * cc + 3]),
                                      pack_bf16(f[8 * cc + 4], f[8 * cc + 5]), pack_bf16(f[8 * cc + 6], f[8 * cc + 7]));
          *reinterpret_cast<uint4*>(hrow + ((cc ^ (lane & 7)) << 4)) = pk;
        }
        if (warp == 4 && lane == 0) EV(10, si);
        fence_proxy_async_smem();
        if (warp == 4 && lane == 0) EV(11, si);
        __syncwarp();
        if (lane == 0) {
          if (a.store_h) {
            tma_store_2d(&tmH, sHb + par * 16384 + 32 * q * 128, n0, r0 + 32 * q);
          }
          bulk_commit();                  // (an empty group without a store: the wait counts stay aligned)
          mbar_arrive(&hfull[hb]);
          if (warp == 4) EV(5, si);
        }
        ++hi;
        bv0 = nb0;
        bv1 = nb1;
        if (c == (NC > 1 ? 1 : 0) && p_e >= 0) store_p();     // previous tile's head projections
      }
      p_e = e; p_row = row; p_it = it;
    }
    if (p_e >= 0) store_p();
    if (lane == 0) bulk_wait<0>();
  }
#ifdef SMES_TRACE
  if (threadIdx.x == 128) g_trace[blockIdx.x * 16 + 13] = clock64() - t_start;
  if (threadIdx.x == 32) g_trace[blockIdx.x * 16 + 14] = clock64() - t_start;
  if (threadIdx.x == 0) g_trace[blockIdx.x * 16 + 15] = clock64() - t_start;
  if (threadIdx.x == 128) g_trace[blockIdx.x * 16 + 11] = gtimer();
#endif
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_dealloc(tmem_base, 512);
}


// ============================================================================ forward, CTA pairs
// mlp_fwd2: the same chained forward on a 2-CTA cluster.  The pair runs two consecutive 128-row
// tiles of one expert as one M = 256 tcgen05 MMA (cta_group::2): each CTA holds its own X tile and
// HALF of every W1 / G k-block (N split), so the per-SM W1 traffic -- the L2 stream that bounds
// the single-CTA kernel -- halves.  The leader CTA (rank 0) issues every MMA; transaction bytes of
// both CTAs land on the leader's barriers; MMA completions are multicast to both CTAs; epilogue
// handshakes arrive on the leader's barriers.  Work units are tile pairs inside an expert segment
// (an odd tail tile runs with an idle peer row block whose outputs are not stored).
template <int DK>
struct Fwd2Smem {
  static constexpr int kXS = DK <= 2 ? DK + 2 : DK <= 4 ? DK + 1 : DK;   // X ring (16 KB slots)
  static constexpr int kWS = DK <= 4 ? 8 : 2;          // W1 half k-blocks (8 KB: 64 n x 64 k)
  static constexpr int kGS = 2;                        // G halves (2 KB: 2 x {64 f, 8 t})
  static constexpr int kOffX = 0;
  static constexpr int kOffW = kOffX + kXS * 16384;
  static constexpr int kOffG = kOffW + kWS * 8192;
  static constexpr int kOffH = kOffG + kGS * 2048;
  static constexpr int kOffBias = kOffH + 2 * 32768;   // H double-buffered
  static constexpr int kOffBar = kOffBias + kEpiWarps * 256;
  static constexpr int kOffSeg = kOffBar + 512;
  static constexpr int kBytes = kOffSeg + 2 * 257 * 4 + 1024;
  static_assert(kBytes <= 232448, "mlp_fwd2 smem");
};

template <int DK>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    mlp_fwd2_kernel(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmW1,
                    const __grid_constant__ CUtensorMap tmG, const __grid_constant__ CUtensorMap tmH,
                    const FwdArgs a) {
  pdl_wait();
  using S = Fwd2Smem<DK>;
  extern __shared__ __align__(16) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);   // stays in the shared window
  uint8_t* sX = smem + S::kOffX;
  uint8_t* sW = smem + S::kOffW;
  uint8_t* sG = smem + S::kOffG;
  uint8_t* sH = smem + S::kOffH;
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + S::kOffBar);
  uint64_t* xfull = bar;
  uint64_t* xempty = xfull + S::kXS;
  uint64_t* wfull = xempty + S::kXS;
  uint64_t* wempty = wfull + S::kWS;
  uint64_t* gfull = wempty + S::kWS;
  uint64_t* gempty = gfull + S::kGS;
  uint64_t* sfull = gempty + S::kGS;        // [2]
  uint64_t* sempty = sfull + 2;             // [2]  (leader: 16 epilogue warps of the pair)
  uint64_t* hfull = sempty + 2;             // [2]  (leader: 16)
  uint64_t* hempty = hfull + 2;             // [2]
  uint64_t* pfull = hempty + 2;             // [2]
  uint64_t* pempty = pfull + 2;             // [2]  (leader: 8)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(pempty + 2);
  int* seg_s = reinterpret_cast<int*>(smem + S::kOffSeg);
  int* upref = seg_s + 257;                 // tile-pair units per expert, prefix

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const int NC = a.d_ff / CH;
  for (int i = threadIdx.x; i <= a.E; i += blockDim.x) seg_s[i] = a.seg[i];
  __syncthreads();
  if (threadIdx.x == 0) {
    int u = 0;
    for (int e = 0; e < a.E; ++e) {
      upref[e] = u;
      u += ((seg_s[e + 1] - seg_s[e]) / BM + 1) / 2;
    }
    upref[a.E] = u;
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmX); tma_prefetch(&tmW1); tma_prefetch(&tmG); tma_prefetch(&tmH);
  }
  if (warp == 1 && lane == 0) {
    for (int i = 0; i < S::kXS; ++i) { mbar_init(&xfull[i], 1); mbar_init(&xempty[i], 1); }
    for (int i = 0; i < S::kWS; ++i) { mbar_init(&wfull[i], 1); mbar_init(&wempty[i], 1); }
    for (int i = 0; i < S::kGS; ++i) { mbar_init(&gfull[i], 1); mbar_init(&gempty[i], 1); }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&sfull[i], 1); mbar_init(&sempty[i], 2 * kEpiWarps);
      mbar_init(&pfull[i], 1); mbar_init(&pempty[i], kEpiWarps);
    }
    for (int i = 0; i < 2; ++i) { mbar_init(&hfull[i], 2 * kEpiWarps); mbar_init(&hempty[i], 1); }
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc_2sm(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int num_units = upref[a.E];
#ifdef SMES_TRACE
  const long long t_start = clock64();
  if (threadIdx.x == 0) g_trace[blockIdx.x * 16 + 10] = gtimer();
  int n_my_units = 0;
#endif
  const int cl = blockIdx.x >> 1, ncl = gridDim.x >> 1;
  // decode a unit: expert, first tile row, tiles in the pair (1 or 2)
  auto decode = [&](int u, int& e, int& row_pair, int& nt) {
    int lo = 0, hi = a.E - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (upref[mid] <= u) lo = mid; else hi = mid - 1;
    }
    e = lo;
    const int j = u - upref[e];
    row_pair = seg_s[e] + 2 * j * BM;
    const int tiles = (seg_s[e + 1] - seg_s[e]) / BM;
    nt = min(2, tiles - 2 * j);
  };
  constexpr uint16_t kPair = 0x3;

  if (warp == 0) {
    if (lane == 0) {
      // ================= TMA producer (both CTAs): own X tile, own half of W1 (G: warp 2)
      int xi = 0, wi = 0;
      for (int u = cl; u < num_units; u += ncl) {
        int e, rp, nt;
        decode(u, e, rp, nt);
        const bool valid = (int)rank < nt;
        const int r0 = rp + (int)rank * BM;
        for (int kb = 0; kb < DK; ++kb, ++xi) {
          const int s = slot_of(xi, S::kXS);
          mbar_wait(&xempty[s], par_of(xi, S::kXS) ^ 1);
          if (rank == 0) mbar_expect_tx(&xfull[s], nt * 16384);
          if (valid) tma_load_2d_2sm(sX + s * 16384, &tmX, &xfull[s], kb * 64, r0);
        }
        for (int c = 0; c < NC; ++c) {
          for (int kb = 0; kb < DK; ++kb, ++wi) {
            const int s = slot_of(wi, S::kWS);
            mbar_wait(&wempty[s], par_of(wi, S::kWS) ^ 1);
            if (rank == 0) mbar_expect_tx(&wfull[s], 2 * 8192);
            tma_load_3d_2sm(sW + s * 8192, &tmW1, &wfull[s], kb * 64, c * CH + 64 * rank, e);
          }
        }
      }
    }
  } else if (warp == 2) {
    if (lane == 0) {
      // ================= G producer (both CTAs): own 8 task rows of G[c]; released by the P-MMA, so it
      // runs on its own warp and never holds back the W1 stream of the S-MMA
      int gi = 0;
      for (int u = cl; u < num_units; u += ncl) {
        int e, rp, nt;
        decode(u, e, rp, nt);
        for (int c = 0; c < NC; ++c, ++gi) {
          const int s = slot_of(gi, S::kGS);
          mbar_wait(&gempty[s], par_of(gi, S::kGS) ^ 1);
          if (rank == 0) mbar_expect_tx(&gfull[s], 2 * 2048);
          tma_load_3d_2sm(sG + s * 2048, &tmG, &gfull[s], c * CH, 8 * rank, e);
          tma_load_3d_2sm(sG + s * 2048 + 1024, &tmG, &gfull[s], c * CH + 64, 8 * rank, e);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && rank == 0) {
      // ================= S-MMA issuer (leader): S_c = X W1[c]^T over the pair, M = 256
      constexpr uint32_t idS = umma_idesc_bf16(2 * BM, CH, 0, 0);
      int xi = 0, wi = 0, si = 0;
      for (int u = cl; u < num_units; u += ncl) {
        const int xbase = xi;
        for (int c = 0; c < NC; ++c, ++si) {
          const int sb = si & 1;
          mbar_wait(&sempty[sb], (uint32_t)(((si >> 1) & 1) ^ 1));
          EV(0, si);
          tc_fence_after();
          const uint32_t tS = tmem_base + sb * CH;
          for (int kb = 0; kb < DK; ++kb, ++wi) {
            const int xs = slot_of(xbase + kb, S::kXS);
            if (c == 0) mbar_wait(&xfull[xs], par_of(xbase + kb, S::kXS));
            const int ws = slot_of(wi, S::kWS);
            mbar_wait(&wfull[ws], par_of(wi, S::kWS));
            tc_fence_after();
            const uint32_t x_addr = smem_u32(sX + xs * 16384), w_addr = smem_u32(sW + ws * 8192);
#pragma unroll
            for (int k = 0; k < 4; ++k)
              tc_mma_f16_2sm(tS, umma_desc_sw128(x_addr + k * 32, 16, 1024),
                             umma_desc_sw128(w_addr + k * 32, 16, 1024), idS, (kb | k) != 0);
            tc_commit_2sm_mc(&wempty[ws], kPair);
            if (c == NC - 1) tc_commit_2sm_mc(&xempty[xs], kPair);
          }
          tc_commit_2sm_mc(&sfull[sb], kPair);
          EV(1, si);
        }
        xi = xbase + DK;
      }
    }
  } else if (warp == 3) {
    if (lane == 0 && rank == 0) {
      // ================= P-MMA issuer (leader): P += H_c G[c]^T over the pair, N = 16
      constexpr uint32_t idP = umma_idesc_bf16(2 * BM, 16, 0, 0);
      int gi = 0, hi = 0, it = 0;
      for (int u = cl; u < num_units; u += ncl, ++it) {
        const int pb = it & 1;
        const uint32_t tP = tmem_base + 256 + pb * 16;
        for (int c = 0; c < NC; ++c, ++gi, ++hi) {
          const int hb = hi & 1;
          mbar_wait(&hfull[hb], (uint32_t)((hi >> 1) & 1));
          const int gs = slot_of(gi, S::kGS);
          mbar_wait(&gfull[gs], par_of(gi, S::kGS));
          if (c == 0) mbar_wait(&pempty[pb], (uint32_t)(((it >> 1) & 1) ^ 1));
          EV(6, gi);
          tc_fence_after();
          const uint32_t h_addr = smem_u32(sH + hb * 32768), g_addr = smem_u32(sG + gs * 2048);
#pragma unroll
          for (int k = 0; k < CH / 16; ++k) {
            const int atom = k >> 2, kk = k & 3;
            tc_mma_f16_2sm(tP, umma_desc_sw128(h_addr + atom * 16384 + kk * 32, 16, 1024),
                           umma_desc_sw128(g_addr + atom * 1024 + kk * 32, 16, 1024), idP, (c | k) != 0);
          }
          tc_commit_2sm_mc(&hempty[hb], kPair);
          tc_commit_2sm_mc(&gempty[gs], kPair);
          EV(7, gi);
        }
        tc_commit_2sm_mc(&pfull[pb], kPair);
      }
    }
  } else if (warp >= 4) {
    // ================= epilogue (both CTAs): own 128 rows; handshakes on the leader's barriers.
    // H is double-buffered and a unit's P is read after the NEXT unit's first chunk, so neither the
    // P-MMA nor the head projections sit between two S chunks on the critical path.
    const int q = warp & 3;
    const int par = (warp - 4) >> 2;
    float* sbias = reinterpret_cast<float*>(smem + S::kOffBias) + (warp - 4) * 64;
    const uint32_t lead_sempty0 = mapa_shared(smem_u32(&sempty[0]), 0);
    const uint32_t lead_sempty1 = mapa_shared(smem_u32(&sempty[1]), 0);
    const uint32_t lead_hfull0 = mapa_shared(smem_u32(&hfull[0]), 0);
    const uint32_t lead_hfull1 = mapa_shared(smem_u32(&hfull[1]), 0);
    const uint32_t lead_pempty0 = mapa_shared(smem_u32(&pempty[0]), 0);
    const uint32_t lead_pempty1 = mapa_shared(smem_u32(&pempty[1]), 0);
    int si = 0, hi = 0, it = 0;
    // the unit whose P is pending: expert, row, validity
    int p_e = -1, p_row = 0, p_it = 0;
    bool p_valid = false;
    auto store_p = [&]() {
      const int pb = p_it & 1;
      mbar_wait(&pfull[pb], (uint32_t)((p_it >> 1) & 1));
      tc_fence_after();
      if (par == 0) {
        uint32_t t0[16];
        tmem_ld16(tmem_base + ((uint32_t)(32 * q) << 16) + 256 + pb * 16, t0);
        tmem_ld_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(pb ? lead_pempty1 : lead_pempty0);
        if (p_valid) {
          float* prow = a.P + (size_t)p_row * a.ldp;
          const float* ce = a.c + (size_t)p_e * a.ldg;
#pragma unroll
          for (int t = 0; t < 16; t += 4) {
            if (t < a.ldp) {
              float4 v;
              v.x = __uint_as_float(t0[t + 0]) + ce[t + 0];
              v.y = __uint_as_float(t0[t + 1]) + ce[t + 1];
              v.z = __uint_as_float(t0[t + 2]) + ce[t + 2];
              v.w = __uint_as_float(t0[t + 3]) + ce[t + 3];
              *reinterpret_cast<float4*>(prow + t) = v;
            }
          }
        }
      }
      p_e = -1;
    };
    // fc1 bias of the next chunk fetched one chunk ahead (see mlp_fwd)
    float nb0 = 0.f, nb1 = 0.f;
    auto fetch_bias = [&](int u, int c) {
      if (u < num_units) {
        int e2, rp2, nt2;
        decode(u, e2, rp2, nt2);
        const float* bp = a.b1 + (size_t)e2 * a.d_ff + c * CH + par * 64 + lane;
        nb0 = __ldg(bp);
        nb1 = __ldg(bp + 32);
      }
    };
    fetch_bias(cl, 0);
    for (int u = cl; u < num_units; u += ncl, ++it) {
      int e, rp, nt;
      decode(u, e, rp, nt);
      const bool valid = (int)rank < nt;
      const int r0 = rp + (int)rank * BM;
      const int row = r0 + 32 * q + lane;
      for (int c = 0; c < NC; ++c, ++si) {
        const int n0 = c * CH + par * 64;
        const float bv0 = nb0, bv1 = nb1;
        if (c + 1 < NC) fetch_bias(u, c + 1); else fetch_bias(u + ncl, 0);
        const int sb = si & 1;
        mbar_wait(&sfull[sb], (uint32_t)((si >> 1) & 1));
        if (warp == 4 && lane == 0) EV(2, si);
        tc_fence_after();
        float f[64];
        {
          uint32_t t0[32], t1[32];
          const uint32_t ta = tmem_base + ((uint32_t)(32 * q) << 16) + sb * CH + par * 64;
          tmem_ld32(ta, t0);
          tmem_ld32(ta + 32, t1);
          tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < 32; ++j) { f[j] = __uint_as_float(t0[j]); f[32 + j] = __uint_as_float(t1[j]); }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(sb ? lead_sempty1 : lead_sempty0);
        if (warp == 4 && lane == 0) EV(3, si);
        sbias[lane] = bv0;
        sbias[32 + lane] = bv1;
        __syncwarp();
#pragma unroll
        for (int j = 0; j < 64; j += 4) {
          const float4 bb = *reinterpret_cast<const float4*>(sbias + j);
          f[j] = fmaxf(f[j] + bb.x, 0.f);
          f[j + 1] = fmaxf(f[j + 1] + bb.y, 0.f);
          f[j + 2] = fmaxf(f[j + 2] + bb.z, 0.f);
          f[j + 3] = fmaxf(f[j + 3] + bb.w, 0.f);
        }
        if (valid) {
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const uint32_t w = pos_mask32(f + h * 32);
            if (a.bits != nullptr) a.bits[(size_t)((n0 >> 5) + h) * a.bits_ld + row] = w;
          }
        }
        const int hb = hi & 1;
        mbar_wait(&hempty[hb], (uint32_t)(((hi >> 1) & 1) ^ 1));
        if (warp == 4 && lane == 0) EV(4, si);
        if (lane == 0) bulk_wait_read<1>();     // this buffer's store (two chunks ago) has been read
        __syncwarp();
        uint8_t* hbuf = sH + hb * 32768 + par * 16384;
        uint8_t* hrow = hbuf + (32 * q + lane) * 128;
#pragma unroll
        for (int cc = 0; cc < 8; ++cc) {
          const uint4 pk = make_uint4(pack_bf16(f[8 * cc], f[8 * cc + 1]), pack_bf16(f[8 * cc + 2], f[8 * cc + 3]),
                                      pack_bf16(f[8 * cc + 4], f[8 * cc + 5]), pack_bf16(f[8 * cc + 6], f[8 * cc + 7]));
          *reinterpret_cast<uint4*>(hrow + ((cc ^ (lane & 7)) << 4)) = pk;
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          if (a.store_h && valid) tma_store_2d(&tmH, hbuf + 32 * q * 128, n0, r0 + 32 * q);
          bulk_commit();                          // one group per chunk (possibly empty) keeps wait_read<1> exact
          mbar_arrive_cluster(hb ? lead_hfull1 : lead_hfull0);
          if (warp == 4) EV(5, si);
        }
        ++hi;
        if (c == 0 && p_e >= 0) store_p();      // previous unit's head projections
      }
      p_e = e; p_row = row; p_valid = valid; p_it = it;
    }
    if (p_e >= 0) store_p();
    if (lane == 0) bulk_wait<0>();
  }
#ifdef SMES_TRACE
  if (threadIdx.x == 128) {
    g_trace[blockIdx.x * 16 + 13] = clock64() - t_start;
    for (int u = cl; u < num_units; u += ncl) ++n_my_units;
    g_trace[blockIdx.x * 16 + 12] = n_my_units;
  }
  if (threadIdx.x == 32) g_trace[blockIdx.x * 16 + 14] = clock64() - t_start;
  if (threadIdx.x == 0) g_trace[blockIdx.x * 16 + 15] = clock64() - t_start;
  if (threadIdx.x == 128) g_trace[blockIdx.x * 16 + 11] = gtimer();
#endif
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  if (warp == 2) tmem_dealloc_2sm(tmem_base, 512);
}

// ============================================================================ dgrad
template <int DK>     // d / 64 (the output width of dX)
struct DgSmem {
  static constexpr int kCS = 2;                         // C tile ring (16 KB: {64 t, 128 rows}, K = 16 used)
  static constexpr int kGS = 2;                         // G ring (chunk: 2 x {64 f, 16 t} = 4 KB, MN-major B)
  static constexpr int kWS = DK <= 4 ? 3 : 2;           // W1 k-block ring: 64 f x d (DK x 8 KB boxes {64 j, 64 f})
  static constexpr int kWB = DK * 8192;
  static constexpr int kOffC = 0;
  static constexpr int kOffG = kOffC + kCS * 16384;
  static constexpr int kOffW = kOffG + kGS * 4096;
  // dH chunk double buffer (2 x 16 KB atoms each): the epilogue stages chunk c+1 while the dX
  // MMAs read chunk c.  The dX store staging (8 warps x 4 KB) aliases the buffer the next chunk
  // writes: every writer drains its own bulk stores (bulk_wait_read) before reusing it.
  static constexpr int kOffH = kOffW + kWS * kWB;
  static constexpr int kOffBar = kOffH + 2 * 32768;
  static constexpr int kOffSeg = kOffBar + 512;
  static constexpr int kBytes = kOffSeg + 257 * 4 + 1024;
  static_assert(kBytes <= 232448, "mlp_dgrad smem");
};

template <int DK>
__global__ void __launch_bounds__(kThreads, 1)
    mlp_dgrad_kernel(const __grid_constant__ CUtensorMap tmC, const __grid_constant__ CUtensorMap tmG,
                     const __grid_constant__ CUtensorMap tmW1, const __grid_constant__ CUtensorMap tmDX,
                     const __grid_constant__ CUtensorMap tmDH, const DgradArgs a) {
  pdl_wait();
  using S = DgSmem<DK>;
  constexpr int D = DK * 64;
  extern __shared__ __align__(16) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);   // stays in the shared window
  uint8_t* sC = smem + S::kOffC;
  uint8_t* sG = smem + S::kOffG;
  uint8_t* sW = smem + S::kOffW;
  uint8_t* sH = smem + S::kOffH;
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + S::kOffBar);
  uint64_t* cfull = bar;                   // [kCS]
  uint64_t* cempty = cfull + S::kCS;
  uint64_t* gfull = cempty + S::kCS;       // [kGS]
  uint64_t* gempty = gfull + S::kGS;
  uint64_t* wfull = gempty + S::kGS;       // [kWS]
  uint64_t* wempty = wfull + S::kWS;
  uint64_t* sfull = wempty + S::kWS;       // [2]
  uint64_t* sempty = sfull + 2;
  uint64_t* hfull = sempty + 2;            // [2]
  uint64_t* hempty = hfull + 2;            // [2]
  uint64_t* dfull = hempty + 2;            // [1] dX accumulator
  uint64_t* dempty = dfull + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(dempty + 1);
  int* seg_s = reinterpret_cast<int*>(smem + S::kOffSeg);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int NC = a.d_ff / CH;
  for (int i = threadIdx.x; i <= a.E; i += blockDim.x) seg_s[i] = a.seg[i];
  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmC); tma_prefetch(&tmG); tma_prefetch(&tmW1); tma_prefetch(&tmDX); tma_prefetch(&tmDH);
  }
  if (warp == 1 && lane == 0) {
    for (int i = 0; i < S::kCS; ++i) { mbar_init(&cfull[i], 1); mbar_init(&cempty[i], 1); }
    for (int i = 0; i < S::kGS; ++i) { mbar_init(&gfull[i], 1); mbar_init(&gempty[i], 1); }
    for (int i = 0; i < S::kWS; ++i) { mbar_init(&wfull[i], 1); mbar_init(&wempty[i], 1); }
    for (int i = 0; i < 2; ++i) { mbar_init(&sfull[i], 1); mbar_init(&sempty[i], kEpiWarps); }
    for (int i = 0; i < 2; ++i) { mbar_init(&hfull[i], kEpiWarps); mbar_init(&hempty[i], 1); }
    mbar_init(dfull, 1);
    mbar_init(dempty, kEpiWarps);
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int num_tiles = seg_s[a.E] / BM;
  // TMEM: S double buffer at [0, 256), dX accumulator at [256, 256 + D)

  if (warp == 0) {
    if (lane == 0) {
      int ci = 0, wi = 0;
      for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++ci) {
        const int r0 = tile * BM;
        const int e = find_group(seg_s, a.E, r0);
        {
          const int s = slot_of(ci, S::kCS);
          mbar_wait(&cempty[s], par_of(ci, S::kCS) ^ 1);
          mbar_expect_tx(&cfull[s], 16384);
          tma_load_2d(sC + s * 16384, &tmC, &cfull[s], 0, r0);                   // box {64 t, 128 rows}
        }
        for (int c = 0; c < NC; ++c) {
          for (int kb = 0; kb < CH / 64; ++kb, ++wi) {
            const int s = slot_of(wi, S::kWS);
            mbar_wait(&wempty[s], par_of(wi, S::kWS) ^ 1);
            mbar_expect_tx(&wfull[s], S::kWB);
#pragma unroll
            for (int j = 0; j < DK; ++j)                                          // box {64 j, 64 f, 1}
              tma_load_3d(sW + s * S::kWB + j * 8192, &tmW1, &wfull[s], 64 * j, c * CH + kb * 64, e);
          }
        }
      }
    }
  } else if (warp == 3) {
    if (lane == 0) {
      // ================= G producer: released by the S-MMA.  In the W1 producer's order a G chunk
      // queued behind W1 k-blocks and held the in-order MMA issuer (S-MMA before dX-MMA) back
      int gi = 0;
      for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
        const int e = find_group(seg_s, a.E, tile * BM);
        for (int c = 0; c < NC; ++c, ++gi) {
          const int s = slot_of(gi, S::kGS);
          mbar_wait(&gempty[s], par_of(gi, S::kGS) ^ 1);
          mbar_expect_tx(&gfull[s], 4096);
          tma_load_3d(sG + s * 4096, &tmG, &gfull[s], c * CH, 0, e);              // box {64 f, 16 t, 1}
          tma_load_3d(sG + s * 4096 + 2048, &tmG, &gfull[s], c * CH + 64, 0, e);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idS = umma_idesc_bf16(BM, CH, 0, 1);     // A = C (K-major), B = G (MN-major)
      constexpr uint32_t idD = umma_idesc_bf16(BM, D, 0, 1);      // A = dH (K-major), B = W1 (MN-major)
      int ci = 0, gi = 0, wi = 0, si = 0, hi = 0, it = 0;
      for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++ci, ++it) {
        const int cs = slot_of(ci, S::kCS);
        mbar_wait(&cfull[cs], par_of(ci, S::kCS));
        const uint32_t c_addr = smem_u32(sC + cs * 16384);
        auto s_mma = [&](int c) {
          const int sb = si & 1;
          mbar_wait(&sempty[sb], (uint32_t)(((si >> 1) & 1) ^ 1));
          const int gs = slot_of(gi, S::kGS);
          mbar_wait(&gfull[gs], par_of(gi, S::kGS));
          tc_fence_after();
          const uint32_t g_addr = smem_u32(sG + gs * 4096);
          // K = 16 (tasks), one MMA; B MN-major: two 64-wide f atoms 2 KB apart
          tc_mma_f16(tmem_base + sb * CH, umma_desc_sw128(c_addr, 16, 1024), umma_desc_sw128(g_addr, 2048, 1024),
                     idS, 0u);
          tc_commit(&sfull[sb]);
          tc_commit(&gempty[gs]);
          EV(0, si);
          ++gi; ++si;
        };
        s_mma(0);
        for (int c = 0; c < NC; ++c) {
          if (c + 1 < NC) s_mma(c + 1);
          if (c == NC - 1) tc_commit(&cempty[cs]);
          const int hb = hi & 1;
          mbar_wait(&hfull[hb], (uint32_t)((hi >> 1) & 1));
          EV(1, hi);
          // the dX accumulator must be drained by the previous tile's epilogue
          if (c == 0) mbar_wait(dempty, (uint32_t)((it & 1) ^ 1));
          EV(2, hi);
          tc_fence_after();
          const uint32_t h_addr = smem_u32(sH + hb * 32768);
          for (int kb = 0; kb < CH / 64; ++kb, ++wi) {
            const int ws = slot_of(wi, S::kWS);
            mbar_wait(&wfull[ws], par_of(wi, S::kWS));
            tc_fence_after();
            const uint32_t w_addr = smem_u32(sW + ws * S::kWB);
#pragma unroll
            for (int k = 0; k < 4; ++k)
              tc_mma_f16(tmem_base + 256, umma_desc_sw128(h_addr + kb * 16384 + k * 32, 16, 1024),
                         umma_desc_sw128(w_addr + k * 2048, 8192, 1024), idD, (c | kb | k) != 0);
            tc_commit(&wempty[ws]);
          }
          tc_commit(&hempty[hb]);
          EV(3, hi);
          ++hi;
        }
        tc_commit(dfull);
      }
    }
  } else if (warp >= 4) {
    const int q = warp & 3;
    const int par = (warp - 4) >> 2;
    int si = 0, hi = 0, it = 0;
    // dX of a finished tile is drained after chunk 0 of the next tile: that chunk's dH work then
    // overlaps the tile's last dX MMAs, and the next dX MMAs start as soon as the drain is done
    int d_it = -1, d_r0 = 0;
    auto drain = [&]() {
      // dX tile: TMEM [256, 256 + D) -> bf16 -> TMA store, 64-column chunks split by parity
      mbar_wait(dfull, (uint32_t)(d_it & 1));
      tc_fence_after();
      // all dX MMAs of that tile are complete and the chunk just staged sits in the other dH
      // buffer: stage in the one the next chunk writes
      uint8_t* stg = sH + (hi & 1) * 32768 + (warp - 4) * 4096;
      for (int cc = par; cc < DK; cc += 2) {
        uint32_t t0[32], t1[32];
        const uint32_t ta = tmem_base + ((uint32_t)(32 * q) << 16) + 256 + cc * 64;
        tmem_ld32(ta, t0);
        tmem_ld32(ta + 32, t1);
        tmem_ld_wait();
        if (lane == 0) bulk_wait_read<0>();
        __syncwarp();
        uint4* rowp = reinterpret_cast<uint4*>(stg + lane * 128);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const uint32_t* src = k < 4 ? t0 : t1;
          const int o = (k & 3) * 8;
          rowp[k ^ (lane & 7)] = make_uint4(
              pack_bf16(__uint_as_float(src[o]), __uint_as_float(src[o + 1])),
              pack_bf16(__uint_as_float(src[o + 2]), __uint_as_float(src[o + 3])),
              pack_bf16(__uint_as_float(src[o + 4]), __uint_as_float(src[o + 5])),
              pack_bf16(__uint_as_float(src[o + 6]), __uint_as_float(src[o + 7])));
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          tma_store_2d(&tmDX, stg, cc * 64, d_r0 + 32 * q);
          bulk_commit();
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(dempty);
      d_it = -1;
    };
    // relu-mask words of the next chunk are fetched one chunk ahead: the S-MMA (K = T) is always
    // ready first, so a mask load issued at the chunk start stalled the epilogue ~1.5 k cycles
    uint32_t nm0 = 0u, nm1 = 0u;
    auto fetch_mask = [&](int tile, int c) {
      if (tile < num_tiles) {
        const int rr = tile * BM + 32 * q + lane, nn = c * CH + par * 64;
        nm0 = __ldg(&a.bits[(size_t)(nn >> 5) * a.bits_ld + rr]);
        nm1 = __ldg(&a.bits[(size_t)((nn >> 5) + 1) * a.bits_ld + rr]);
      }
    };
    fetch_mask(blockIdx.x, 0);
    for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++it) {
      const int r0 = tile * BM;
      for (int c = 0; c < NC; ++c, ++si) {
        const int n0 = c * CH + par * 64;
        const uint32_t m0 = nm0, m1 = nm1;
        if (c + 1 < NC) fetch_mask(tile, c + 1); else fetch_mask(tile + gridDim.x, 0);
        const int sb = si & 1;
        mbar_wait(&sfull[sb], (uint32_t)((si >> 1) & 1));
        if (warp == 4 && lane == 0) EV(4, si);
        tc_fence_after();
        float f[64];
        {
          uint32_t t0[32], t1[32];
          const uint32_t ta = tmem_base + ((uint32_t)(32 * q) << 16) + sb * CH + par * 64;
          tmem_ld32(ta, t0);
          tmem_ld32(ta + 32, t1);
          tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            f[j] = ((m0 >> j) & 1u) ? __uint_as_float(t0[j]) : 0.f;
            f[32 + j] = ((m1 >> j) & 1u) ? __uint_as_float(t1[j]) : 0.f;
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&sempty[sb]);
        if (warp == 4 && lane == 0) EV(5, si);
        const int hb = hi & 1;
        mbar_wait(&hempty[hb], (uint32_t)(((hi >> 1) & 1) ^ 1));
        if (warp == 4 && lane == 0) EV(6, si);
        if (lane == 0) bulk_wait_read<0>();     // own dH / dX-staging stores out of this buffer
        __syncwarp();
        uint8_t* hbuf = sH + hb * 32768;
        uint8_t* hrow = hbuf + par * 16384 + (32 * q + lane) * 128;
#pragma unroll
        for (int cc = 0; cc < 8; ++cc) {
          const uint4 pk = make_uint4(pack_bf16(f[8 * cc], f[8 * cc + 1]), pack_bf16(f[8 * cc + 2], f[8 * cc + 3]),
                                      pack_bf16(f[8 * cc + 4], f[8 * cc + 5]), pack_bf16(f[8 * cc + 6], f[8 * cc + 7]));
          *reinterpret_cast<uint4*>(hrow + ((cc ^ (lane & 7)) << 4)) = pk;
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          if (a.store_dh) {
            tma_store_2d(&tmDH, hbuf + par * 16384 + 32 * q * 128, n0, r0 + 32 * q);
            bulk_commit();
          }
          mbar_arrive(&hfull[hb]);
          if (warp == 4) EV(7, si);
        }
        ++hi;
        if (c == 0 && d_it >= 0) drain();      // previous tile's dX
      }
      d_it = it; d_r0 = r0;
    }
    if (d_it >= 0) drain();
    if (lane == 0) bulk_wait<0>();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_dealloc(tmem_base, 512);
}

// ============================================================================ dgrad, CTA pairs
// mlp_dgrad2: the dgrad on 2-CTA clusters.  Each CTA of the pair loads half of every W1 k-block
// (N = d split) and half of every G chunk (N = 128 f split); the leader issues M = 256 MMAs.
// The single-CTA kernel streams 256 KB of W1 per 128-row tile from L2 and is bound by that stream
// (ncu: producer waiting on W slots, epilogue waiting on S behind the starved dX MMAs).
template <int DK>
struct Dg2Smem {
  static constexpr int kCS = 2;
  static constexpr int kGS = 2;                         // G halves: {64 f, 16 t} = 2 KB
  static constexpr int kWB = DK / 2 * 8192;             // W1 half k-block: DK/2 boxes {64 j, 64 f}
  static constexpr int kWS = DK <= 2 ? 8 : 6;
  static constexpr int kOffC = 0;
  static constexpr int kOffG = kOffC + kCS * 16384;
  static constexpr int kOffW = kOffG + kGS * 2048;
  // dH double buffer; the dX store staging aliases the buffer the next chunk writes (see mlp_dgrad)
  static constexpr int kOffH = kOffW + kWS * kWB;
  static constexpr int kOffBar = kOffH + 2 * 32768;
  static constexpr int kOffSeg = kOffBar + 512;
  static constexpr int kBytes = kOffSeg + 2 * 257 * 4 + 1024;
  static_assert(kBytes <= 232448, "mlp_dgrad2 smem");
};

template <int DK>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    mlp_dgrad2_kernel(const __grid_constant__ CUtensorMap tmC, const __grid_constant__ CUtensorMap tmG,
                      const __grid_constant__ CUtensorMap tmW1, const __grid_constant__ CUtensorMap tmDX,
                      const __grid_constant__ CUtensorMap tmDH, const DgradArgs a) {
  pdl_wait();
  using S = Dg2Smem<DK>;
  constexpr int D = DK * 64;
  extern __shared__ __align__(16) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);   // stays in the shared window
  uint8_t* sC = smem + S::kOffC;
  uint8_t* sG = smem + S::kOffG;
  uint8_t* sW = smem + S::kOffW;
  uint8_t* sH = smem + S::kOffH;
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + S::kOffBar);
  uint64_t* cfull = bar;
  uint64_t* cempty = cfull + S::kCS;
  uint64_t* gfull = cempty + S::kCS;
  uint64_t* gempty = gfull + S::kGS;
  uint64_t* wfull = gempty + S::kGS;
  uint64_t* wempty = wfull + S::kWS;
  uint64_t* sfull = wempty + S::kWS;       // [2]
  uint64_t* sempty = sfull + 2;            // [2] (leader: 16)
  uint64_t* hfull = sempty + 2;            // [2] (leader: 16)
  uint64_t* hempty = hfull + 2;            // [2]
  uint64_t* dfull = hempty + 2;
  uint64_t* dempty = dfull + 1;            // (leader: 16)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(dempty + 1);
  int* seg_s = reinterpret_cast<int*>(smem + S::kOffSeg);
  int* upref = seg_s + 257;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const int NC = a.d_ff / CH;
  for (int i = threadIdx.x; i <= a.E; i += blockDim.x) seg_s[i] = a.seg[i];
  __syncthreads();
  if (threadIdx.x == 0) {
    int u = 0;
    for (int e = 0; e < a.E; ++e) {
      upref[e] = u;
      u += ((seg_s[e + 1] - seg_s[e]) / BM + 1) / 2;
    }
    upref[a.E] = u;
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmC); tma_prefetch(&tmG); tma_prefetch(&tmW1); tma_prefetch(&tmDX); tma_prefetch(&tmDH);
  }
  if (warp == 1 && lane == 0) {
    for (int i = 0; i < S::kCS; ++i) { mbar_init(&cfull[i], 1); mbar_init(&cempty[i], 1); }
    for (int i = 0; i < S::kGS; ++i) { mbar_init(&gfull[i], 1); mbar_init(&gempty[i], 1); }
    for (int i = 0; i < S::kWS; ++i) { mbar_init(&wfull[i], 1); mbar_init(&wempty[i], 1); }
    for (int i = 0; i < 2; ++i) { mbar_init(&sfull[i], 1); mbar_init(&sempty[i], 2 * kEpiWarps); }
    for (int i = 0; i < 2; ++i) { mbar_init(&hfull[i], 2 * kEpiWarps); mbar_init(&hempty[i], 1); }
    mbar_init(dfull, 1);
    mbar_init(dempty, 2 * kEpiWarps);
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc_2sm(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int num_units = upref[a.E];
  const int cl = blockIdx.x >> 1, ncl = gridDim.x >> 1;
  auto decode = [&](int u, int& e, int& row_pair, int& nt) {
    int lo = 0, hi = a.E - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (upref[mid] <= u) lo = mid; else hi = mid - 1;
    }
    e = lo;
    const int j = u - upref[e];
    row_pair = seg_s[e] + 2 * j * BM;
    const int tiles = (seg_s[e + 1] - seg_s[e]) / BM;
    nt = min(2, tiles - 2 * j);
  };
  constexpr uint16_t kPair = 0x3;

  if (warp == 0) {
    if (lane == 0) {
      int ci = 0, wi = 0;
      for (int u = cl; u < num_units; u += ncl, ++ci) {
        int e, rp, nt;
        decode(u, e, rp, nt);
        const bool valid = (int)rank < nt;
        const int r0 = rp + (int)rank * BM;
        {
          const int s = slot_of(ci, S::kCS);
          mbar_wait(&cempty[s], par_of(ci, S::kCS) ^ 1);
          if (rank == 0) mbar_expect_tx(&cfull[s], nt * 16384);
          if (valid) tma_load_2d_2sm(sC + s * 16384, &tmC, &cfull[s], 0, r0);
        }
        for (int c = 0; c < NC; ++c) {
          for (int kb = 0; kb < CH / 64; ++kb, ++wi) {
            const int s = slot_of(wi, S::kWS);
            mbar_wait(&wempty[s], par_of(wi, S::kWS) ^ 1);
            if (rank == 0) mbar_expect_tx(&wfull[s], 2 * S::kWB);
#pragma unroll
            for (int j = 0; j < DK / 2; ++j)
              tma_load_3d_2sm(sW + s * S::kWB + j * 8192, &tmW1, &wfull[s], 64 * (j + rank * (DK / 2)),
                              c * CH + kb * 64, e);
          }
        }
      }
    }
  } else if (warp == 3) {
    if (lane == 0) {
      // ================= G producer (both CTAs, own half): off the W1 stream (see mlp_dgrad)
      int gi = 0;
      for (int u = cl; u < num_units; u += ncl) {
        int e, rp, nt;
        decode(u, e, rp, nt);
        for (int c = 0; c < NC; ++c, ++gi) {
          const int s = slot_of(gi, S::kGS);
          mbar_wait(&gempty[s], par_of(gi, S::kGS) ^ 1);
          if (rank == 0) mbar_expect_tx(&gfull[s], 2 * 2048);
          tma_load_3d_2sm(sG + s * 2048, &tmG, &gfull[s], c * CH + 64 * rank, 0, e);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && rank == 0) {
      constexpr uint32_t idS = umma_idesc_bf16(2 * BM, CH, 0, 1);
      constexpr uint32_t idD = umma_idesc_bf16(2 * BM, D, 0, 1);
      int ci = 0, gi = 0, wi = 0, si = 0, hi = 0, it = 0;
      for (int u = cl; u < num_units; u += ncl, ++ci, ++it) {
        const int cs = slot_of(ci, S::kCS);
        mbar_wait(&cfull[cs], par_of(ci, S::kCS));
        const uint32_t c_addr = smem_u32(sC + cs * 16384);
        auto s_mma = [&](int c) {
          const int sb = si & 1;
          mbar_wait(&sempty[sb], (uint32_t)(((si >> 1) & 1) ^ 1));
          const int gs = slot_of(gi, S::kGS);
          mbar_wait(&gfull[gs], par_of(gi, S::kGS));
          tc_fence_after();
          tc_mma_f16_2sm(tmem_base + sb * CH, umma_desc_sw128(c_addr, 16, 1024),
                         umma_desc_sw128(smem_u32(sG + gs * 2048), 2048, 1024), idS, 0u);
          tc_commit_2sm_mc(&sfull[sb], kPair);
          tc_commit_2sm_mc(&gempty[gs], kPair);
          ++gi; ++si;
        };
        s_mma(0);
        for (int c = 0; c < NC; ++c) {
          if (c + 1 < NC) s_mma(c + 1);
          if (c == NC - 1) tc_commit_2sm_mc(&cempty[cs], kPair);
          const int hb = hi & 1;
          mbar_wait(&hfull[hb], (uint32_t)((hi >> 1) & 1));
          if (c == 0) mbar_wait(dempty, (uint32_t)((it & 1) ^ 1));
          tc_fence_after();
          const uint32_t h_addr = smem_u32(sH + hb * 32768);
          for (int kb = 0; kb < CH / 64; ++kb, ++wi) {
            const int ws = slot_of(wi, S::kWS);
            mbar_wait(&wfull[ws], par_of(wi, S::kWS));
            tc_fence_after();
            const uint32_t w_addr = smem_u32(sW + ws * S::kWB);
#pragma unroll
            for (int k = 0; k < 4; ++k)
              tc_mma_f16_2sm(tmem_base + 256, umma_desc_sw128(h_addr + kb * 16384 + k * 32, 16, 1024),
                             umma_desc_sw128(w_addr + k * 2048, 8192, 1024), idD, (c | kb | k) != 0);
            tc_commit_2sm_mc(&wempty[ws], kPair);
          }
          tc_commit_2sm_mc(&hempty[hb], kPair);
          ++hi;
        }
        tc_commit_2sm_mc(dfull, kPair);
      }
    }
  } else if (warp >= 4) {
    const int q = warp & 3;
    const int par = (warp - 4) >> 2;
    const uint32_t lead_sempty0 = mapa_shared(smem_u32(&sempty[0]), 0);
    const uint32_t lead_sempty1 = mapa_shared(smem_u32(&sempty[1]), 0);
    const uint32_t lead_hfull0 = mapa_shared(smem_u32(&hfull[0]), 0);
    const uint32_t lead_hfull1 = mapa_shared(smem_u32(&hfull[1]), 0);
    const uint32_t lead_dempty = mapa_shared(smem_u32(dempty), 0);
    int si = 0, hi = 0, it = 0;
    // dX of a finished unit is drained after chunk 0 of the next unit (see mlp_dgrad); staging in
    // the dH buffer the next chunk writes
    int d_it = -1, d_r0 = 0;
    bool d_valid = false;
    auto drain = [&]() {
      uint8_t* stg = sH + (hi & 1) * 32768 + (warp - 4) * 4096;
      mbar_wait(dfull, (uint32_t)(d_it & 1));
      tc_fence_after();
      for (int cc = par; cc < DK; cc += 2) {
        uint32_t t0[32], t1[32];
        const uint32_t ta = tmem_base + ((uint32_t)(32 * q) << 16) + 256 + cc * 64;
        tmem_ld32(ta, t0);
        tmem_ld32(ta + 32, t1);
        tmem_ld_wait();
        if (cc + 2 >= DK) {   // last TMEM read of this tile: hand the accumulator back early
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive_cluster(lead_dempty);
        }
        if (!d_valid) continue;
        if (lane == 0) bulk_wait_read<0>();
        __syncwarp();
        uint4* rowp = reinterpret_cast<uint4*>(stg + lane * 128);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const uint32_t* src = k < 4 ? t0 : t1;
          const int o = (k & 3) * 8;
          rowp[k ^ (lane & 7)] = make_uint4(
              pack_bf16(__uint_as_float(src[o]), __uint_as_float(src[o + 1])),
              pack_bf16(__uint_as_float(src[o + 2]), __uint_as_float(src[o + 3])),
              pack_bf16(__uint_as_float(src[o + 4]), __uint_as_float(src[o + 5])),
              pack_bf16(__uint_as_float(src[o + 6]), __uint_as_float(src[o + 7])));
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          tma_store_2d(&tmDX, stg, cc * 64, d_r0 + 32 * q);
          bulk_commit();
        }
      }
      d_it = -1;
    };
    // relu-mask words fetched one chunk ahead (see mlp_dgrad)
    uint32_t nm0 = 0u, nm1 = 0u;
    auto fetch_mask = [&](int u, int c) {
      nm0 = nm1 = 0u;
      if (u < num_units) {
        int e2, rp2, nt2;
        decode(u, e2, rp2, nt2);
        if ((int)rank < nt2) {
          const int rr = rp2 + (int)rank * BM + 32 * q + lane, nn = c * CH + par * 64;
          nm0 = __ldg(&a.bits[(size_t)(nn >> 5) * a.bits_ld + rr]);
          nm1 = __ldg(&a.bits[(size_t)((nn >> 5) + 1) * a.bits_ld + rr]);
        }
      }
    };
    fetch_mask(cl, 0);
    for (int u = cl; u < num_units; u += ncl, ++it) {
      int e, rp, nt;
      decode(u, e, rp, nt);
      const bool valid = (int)rank < nt;
      const int r0 = rp + (int)rank * BM;
      for (int c = 0; c < NC; ++c, ++si) {
        const int n0 = c * CH + par * 64;
        const uint32_t m0 = nm0, m1 = nm1;
        if (c + 1 < NC) fetch_mask(u, c + 1); else fetch_mask(u + ncl, 0);
        const int sb = si & 1;
        mbar_wait(&sfull[sb], (uint32_t)((si >> 1) & 1));
        tc_fence_after();
        float f[64];
        {
          uint32_t t0[32], t1[32];
          const uint32_t ta = tmem_base + ((uint32_t)(32 * q) << 16) + sb * CH + par * 64;
          tmem_ld32(ta, t0);
          tmem_ld32(ta + 32, t1);
          tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            f[j] = ((m0 >> j) & 1u) ? __uint_as_float(t0[j]) : 0.f;
            f[32 + j] = ((m1 >> j) & 1u) ? __uint_as_float(t1[j]) : 0.f;
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(sb ? lead_sempty1 : lead_sempty0);
        const int hb = hi & 1;
        mbar_wait(&hempty[hb], (uint32_t)(((hi >> 1) & 1) ^ 1));
        if (lane == 0) bulk_wait_read<0>();     // own dH / dX-staging stores out of this buffer
        __syncwarp();
        uint8_t* hbuf = sH + hb * 32768;
        uint8_t* hrow = hbuf + par * 16384 + (32 * q + lane) * 128;
#pragma unroll
        for (int cc = 0; cc < 8; ++cc) {
          const uint4 pk = make_uint4(pack_bf16(f[8 * cc], f[8 * cc + 1]), pack_bf16(f[8 * cc + 2], f[8 * cc + 3]),
                                      pack_bf16(f[8 * cc + 4], f[8 * cc + 5]), pack_bf16(f[8 * cc + 6], f[8 * cc + 7]));
          *reinterpret_cast<uint4*>(hrow + ((cc ^ (lane & 7)) << 4)) = pk;
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          if (a.store_dh && valid) {
            tma_store_2d(&tmDH, hbuf + par * 16384 + 32 * q * 128, n0, r0 + 32 * q);
            bulk_commit();
          }
          mbar_arrive_cluster(hb ? lead_hfull1 : lead_hfull0);
        }
        ++hi;
        if (c == 0 && d_it >= 0) drain();      // previous unit's dX (see mlp_dgrad)
      }
      d_it = it; d_r0 = r0; d_valid = valid;
    }
    if (d_it >= 0) drain();
    if (lane == 0) bulk_wait<0>();
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  if (warp == 2) tmem_dealloc_2sm(tmem_base, 512);
}


// ============================================================================ fc1 weight gradient
// mlp_wgrad: one CTA per (expert e, 128-wide d_ff chunk c); the K loop runs over the expert's
// packed rows in 128-row blocks and recomputes dH on the fly instead of reading it:
//   S  = C_blk G_e[:, c]        (K = T)      -> TMEM
//   dH = S * relu-mask          (epilogue)   -> smem, MN-major A operand (M = d_ff chunk, K = rows)
//   dW1[c] += dH^T X_blk        (N = d)      -> TMEM, fp32
//   db1[c] += dH^T 1            (N = 16 against a constant ones tile)
// so dH never goes to HBM (training.py:180-191 for fc1: dW = d_pre^T X, db = colsum(d_pre)).
struct WgradArgs {
  const int* seg;
  int E, d, d_ff;
  const uint32_t* bits;
  int bits_ld;
  float* dW;                     // (E, d_ff, d)
  float* db;                     // (E, d_ff)
};

template <int DK>
struct WgSmem {
  static constexpr int kXS = 3;                          // X ring: 64-row sub-blocks (DK x 8 KB boxes)
  static constexpr int kXB = DK * 8192;
  static constexpr int kCS = 2;                          // C ring: {64 t, 128 rows} boxes
  static constexpr int kOffX = 0;
  static constexpr int kOffC = kOffX + kXS * kXB;
  static constexpr int kOffG = kOffC + kCS * 16384;      // G chunk: 2 x {64 f, 16 t}
  static constexpr int kOffDH = kOffG + 4096;            // 2 buffers x (2 halves x 128 rows x 128 B)
  static constexpr int kOffOnes = kOffDH + 2 * 32768;    // 64 x 64 bf16, column 0 = 1
  static constexpr int kOffBar = kOffOnes + 8192;
  static constexpr int kBytes = kOffBar + 256 + 1024;
  static_assert(kBytes <= 232448, "mlp_wgrad smem");
};

template <int DK>
__global__ void __launch_bounds__(kThreads, 1)
    mlp_wgrad_kernel(const __grid_constant__ CUtensorMap tmC, const __grid_constant__ CUtensorMap tmG,
                     const __grid_constant__ CUtensorMap tmX, const WgradArgs a) {
  pdl_wait();
  using S = WgSmem<DK>;
  constexpr int D = DK * 64;
  extern __shared__ __align__(16) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);   // stays in the shared window
  uint8_t* sX = smem + S::kOffX;
  uint8_t* sC = smem + S::kOffC;
  uint8_t* sG = smem + S::kOffG;
  uint8_t* sDH = smem + S::kOffDH;
  uint8_t* sOnes = smem + S::kOffOnes;
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + S::kOffBar);
  uint64_t* xfull = bar;                    // [kXS]
  uint64_t* xempty = xfull + S::kXS;
  uint64_t* cfull = xempty + S::kXS;        // [kCS]
  uint64_t* cempty = cfull + S::kCS;
  uint64_t* gfull = cempty + S::kCS;        // [1]
  uint64_t* sfull = gfull + 1;              // [1]
  uint64_t* sempty = sfull + 1;             // [1]
  uint64_t* dhfull = sempty + 1;            // [2]
  uint64_t* dhempty = dhfull + 2;           // [2]
  uint64_t* accfull = dhempty + 2;          // [1]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(accfull + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int NC = a.d_ff / CH;
  const int e = blockIdx.x / NC, c = blockIdx.x % NC;
  const int row_lo = a.seg[e];
  const int nkb = (a.seg[e + 1] - row_lo) / BM;
  {
    uint32_t* o32 = reinterpret_cast<uint32_t*>(sOnes);
    for (int i = threadIdx.x; i < 8192 / 4; i += blockDim.x) o32[i] = 0u;
    __syncthreads();
    if (threadIdx.x < 64) {
      const int k = threadIdx.x;
      reinterpret_cast<__nv_bfloat16*>(sOnes + k * 128 + (k & 7) * 16)[0] = __float2bfloat16_rn(1.f);
    }
    fence_proxy_async_smem();
  }
  if (warp == 0 && lane == 0) { tma_prefetch(&tmC); tma_prefetch(&tmG); tma_prefetch(&tmX); }
  if (warp == 1 && lane == 0) {
    for (int i = 0; i < S::kXS; ++i) { mbar_init(&xfull[i], 1); mbar_init(&xempty[i], 1); }
    for (int i = 0; i < S::kCS; ++i) { mbar_init(&cfull[i], 1); mbar_init(&cempty[i], 1); }
    mbar_init(gfull, 1);
    mbar_init(sfull, 1);
    mbar_init(sempty, kEpiWarps);
    for (int i = 0; i < 2; ++i) { mbar_init(&dhfull[i], kEpiWarps); mbar_init(&dhempty[i], 1); }
    mbar_init(accfull, 1);
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  // TMEM: S [0, 128), dW1 [128, 128 + D), ones-product (db) [384, 400)

  if (warp == 0) {
    if (lane == 0 && nkb > 0) {
      mbar_expect_tx(gfull, 4096);
      tma_load_3d(sG, &tmG, gfull, c * CH, 0, e);
      tma_load_3d(sG + 2048, &tmG, gfull, c * CH + 64, 0, e);
      for (int kb = 0; kb < nkb; ++kb) {
        const int r0 = row_lo + kb * BM;
        {
          const int s = kb % S::kCS;
          mbar_wait(&cempty[s], par_of(kb, S::kCS) ^ 1);
          mbar_expect_tx(&cfull[s], 16384);
          tma_load_2d(sC + s * 16384, &tmC, &cfull[s], 0, r0);
        }
        for (int hh = 0; hh < 2; ++hh) {
          const int sub = 2 * kb + hh;
          const int s = slot_of(sub, S::kXS);
          mbar_wait(&xempty[s], par_of(sub, S::kXS) ^ 1);
          mbar_expect_tx(&xfull[s], S::kXB);
#pragma unroll
          for (int j = 0; j < DK; ++j) tma_load_2d(sX + s * S::kXB + j * 8192, &tmX, &xfull[s], 64 * j, r0 + 64 * hh);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && nkb > 0) {
      constexpr uint32_t idS = umma_idesc_bf16(BM, CH, 0, 1);   // A = C (K-major), B = G (MN-major)
      constexpr uint32_t idW = umma_idesc_bf16(BM, D, 1, 1);    // A = dH (MN-major), B = X (MN-major)
      constexpr uint32_t idB = umma_idesc_bf16(BM, 16, 1, 1);   // A = dH, B = ones
      const uint32_t g_addr = smem_u32(sG), ones = smem_u32(sOnes);
      mbar_wait(gfull, 0);
      auto s_mma = [&](int kb) {
        const int cs = kb % S::kCS;
        mbar_wait(&cfull[cs], par_of(kb, S::kCS));
        mbar_wait(sempty, (uint32_t)((kb & 1) ^ 1));
        tc_fence_after();
        tc_mma_f16(tmem_base, umma_desc_sw128(smem_u32(sC + cs * 16384), 16, 1024),
                   umma_desc_sw128(g_addr, 2048, 1024), idS, 0u);
        tc_commit(sfull);
        tc_commit(&cempty[cs]);
      };
      s_mma(0);
      for (int kb = 0; kb < nkb; ++kb) {
        if (kb + 1 < nkb) s_mma(kb + 1);
        const int db = kb & 1;
        mbar_wait(&dhfull[db], (uint32_t)((kb >> 1) & 1));
        const int s0 = slot_of(2 * kb, S::kXS), s1 = slot_of(2 * kb + 1, S::kXS);
        mbar_wait(&xfull[s0], par_of(2 * kb, S::kXS));
        mbar_wait(&xfull[s1], par_of(2 * kb + 1, S::kXS));
        tc_fence_after();
        const uint32_t dh = smem_u32(sDH + db * 32768);
#pragma unroll
        for (int k = 0; k < BM / 16; ++k) {
          const uint32_t xs = smem_u32(sX + (k < 4 ? s0 : s1) * S::kXB) + (k & 3) * 2048;
          const uint64_t ad = umma_desc_sw128(dh + k * 2048, 16384, 1024);
          const uint32_t acc = (kb | k) != 0;
          tc_mma_f16(tmem_base + 128, ad, umma_desc_sw128(xs, 8192, 1024), idW, acc);
          tc_mma_f16(tmem_base + 384, ad, umma_desc_sw128(ones + (k & 3) * 2048, 8192, 1024), idB, acc);
          if (k == 3) tc_commit(&xempty[s0]);
        }
        tc_commit(&xempty[s1]);
        tc_commit(&dhempty[db]);
      }
      tc_commit(accfull);
    }
  } else if (warp >= 4) {
    const int q = warp & 3;
    const int par = (warp - 4) >> 2;
    const int f0 = c * CH + par * 64;
    for (int kb = 0; kb < nkb; ++kb) {
      const int row = row_lo + kb * BM + 32 * q + lane;
      const uint32_t m0 = __ldg(&a.bits[(size_t)(f0 >> 5) * a.bits_ld + row]);
      const uint32_t m1 = __ldg(&a.bits[(size_t)((f0 >> 5) + 1) * a.bits_ld + row]);
      mbar_wait(sfull, (uint32_t)(kb & 1));
      tc_fence_after();
      uint32_t t0[32], t1[32];
      const uint32_t ta = tmem_base + ((uint32_t)(32 * q) << 16) + par * 64;
      tmem_ld32(ta, t0);
      tmem_ld32(ta + 32, t1);
      tmem_ld_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(sempty);
      const int db = kb & 1;
      mbar_wait(&dhempty[db], (uint32_t)(((kb >> 1) & 1) ^ 1));
      uint8_t* hrow = sDH + db * 32768 + par * 16384 + (32 * q + lane) * 128;
#pragma unroll
      for (int cc = 0; cc < 8; ++cc) {
        float v[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int j = cc * 8 + i;
          const uint32_t w = j < 32 ? m0 : m1;
          const uint32_t raw = j < 32 ? t0[j] : t1[j - 32];
          v[i] = ((w >> (j & 31)) & 1u) ? __uint_as_float(raw) : 0.f;
        }
        const uint4 pk = make_uint4(pack_bf16(v[0], v[1]), pack_bf16(v[2], v[3]), pack_bf16(v[4], v[5]),
                                    pack_bf16(v[6], v[7]));
        *reinterpret_cast<uint4*>(hrow + ((cc ^ (lane & 7)) << 4)) = pk;
      }
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(&dhfull[db]);
    }
    // dW1 rows f = c*128 + 32q + lane, columns split by parity; db from the ones product
    const int f = c * CH + 32 * q + lane;
    float* dwrow = a.dW + ((size_t)e * a.d_ff + f) * D;
    if (nkb > 0) {
      mbar_wait(accfull, 0);
      tc_fence_after();
    }
#pragma unroll
    for (int cc = 0; cc < DK; ++cc) {
      const int col = par * (D / 2) + cc * 32;
      if (cc * 32 >= D / 2) break;
      uint32_t t0[32];
      if (nkb > 0) {
        tmem_ld32(tmem_base + ((uint32_t)(32 * q) << 16) + 128 + col, t0);
        tmem_ld_wait();
      } else {
#pragma unroll
        for (int j = 0; j < 32; ++j) t0[j] = 0u;
      }
#pragma unroll
      for (int j = 0; j < 32; j += 4)
        *reinterpret_cast<float4*>(dwrow + col + j) = make_float4(__uint_as_float(t0[j]), __uint_as_float(t0[j + 1]),
                                                                  __uint_as_float(t0[j + 2]), __uint_as_float(t0[j + 3]));
    }
    if (par == 0) {
      float bsum = 0.f;
      if (nkb > 0) {
        uint32_t t0[32];
        tmem_ld32(tmem_base + ((uint32_t)(32 * q) << 16) + 384, t0);
        tmem_ld_wait();
        bsum = __uint_as_float(t0[0]);
      }
      a.db[(size_t)e * a.d_ff + f] = bsum;
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_dealloc(tmem_base, 512);
}

}  // namespace mlp

// ---------------------------------------------------------------- host side
typedef CUresult (*EncodeTiledFn2)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn2 encode_fn() {
  static EncodeTiledFn2 fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn2>(p);
  }
  return fn;
}

// bf16 tensor map, SW128; dims innermost first
static int bf16_map(CUtensorMap* m, int rank, const void* ptr, const uint64_t* dims, const uint64_t* strides_bytes,
                    const uint32_t* box) {
  EncodeTiledFn2 enc = encode_fn();
  if (!enc) return set_error(SMES_ERR_CUDA, "cuTensorMapEncodeTiled unavailable (no CUDA driver?)");
  cuuint64_t d[3], s[2];
  cuuint32_t b[3], e[3] = {1, 1, 1};
  for (int i = 0; i < rank; ++i) { d[i] = dims[i]; b[i] = box[i]; }
  for (int i = 0; i < rank - 1; ++i) s[i] = strides_bytes[i];
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, rank, const_cast<void*>(ptr), d, s, b, e,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return set_error(SMES_ERR_CUDA, "cuTensorMapEncodeTiled failed (code %d)", (int)r);
  return SMES_OK;
}

static int sm_count() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

// CTA-pair kernels: as many pairs as can be co-resident (GPC boundaries can leave an SM of a
// pair unusable -- a grid of sm_count() CTAs would then run some pairs as a second wave).
template <typename K>
static int pair_grid(K kernel, int smem) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(sm_count() & ~1);
  cfg.blockDim = dim3(mlp::kThreads);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2; attr[0].val.clusterDim.y = 1; attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int nc = 0;
  if (cudaOccupancyMaxActiveClusters(&nc, (void*)kernel, &cfg) != cudaSuccess || nc <= 0) {
    cudaGetLastError();
    return sm_count() & ~1;
  }
  return 2 * std::min(nc, sm_count() / 2);
}
#ifdef SMES_TRACE
extern "C" int smes_debug_trace(void* host_out, int clear) {
  if (clear == 3) {
    auto k = smes::mlp::mlp_fwd2_kernel<4>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smes::mlp::Fwd2Smem<4>::kBytes);
    return pair_grid(k, smes::mlp::Fwd2Smem<4>::kBytes);
  }
  static unsigned long long z[148 * 16];
  if (clear == 2) return (int)cudaMemcpyFromSymbol(host_out, smes::mlp::g_ev, sizeof(long long) * 4 * 12 * 64);
  if (clear) return (int)cudaMemcpyToSymbol(smes::mlp::g_trace, z, sizeof(z));
  return (int)cudaMemcpyFromSymbol(host_out, smes::mlp::g_trace, sizeof(z));
}
#endif

}  // namespace smes

using namespace smes;

extern "C" {

static int mlp_fwd_impl(const void* X, long ldx, long rows_cap, const int* gather, long n_src, const void* W1,
                        const float* b1, const void* G, const float* c, int ldg, int E, int d, int d_ff,
                        const int* seg, uint32_t* bits, long bits_ld, void* H, long ldh, float* P, long ldp,
                        void* stream, const void* pack_src = nullptr, long pack_ld = 0) {
  // pack mode: X is the packed output (written by the kernel); rows come from pack_src[gather[r]]
  const bool pack = pack_src != nullptr;
  const int* tma_gather = pack ? nullptr : gather;
  if (E < 1 || E > 256) return set_error(SMES_ERR_SHAPE, "mlp_fwd: expert count %d outside [1, 256]", E);
  if (d % 64 || d < 64 || d > 512) return set_error(SMES_ERR_SHAPE, "mlp_fwd: d=%d must be a multiple of 64 in [64, 512]", d);
  if (d_ff % 128 || d_ff < 128) return set_error(SMES_ERR_SHAPE, "mlp_fwd: d_ff=%d must be a multiple of 128", d_ff);
  if (ldg < 1 || ldg > 16 || ldp > 16 || ldp % 4 || ldp > ldg)
    return set_error(SMES_ERR_SHAPE, "mlp_fwd: ldg=%d ldp=%ld (need ldp <= ldg <= 16, ldp %% 4 == 0)", ldg, ldp);
  if ((ldx * 2) % 16 || (ldh * 2) % 16) return set_error(SMES_ERR_SHAPE, "mlp_fwd: row strides must be 16-byte aligned");
  CUtensorMap tx, tw, tg, th;
  int rc;
  {
    // gathered: X is the source ((n_src, ldx) rows), one row per box (4 per gather4 op)
    uint64_t dims[2] = {(uint64_t)d, (uint64_t)(tma_gather ? n_src : rows_cap)}, str[1] = {(uint64_t)ldx * 2};
    uint32_t box[2] = {64, tma_gather ? 1u : 128u};
    if ((rc = bf16_map(&tx, 2, X, dims, str, box))) return rc;
  }
  {
    uint64_t dims[3] = {(uint64_t)d, (uint64_t)d_ff, (uint64_t)E};
    uint64_t str[2] = {(uint64_t)d * 2, (uint64_t)d_ff * d * 2};
    uint32_t box[3] = {64, 128, 1};
    if ((rc = bf16_map(&tw, 3, W1, dims, str, box))) return rc;
  }
  {
    uint64_t dims[3] = {(uint64_t)d_ff, (uint64_t)ldg, (uint64_t)E};
    uint64_t str[2] = {(uint64_t)d_ff * 2, (uint64_t)ldg * d_ff * 2};
    uint32_t box[3] = {64, 16, 1};
    if ((rc = bf16_map(&tg, 3, G, dims, str, box))) return rc;
  }
  {
    const void* hp = H != nullptr ? H : X;     // map unused when H is not stored
    uint64_t dims[2] = {(uint64_t)d_ff, (uint64_t)rows_cap}, str[1] = {(uint64_t)(H != nullptr ? ldh : ldx) * 2};
    uint32_t box[2] = {64, 32};
    if (H == nullptr) dims[0] = (uint64_t)d;
    if ((rc = bf16_map(&th, 2, hp, dims, str, box))) return rc;
  }
  mlp::FwdArgs args{seg, E, d, d_ff, (int)ldp, b1, c, ldg, bits, (int)bits_ld, P, H != nullptr ? 1 : 0, tma_gather,
                    reinterpret_cast<const __nv_bfloat16*>(pack_src), pack_ld};
  if (pack) args.gather = gather;   // read by the gather warp (tma_gather stays off: no gather4 ops)
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  cudaError_t e;
#define SMES_FWD_CASE(DK)                                                                              \
  case DK: {                                                                                           \
    auto k = pack ? mlp::mlp_fwd_kernel<DK, true> : mlp::mlp_fwd_kernel<DK, false>;                  \
    const int sm = mlp::FwdSmem<DK>::kBytes;                                                           \
    e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);                      \
    if (e != cudaSuccess) return set_error(SMES_ERR_CUDA, "mlp_fwd smem attribute: %s", cudaGetErrorString(e)); \
    smes_launch(k, sm_count(), mlp::kThreads, sm, st, tx, tw, tg, th, args);                                    \
    break;                                                                                             \
  }
  switch (d / 64) {
    SMES_FWD_CASE(1)
    SMES_FWD_CASE(2)
    SMES_FWD_CASE(4)
    SMES_FWD_CASE(8)
    default:
      return set_error(SMES_ERR_SHAPE, "mlp_fwd: d=%d not instantiated (64, 128, 256, 512)", d);
  }
#undef SMES_FWD_CASE
  e = cudaGetLastError();
  if (e != cudaSuccess) return set_error(SMES_ERR_CUDA, "mlp_fwd launch: %s", cudaGetErrorString(e));
  return SMES_OK;
}

int smes_mlp_fwd(const void* X, long ldx, long rows_cap, const void* W1, const float* b1, const void* G,
                 const float* c, int ldg, int E, int d, int d_ff, const int* seg, uint32_t* bits, long bits_ld,
                 void* H, long ldh, float* P, long ldp, void* stream) {
  return mlp_fwd_impl(X, ldx, rows_cap, nullptr, 0, W1, b1, G, c, ldg, E, d, d_ff, seg, bits, bits_ld, H, ldh, P,
                      ldp, stream);
}

int smes_mlp_fwd_gather(const void* src, long ld_src, long n_src, const int32_t* gather, long rows_cap,
                        const void* W1, const float* b1, const void* G, const float* c, int ldg, int E, int d,
                        int d_ff, const int* seg, uint32_t* bits, long bits_ld, void* H, long ldh, float* P, long ldp,
                        void* stream) {
  if (gather == nullptr || n_src < 1) return set_error(SMES_ERR_SHAPE, "mlp_fwd_gather: empty source");
  if (reinterpret_cast<uintptr_t>(gather) % 16) return set_error(SMES_ERR_SHAPE, "mlp_fwd_gather: row table must be 16-byte aligned");
  return mlp_fwd_impl(src, ld_src, rows_cap, gather, n_src, W1, b1, G, c, ldg, E, d, d_ff, seg, bits, bits_ld, H,
                      ldh, P, ldp, stream);
}

int smes_mlp_fwd_pack(const void* src, long ld_src, const int32_t* gather, void* X, long ldx, long rows_cap,
                      const void* W1, const float* b1, const void* G, const float* c, int ldg, int E, int d, int d_ff,
                      const int* seg, uint32_t* bits, long bits_ld, void* H, long ldh, float* P, long ldp,
                      void* stream) {
  if (src == nullptr || gather == nullptr || X == nullptr) return set_error(SMES_ERR_SHAPE, "mlp_fwd_pack: null operand");
  if (reinterpret_cast<uintptr_t>(gather) % 16 || (ld_src * 2) % 16 || reinterpret_cast<uintptr_t>(src) % 16)
    return set_error(SMES_ERR_SHAPE, "mlp_fwd_pack: row table and source rows must be 16-byte aligned");
  return mlp_fwd_impl(X, ldx, rows_cap, gather, 0, W1, b1, G, c, ldg, E, d, d_ff, seg, bits, bits_ld, H, ldh, P, ldp,
                      stream, src, ld_src);
}

int smes_mlp_fwd2(const void* X, long ldx, long rows_cap, const void* W1, const float* b1, const void* G,
                 const float* c, int ldg, int E, int d, int d_ff, const int* seg, uint32_t* bits, long bits_ld,
                 void* H, long ldh, float* P, long ldp, void* stream) {
  if (E < 1 || E > 256) return set_error(SMES_ERR_SHAPE, "mlp_fwd2: expert count %d outside [1, 256]", E);
  if (d % 64 || d < 64 || d > 512) return set_error(SMES_ERR_SHAPE, "mlp_fwd2: d=%d must be a multiple of 64 in [64, 512]", d);
  if (d_ff % 128 || d_ff < 128) return set_error(SMES_ERR_SHAPE, "mlp_fwd2: d_ff=%d must be a multiple of 128", d_ff);
  if (ldg < 1 || ldg > 16 || ldp > 16 || ldp % 4 || ldp > ldg)
    return set_error(SMES_ERR_SHAPE, "mlp_fwd2: ldg=%d ldp=%ld (need ldp <= ldg <= 16, ldp %% 4 == 0)", ldg, ldp);
  if ((ldx * 2) % 16 || (ldh * 2) % 16) return set_error(SMES_ERR_SHAPE, "mlp_fwd2: row strides must be 16-byte aligned");
  CUtensorMap tx, tw, tg, th;
  int rc;
  {
    uint64_t dims[2] = {(uint64_t)d, (uint64_t)rows_cap}, str[1] = {(uint64_t)ldx * 2};
    uint32_t box[2] = {64, 128};
    if ((rc = bf16_map(&tx, 2, X, dims, str, box))) return rc;
  }
  {
    uint64_t dims[3] = {(uint64_t)d, (uint64_t)d_ff, (uint64_t)E};
    uint64_t str[2] = {(uint64_t)d * 2, (uint64_t)d_ff * d * 2};
    uint32_t box[3] = {64, 64, 1};                     // each CTA of the pair loads half of a W1 k-block
    if ((rc = bf16_map(&tw, 3, W1, dims, str, box))) return rc;
  }
  {
    uint64_t dims[3] = {(uint64_t)d_ff, (uint64_t)ldg, (uint64_t)E};
    uint64_t str[2] = {(uint64_t)d_ff * 2, (uint64_t)ldg * d_ff * 2};
    uint32_t box[3] = {64, 8, 1};                      // 8 task rows per CTA (N = 16 over the pair)
    if ((rc = bf16_map(&tg, 3, G, dims, str, box))) return rc;
  }
  {
    const void* hp = H != nullptr ? H : X;     // map unused when H is not stored
    uint64_t dims[2] = {(uint64_t)d_ff, (uint64_t)rows_cap}, str[1] = {(uint64_t)(H != nullptr ? ldh : ldx) * 2};
    uint32_t box[2] = {64, 32};
    if (H == nullptr) dims[0] = (uint64_t)d;
    if ((rc = bf16_map(&th, 2, hp, dims, str, box))) return rc;
  }
  mlp::FwdArgs args{seg, E, d, d_ff, (int)ldp, b1, c, ldg, bits, (int)bits_ld, P, H != nullptr ? 1 : 0};
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  cudaError_t e;
#define SMES_FWD_CASE(DK)                                                                              \
  case DK: {                                                                                           \
    auto k = mlp::mlp_fwd2_kernel<DK>;                                                                  \
    const int sm = mlp::Fwd2Smem<DK>::kBytes;                                                           \
    e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);                      \
    if (e != cudaSuccess) return set_error(SMES_ERR_CUDA, "mlp_fwd2 smem attribute: %s", cudaGetErrorString(e)); \
    smes_launch(k, pair_grid(k, sm), mlp::kThreads, sm, st, tx, tw, tg, th, args);                                    \
    break;                                                                                             \
  }
  switch (d / 64) {
    SMES_FWD_CASE(1)
    SMES_FWD_CASE(2)
    SMES_FWD_CASE(4)
    SMES_FWD_CASE(8)
    default:
      return set_error(SMES_ERR_SHAPE, "mlp_fwd2: d=%d not instantiated (64, 128, 256, 512)", d);
  }
#undef SMES_FWD_CASE
  e = cudaGetLastError();
  if (e != cudaSuccess) return set_error(SMES_ERR_CUDA, "mlp_fwd2 launch: %s", cudaGetErrorString(e));
  return SMES_OK;
}

int smes_mlp_dgrad(const void* C, long ldc, long rows_cap, const void* G, int ldg, const void* W1, int E, int d,
                   int d_ff, const int* seg, const uint32_t* bits, long bits_ld, void* dX, long lddx, void* dH,
                   long lddh, void* stream) {
  if (E < 1 || E > 256) return set_error(SMES_ERR_SHAPE, "mlp_dgrad: expert count %d outside [1, 256]", E);
  if (d % 64 || d < 64 || d > 256) return set_error(SMES_ERR_SHAPE, "mlp_dgrad: d=%d must be a multiple of 64 in [64, 256]", d);
  if (d_ff % 128 || d_ff < 128) return set_error(SMES_ERR_SHAPE, "mlp_dgrad: d_ff=%d must be a multiple of 128", d_ff);
  if (ldg < 1 || ldg > 16 || ldc < ldg || (ldc * 2) % 16 || (lddx * 2) % 16)
    return set_error(SMES_ERR_SHAPE, "mlp_dgrad: ldg=%d ldc=%ld lddx=%ld", ldg, ldc, lddx);
  CUtensorMap tc, tg, tw, td, th;
  int rc;
  {
    uint64_t dims[2] = {(uint64_t)ldg, (uint64_t)rows_cap}, str[1] = {(uint64_t)ldc * 2};
    uint32_t box[2] = {64, 128};
    if ((rc = bf16_map(&tc, 2, C, dims, str, box))) return rc;
  }
  {
    uint64_t dims[3] = {(uint64_t)d_ff, (uint64_t)ldg, (uint64_t)E};
    uint64_t str[2] = {(uint64_t)d_ff * 2, (uint64_t)ldg * d_ff * 2};
    uint32_t box[3] = {64, 16, 1};
    if ((rc = bf16_map(&tg, 3, G, dims, str, box))) return rc;
  }
  {
    uint64_t dims[3] = {(uint64_t)d, (uint64_t)d_ff, (uint64_t)E};    // W1 (E, d_ff, d): element (j, f)
    uint64_t str[2] = {(uint64_t)d * 2, (uint64_t)d_ff * d * 2};
    uint32_t box[3] = {64, 64, 1};
    if ((rc = bf16_map(&tw, 3, W1, dims, str, box))) return rc;
  }
  {
    uint64_t dims[2] = {(uint64_t)d, (uint64_t)rows_cap}, str[1] = {(uint64_t)lddx * 2};
    uint32_t box[2] = {64, 32};
    if ((rc = bf16_map(&td, 2, dX, dims, str, box))) return rc;
  }
  {
    if (dH != nullptr && (lddh * 2) % 16) return set_error(SMES_ERR_SHAPE, "mlp_dgrad: dH stride must be 16-byte aligned");
    uint64_t dims[2] = {(uint64_t)(dH ? d_ff : d), (uint64_t)rows_cap}, str[1] = {(uint64_t)(dH ? lddh : lddx) * 2};
    uint32_t box[2] = {64, 32};
    if ((rc = bf16_map(&th, 2, dH ? dH : dX, dims, str, box))) return rc;
  }
  mlp::DgradArgs args{seg, E, d, d_ff, bits, (int)bits_ld, dH != nullptr ? 1 : 0};
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  cudaError_t e;
#define SMES_DG_CASE(DK)                                                                               \
  case DK: {                                                                                           \
    auto k = mlp::mlp_dgrad_kernel<DK>;                                                                \
    const int sm = mlp::DgSmem<DK>::kBytes;                                                            \
    e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);                      \
    if (e != cudaSuccess) return set_error(SMES_ERR_CUDA, "mlp_dgrad smem attribute: %s", cudaGetErrorString(e)); \
    smes_launch(k, sm_count(), mlp::kThreads, sm, st, tc, tg, tw, td, th, args);                                   \
    break;                                                                                             \
  }
  switch (d / 64) {
    SMES_DG_CASE(1)
    SMES_DG_CASE(2)
    SMES_DG_CASE(4)
    default:
      return set_error(SMES_ERR_SHAPE, "mlp_dgrad: d=%d not instantiated (64, 128, 256)", d);
  }
#undef SMES_DG_CASE
  e = cudaGetLastError();
  if (e != cudaSuccess) return set_error(SMES_ERR_CUDA, "mlp_dgrad launch: %s", cudaGetErrorString(e));
  return SMES_OK;
}

int smes_mlp_dgrad2(const void* C, long ldc, long rows_cap, const void* G, int ldg, const void* W1, int E, int d,
                   int d_ff, const int* seg, const uint32_t* bits, long bits_ld, void* dX, long lddx, void* dH,
                   long lddh, void* stream) {
  if (E < 1 || E > 256) return set_error(SMES_ERR_SHAPE, "mlp_dgrad2: expert count %d outside [1, 256]", E);
  if (d % 64 || d < 64 || d > 256) return set_error(SMES_ERR_SHAPE, "mlp_dgrad2: d=%d must be a multiple of 64 in [64, 256]", d);
  if (d_ff % 128 || d_ff < 128) return set_error(SMES_ERR_SHAPE, "mlp_dgrad2: d_ff=%d must be a multiple of 128", d_ff);
  if (ldg < 1 || ldg > 16 || ldc < ldg || (ldc * 2) % 16 || (lddx * 2) % 16)
    return set_error(SMES_ERR_SHAPE, "mlp_dgrad2: ldg=%d ldc=%ld lddx=%ld", ldg, ldc, lddx);
  CUtensorMap tc, tg, tw, td, th;
  int rc;
  {
    uint64_t dims[2] = {(uint64_t)ldg, (uint64_t)rows_cap}, str[1] = {(uint64_t)ldc * 2};
    uint32_t box[2] = {64, 128};
    if ((rc = bf16_map(&tc, 2, C, dims, str, box))) return rc;
  }
  {
    uint64_t dims[3] = {(uint64_t)d_ff, (uint64_t)ldg, (uint64_t)E};
    uint64_t str[2] = {(uint64_t)d_ff * 2, (uint64_t)ldg * d_ff * 2};
    uint32_t box[3] = {64, 16, 1};                     // each CTA: one 64-wide f half of the chunk
    if ((rc = bf16_map(&tg, 3, G, dims, str, box))) return rc;
  }
  {
    uint64_t dims[3] = {(uint64_t)d, (uint64_t)d_ff, (uint64_t)E};    // W1 (E, d_ff, d): element (j, f)
    uint64_t str[2] = {(uint64_t)d * 2, (uint64_t)d_ff * d * 2};
    uint32_t box[3] = {64, 64, 1};
    if ((rc = bf16_map(&tw, 3, W1, dims, str, box))) return rc;
  }
  {
    uint64_t dims[2] = {(uint64_t)d, (uint64_t)rows_cap}, str[1] = {(uint64_t)lddx * 2};
    uint32_t box[2] = {64, 32};
    if ((rc = bf16_map(&td, 2, dX, dims, str, box))) return rc;
  }
  {
    if (dH != nullptr && (lddh * 2) % 16) return set_error(SMES_ERR_SHAPE, "mlp_dgrad2: dH stride must be 16-byte aligned");
    uint64_t dims[2] = {(uint64_t)(dH ? d_ff : d), (uint64_t)rows_cap}, str[1] = {(uint64_t)(dH ? lddh : lddx) * 2};
    uint32_t box[2] = {64, 32};
    if ((rc = bf16_map(&th, 2, dH ? dH : dX, dims, str, box))) return rc;
  }
  mlp::DgradArgs args{seg, E, d, d_ff, bits, (int)bits_ld, dH != nullptr ? 1 : 0};
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  cudaError_t e;
#define SMES_DG_CASE(DK)                                                                               \
  case DK: {                                                                                           \
    auto k = mlp::mlp_dgrad2_kernel<DK>;                                                                \
    const int sm = mlp::Dg2Smem<DK>::kBytes;                                                            \
    e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);                      \
    if (e != cudaSuccess) return set_error(SMES_ERR_CUDA, "mlp_dgrad2 smem attribute: %s", cudaGetErrorString(e)); \
    smes_launch(k, pair_grid(k, sm), mlp::kThreads, sm, st, tc, tg, tw, td, th, args);                                   \
    break;                                                                                             \
  }
  switch (d / 64) {
    SMES_DG_CASE(2)
    SMES_DG_CASE(4)
    default:
      return set_error(SMES_ERR_SHAPE, "mlp_dgrad2: d=%d not instantiated (128, 256)", d);
  }
#undef SMES_DG_CASE
  e = cudaGetLastError();
  if (e != cudaSuccess) return set_error(SMES_ERR_CUDA, "mlp_dgrad2 launch: %s", cudaGetErrorString(e));
  return SMES_OK;
}


int smes_mlp_wgrad(const void* C, long ldc, long rows_cap, const void* G, int ldg, const void* X, long ldx, int E, int d,
                   int d_ff, const int* seg, const uint32_t* bits, long bits_ld, float* dW, float* db, void* stream) {
  if (E < 1 || E > 256) return set_error(SMES_ERR_SHAPE, "mlp_wgrad: expert count %d outside [1, 256]", E);
  if (d % 64 || d < 64 || d > 256) return set_error(SMES_ERR_SHAPE, "mlp_wgrad: d=%d must be a multiple of 64 in [64, 256]", d);
  if (d_ff % 128 || d_ff < 128) return set_error(SMES_ERR_SHAPE, "mlp_wgrad: d_ff=%d must be a multiple of 128", d_ff);
  if (ldg < 1 || ldg > 16 || ldc < ldg || (ldc * 2) % 16 || (ldx * 2) % 16)
    return set_error(SMES_ERR_SHAPE, "mlp_wgrad: ldg=%d ldc=%ld ldx=%ld", ldg, ldc, ldx);
  CUtensorMap tc, tg, tx;
  int rc;
  {
    uint64_t dims[2] = {(uint64_t)ldg, (uint64_t)rows_cap}, str[1] = {(uint64_t)ldc * 2};
    uint32_t box[2] = {64, 128};
    if ((rc = bf16_map(&tc, 2, C, dims, str, box))) return rc;
  }
  {
    uint64_t dims[3] = {(uint64_t)d_ff, (uint64_t)ldg, (uint64_t)E};
    uint64_t str[2] = {(uint64_t)d_ff * 2, (uint64_t)ldg * d_ff * 2};
    uint32_t box[3] = {64, 16, 1};
    if ((rc = bf16_map(&tg, 3, G, dims, str, box))) return rc;
  }
  {
    uint64_t dims[2] = {(uint64_t)d, (uint64_t)rows_cap}, str[1] = {(uint64_t)ldx * 2};
    uint32_t box[2] = {64, 64};
    if ((rc = bf16_map(&tx, 2, X, dims, str, box))) return rc;
  }
  mlp::WgradArgs args{seg, E, d, d_ff, bits, (int)bits_ld, dW, db};
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  cudaError_t e;
  const int grid = E * (d_ff / mlp::CH);
#define SMES_WG_CASE(DK)                                                                               \
  case DK: {                                                                                           \
    auto k = mlp::mlp_wgrad_kernel<DK>;                                                                \
    const int sm = mlp::WgSmem<DK>::kBytes;                                                            \
    e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);                      \
    if (e != cudaSuccess) return set_error(SMES_ERR_CUDA, "mlp_wgrad smem attribute: %s", cudaGetErrorString(e)); \
    smes_launch(k, grid, mlp::kThreads, sm, st, tc, tg, tx, args);                                              \
    break;                                                                                             \
  }
  switch (d / 64) {
    SMES_WG_CASE(1)
    SMES_WG_CASE(2)
    SMES_WG_CASE(4)
    default:
      return set_error(SMES_ERR_SHAPE, "mlp_wgrad: d=%d not instantiated (64, 128, 256)", d);
  }
#undef SMES_WG_CASE
  e = cudaGetLastError();
  if (e != cudaSuccess) return set_error(SMES_ERR_CUDA, "mlp_wgrad launch: %s", cudaGetErrorString(e));
  return SMES_OK;
}

}  // extern "C"
