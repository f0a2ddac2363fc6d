// Head folding for the training step.
//
// When the last expert pool is the identity (the BASELINE expert MLP 256->512->256: ReLU
// after fc1, identity after fc2), the task heads compose with it.  For a packed row r of
// expert e with last-pool input H[r] (model.py:202-208, execution.py:126-158):
//
//   P[r, t]  = <head_w_t, O[r]>            = H[r] . G_e[t] + c_e[t],
//   G_e      = head_w W_e   (T x d_in),      c_e = head_w b_e,
//
// and the backward of the combine + heads (training.py:146-191) is rank T per row:
//   d_packed[r] = sum_t C[r, t] head_w_t,    C[r, t] = sum_{(b,k) -> r} w[t,b,k] dlogit[t,b]
//   dH[r]       = C[r] G_e  (then the previous pool's ReLU mask),
//   dW_e        = head_w^T Q_e,   Q_e = C_e^T H_e  (T x d_in, summed over the rows of e; layout (E, ldg, d_in)),
//   db_e        = head_w^T csum_e,   csum_e[t] = sum_{r in e} C[r, t],
//   dW_head     = sum_e (Q_e W_e^T + csum_e b_e^T).
//
// So the training step never materialises O (N_act x d_out) or d_packed: the last pool's
// forward becomes an N = T GEMM on H, its dgrad a K = T GEMM, and its weight gradient a
// T x d_in reduction.  The algebra is exact; only the fp32 summation order differs.
// These kernels build G/c from the weights (every step) and expand Q into dW, db, dW_head.
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "ptx.cuh"
#include "fold_full.cuh"
#include "smes_capi.h"

namespace smes {

// The two T-row contractions over an expert's weight tile run as split-K CUDA-core tile
// kernels: each block loads ONE 64x64 bf16 tile of W_e (one memory latency, 128-byte rows) plus
// the matching T x 64 fp32 slice of the other operand, and writes a T x 64 fp32 partial; a
// fixed-order reduction over the splits (and experts) finishes the job.  Deterministic.
//   FOLD   : part[s, e, t, k] = sum_{j in split s} head_w[t, j] W[e, j, k]     (tile rows j, cols k)
//   UNFOLD : part[s, e, t, j] = sum_{k in split s} Q[e, t, k]  W[e, j, k]      (tile rows j, cols k)
enum { TILE_FOLD = 0, TILE_UNFOLD = 1 };

template <int TM, int MODE>
__device__ __forceinline__ void fold_tile_body(int bx, int by, int bz, int gy, int T, int ldg, int d_out, int d_in,
                                               const float* __restrict__ head_w, const float* __restrict__ Qt,
                                               long q_es, long q_ts, long q_ks, const __nv_bfloat16* __restrict__ W,
                                               float* __restrict__ part) {
  __shared__ float sW[64][65];      // [r][c] (FOLD: r = j, c = k) / [c][r] transposed (UNFOLD: c = j, r = k)
  __shared__ float sX[TM][64];      // [t][r]
  const int e = by;
  const int c0 = bx * 64;           // output column tile (FOLD: k, UNFOLD: j)
  const int r0 = bz * 64;           // reduction split     (FOLD: j, UNFOLD: k)
  const int nr = MODE == TILE_FOLD ? d_out : d_in;
  const int nc = MODE == TILE_FOLD ? d_in : d_out;
  const __nv_bfloat16* We = W + (size_t)e * d_out * d_in;
  // W tile: 64 rows x 64 cols bf16 = 8 KB; thread loads 4 x 16 B (8 bf16 each)
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int idx = threadIdx.x + 128 * u;        // 0..511: row = idx / 8, 8-col group = idx % 8
    const int row = idx >> 3, cg = (idx & 7) * 8;
    // FOLD: W rows are j (= reduction r), cols k (= output c);  UNFOLD: W rows are j (= output c), cols k (= r)
    const int wr = MODE == TILE_FOLD ? r0 + row : c0 + row;
    const int wc = MODE == TILE_FOLD ? c0 + cg : r0 + cg;
    uint4 v = make_uint4(0, 0, 0, 0);
    if (wr < d_out && wc < d_in) v = *reinterpret_cast<const uint4*>(We + (size_t)wr * d_in + wc);
    const __nv_bfloat16* hv = reinterpret_cast<const __nv_bfloat16*>(&v);
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const float f = __bfloat162float(hv[q]);
      if (MODE == TILE_FOLD) sW[row][cg + q] = f; else sW[cg + q][row] = f;   // sW[r][c]
    }
  }
  for (int i = threadIdx.x; i < TM * 64; i += 128) {
    const int t = i >> 6, r = i & 63;
    float x = 0.f;
    if (t < T && r0 + r < nr)
      x = MODE == TILE_FOLD ? head_w[(size_t)t * d_out + r0 + r] : Qt[(size_t)e * q_es + (size_t)t * q_ts + (size_t)(r0 + r) * q_ks];
    sX[t][r] = x;
  }
  __syncthreads();
  const int c = threadIdx.x & 63;
  const int th = threadIdx.x >> 6;          // task half
  constexpr int TH = TM / 2;
  float acc[TH];
#pragma unroll
  for (int i = 0; i < TH; ++i) acc[i] = 0.f;
#pragma unroll 8
  for (int r = 0; r < 64; ++r) {
    const float w = sW[r][c];
#pragma unroll
    for (int i = 0; i < TH; ++i) acc[i] = fmaf(sX[th * TH + i][r], w, acc[i]);
  }
  if (c0 + c < nc) {
    const size_t base = ((size_t)bz * gy + e) * TM;
#pragma unroll
    for (int i = 0; i < TH; ++i) part[(base + th * TH + i) * nc + c0 + c] = acc[i];
  }
}

template <int TM, int MODE>
__global__ void __launch_bounds__(128) fold_tile_kernel(int T, int ldg, int d_out, int d_in,
                                                        const float* __restrict__ head_w,
                                                        const float* __restrict__ Qt, long q_es, long q_ts,
                                                        long q_ks, const __nv_bfloat16* __restrict__ W,
                                                        float* __restrict__ part) {
  pdl_wait();
  fold_tile_body<TM, MODE>(blockIdx.x, blockIdx.y, blockIdx.z, gridDim.y, T, ldg, d_out, d_in, head_w, Qt, q_es, q_ts,
                           q_ks, W, part);
}

template <int TM>
__global__ void __launch_bounds__(256) fold_full_kernel(int T, int ldg, int d_out, int d_in,
                                                        const float* __restrict__ head_w,
                                                        const __nv_bfloat16* __restrict__ W,
                                                        const float* __restrict__ b, __nv_bfloat16* __restrict__ G,
                                                        float* __restrict__ c) {
  pdl_wait();
  extern __shared__ __align__(16) uint8_t fsm[];
  fold_full_body<TM>(blockIdx.x, blockIdx.y, T, ldg, d_out, d_in, head_w, W, b, G, c, fsm);
}

// G[e, t, k] = sum_s part[s, e, t, k] (bf16, rows >= T zero);  c[e, t] = head_w[t] . b[e]
template <int TM>
__global__ void fold_finish_kernel(int E, int T, int ldg, int d_out, int d_in, int splits,
                                   const float* __restrict__ part, const float* __restrict__ head_w,
                                   const float* __restrict__ b, __nv_bfloat16* __restrict__ G,
                                   float* __restrict__ c) {
  pdl_wait();
  const size_t n = (size_t)E * ldg * d_in;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const int k = (int)(i % d_in);
    const int t = (int)((i / d_in) % ldg);
    const int e = (int)(i / ((size_t)d_in * ldg));
    float v = 0.f;
    if (t < T)
      for (int s = 0; s < splits; ++s) v += part[(((size_t)s * E + e) * TM + t) * d_in + k];
    G[i] = __float2bfloat16_rn(v);
  }
  // c: warp per (e, t), lanes over j
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp < E * ldg) {
    const int e = warp / ldg, t = warp % ldg;
    float s = 0.f;
    if (t < T)
      for (int j = lane; j < d_out; j += 32) s = fmaf(head_w[(size_t)t * d_out + j], b[(size_t)e * d_out + j], s);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) c[(size_t)e * ldg + t] = s;
  }
}

// dW_head[t, j] = sum_e sum_s part[s, e, t, j] + sum_e csum[e, t] b[e, j]   (fixed order)
// block = (32 columns j, task t); warp w sums experts e = w, w+8, ...; then warp 0 sums the 8 warps
template <int TM>
__global__ void __launch_bounds__(256) unfold_finish_kernel(int E, int T, int d_out, int splits,
                                                            const float* __restrict__ part,
                                                            const float* __restrict__ csum, long cs_es,
                                                            const float* __restrict__ b, float* __restrict__ out) {
  pdl_wait();
  __shared__ float red[8][32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int t = blockIdx.y, j = blockIdx.x * 32 + lane;
  float acc = 0.f;
  if (j < d_out) {
    for (int e = warp; e < E; e += 8) {
      float v = csum[(size_t)e * cs_es + t] * b[(size_t)e * d_out + j];
      for (int s = 0; s < splits; ++s) v += part[(((size_t)s * E + e) * TM + t) * d_out + j];
      acc += v;
    }
  }
  red[warp][lane] = acc;
  __syncthreads();
  if (warp == 0 && j < d_out) {
    float v = 0.f;
#pragma unroll
    for (int w = 0; w < 8; ++w) v += red[w][lane];
    out[(size_t)t * d_out + j] = v;
  }
}

// dW[e, j, k] = sum_t head_w[t, j] Q[e, t, k];  db[e, j] = sum_t head_w[t, j] csum[e, t]
template <int TM>
__device__ __forceinline__ void unfold_dw_body(int bx, int by, int bz, int T, int ldg, int d_out, int d_in,
                                               const float* __restrict__ Qt, long q_es, long q_ts, long q_ks,
                                               const float* __restrict__ csum, long cs_es,
                                               const float* __restrict__ head_w, float* __restrict__ dW,
                                               float* __restrict__ db) {
  __shared__ float sw[TM][32];
  const int e = bz;
  const int j0 = by * 32;
  const int k = bx * 128 + threadIdx.x;
  for (int i = threadIdx.x; i < TM * 32; i += 128) {
    const int t = i >> 5, j = j0 + (i & 31);
    sw[t][i & 31] = (t < T && j < d_out) ? head_w[(size_t)t * d_out + j] : 0.f;
  }
  __syncthreads();
  if (k < d_in) {
    float q[TM];
    const float* qp = Qt + (size_t)e * q_es + (size_t)k * q_ks;
#pragma unroll
    for (int t = 0; t < TM; ++t) q[t] = t < T ? qp[(size_t)t * q_ts] : 0.f;
    const int jn = min(32, d_out - j0);
    for (int jj = 0; jj < jn; ++jj) {
      float s = 0.f;
#pragma unroll
      for (int t = 0; t < TM; ++t) s = fmaf(sw[t][jj], q[t], s);
      dW[((size_t)e * d_out + j0 + jj) * d_in + k] = s;
    }
  }
  if (bx == 0 && threadIdx.x < 32 && j0 + threadIdx.x < d_out) {
    float s = 0.f;
    for (int t = 0; t < T; ++t) s = fmaf(sw[t][threadIdx.x], csum[(size_t)e * cs_es + t], s);
    db[(size_t)e * d_out + j0 + threadIdx.x] = s;
  }
}

// dW/db (unfold_dw_body) and the split partials of Y = Q W^T (fold_tile_body, UNFOLD) in one
// launch: blocks [0, n1) take the first job, the rest the second -- one launch gap less per step
template <int TM>
__global__ void __launch_bounds__(128) unfold_pair_kernel(int E, int T, int ldg, int d_out, int d_in,
                                                          const float* __restrict__ Qt, long q_es, long q_ts,
                                                          long q_ks, const float* __restrict__ csum, long cs_es,
                                                          const float* __restrict__ head_w,
                                                          const __nv_bfloat16* __restrict__ W, float* __restrict__ dW,
                                                          float* __restrict__ db, float* __restrict__ part) {
  pdl_wait();
  const int g1x = (d_in + 127) / 128, g1y = (d_out + 31) / 32, n1 = g1x * g1y * E;
  const int bid = blockIdx.x;
  if (bid < n1) {
    unfold_dw_body<TM>(bid % g1x, (bid / g1x) % g1y, bid / (g1x * g1y), T, ldg, d_out, d_in, Qt, q_es, q_ts, q_ks,
                       csum, cs_es, head_w, dW, db);
  } else {
    const int r = bid - n1, g2x = (d_out + 63) / 64;
    fold_tile_body<TM, TILE_UNFOLD>(r % g2x, (r / g2x) % E, r / (g2x * E), E, T, ldg, d_out, d_in, nullptr, Qt, q_es,
                                    q_ts, q_ks, W, part);
  }
}

// ---------------------------------------------------------------- tensor-core path (large E*d_out*d_in)
// The same algebra as grouped GEMMs (csrc/gemm.cu):
//   G_e   = head_w W_e       : ragged-K over the rows j of W_e, P = head_w^T shared by every expert
//   dW_e  = head_w^T Q_e     : ragged-K over t (head_w and Q_e split into bf16 hi + lo rows: ~fp32 accuracy)
//   Y_e   = Q_e W_e^T        : ragged-M (K = d_in) -> dW_head = sum_e (Y_e + csum_e b_e^T)
__global__ void fold_prep_kernel(int T, int ldg, int d_out, const float* __restrict__ head_w,
                                 __nv_bfloat16* __restrict__ Pw /* (d_out, ldg) */,
                                 __nv_bfloat16* __restrict__ Wp /* (128, d_out) */) {
  pdl_wait();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (Pw != nullptr && i < d_out * ldg) {
    const int j = i / ldg, t = i % ldg;
    Pw[i] = __float2bfloat16_rn(t < T ? head_w[(size_t)t * d_out + j] : 0.f);
  }
  if (Wp != nullptr && i < 128 * d_out) {
    // rows [0,32): hi(head_w), [32,64): hi(head_w), [64,96): lo(head_w) -- paired with Q hi / lo / hi
    const int m = i / d_out, j = i % d_out;
    const int t = m & 31;
    float v = 0.f;
    if (m < 96 && t < T) {
      const float w = head_w[(size_t)t * d_out + j];
      const float hi = __bfloat162float(__float2bfloat16_rn(w));
      v = m < 64 ? hi : w - hi;
    }
    Wp[i] = __float2bfloat16_rn(v);
  }
}

__global__ void seg_arith_kernel(int n, int step, int32_t* __restrict__ seg) {
  pdl_wait();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i <= n) seg[i] = i * step;
}

// G (bf16) from the fp32 GEMM output; c[e, t] = head_w[t] . b[e]
__global__ void fold_convert_kernel(int E, int T, int ldg, int d_out, int d_in, const float* __restrict__ Gf,
                                    const float* __restrict__ head_w, const float* __restrict__ b,
                                    __nv_bfloat16* __restrict__ G, float* __restrict__ c) {
  pdl_wait();
  const size_t n = (size_t)E * ldg * d_in;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    G[i] = __float2bfloat16_rn(Gf[i]);
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp < E * ldg) {
    const int e = warp / ldg, t = warp % ldg;
    float s = 0.f;
    if (t < T)
      for (int j = lane; j < d_out; j += 32) s = fmaf(head_w[(size_t)t * d_out + j], b[(size_t)e * d_out + j], s);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) c[(size_t)e * ldg + t] = s;
  }
}

// Qbf[e][m] (128 rows per expert): rows t and 64 + t hold bf16(Q), rows 32 + t the bf16 remainder, so
// sum_m Wp[m] Qbf[m] = hi(w) hi(q) + hi(w) lo(q) + lo(w) hi(q) (~fp32 accurate); Y uses rows t, 32 + t
__global__ void unfold_split_kernel(int E, int T, int d_in, const float* __restrict__ Q, long q_es, long q_ts,
                                    long q_ks, __nv_bfloat16* __restrict__ Qbf) {
  pdl_wait();
  const size_t n = (size_t)E * 128 * d_in;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const int k = (int)(i % d_in);
    const int m = (int)((i / d_in) % 128);
    const int e = (int)(i / ((size_t)128 * d_in));
    const int t = m & 31;
    float v = 0.f;
    if (m < 96 && t < T) {
      const float q = Q[(size_t)e * q_es + (size_t)t * q_ts + (size_t)k * q_ks];
      const float hi = __bfloat162float(__float2bfloat16_rn(q));
      v = (m >= 32 && m < 64) ? q - hi : hi;
    }
    Qbf[i] = __float2bfloat16_rn(v);
  }
}

// db[e, j] = sum_t head_w[t, j] csum[e, t]
__global__ void unfold_db_kernel(int E, int T, int d_out, const float* __restrict__ csum, long cs_es,
                                 const float* __restrict__ head_w, float* __restrict__ db) {
  pdl_wait();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= E * d_out) return;
  const int e = i / d_out, j = i % d_out;
  float s = 0.f;
  for (int t = 0; t < T; ++t) s = fmaf(head_w[(size_t)t * d_out + j], csum[(size_t)e * cs_es + t], s);
  db[i] = s;
}

// dW_head[t, j] = sum_e (Y[e*128 + t, j] + Y[e*128 + 32 + t, j] + csum[e, t] b[e, j]), fixed order
__global__ void __launch_bounds__(256) unfold_head_reduce_kernel(int E, int T, int d_out, const float* __restrict__ Y,
                                                                 const float* __restrict__ csum, long cs_es,
                                                                 const float* __restrict__ b, float* __restrict__ out) {
  pdl_wait();
  __shared__ float red[8][32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int t = blockIdx.y, j = blockIdx.x * 32 + lane;
  float acc = 0.f;
  if (j < d_out)
    for (int e = warp; e < E; e += 8) {
      const float* y = Y + ((size_t)e * 128) * d_out + j;
      acc += (y[(size_t)t * d_out] + y[(size_t)(32 + t) * d_out]) + csum[(size_t)e * cs_es + t] * b[(size_t)e * d_out + j];
    }
  red[warp][lane] = acc;
  __syncthreads();
  if (warp == 0 && j < d_out) {
    float v = 0.f;
#pragma unroll
    for (int w = 0; w < 8; ++w) v += red[w][lane];
    out[(size_t)t * d_out + j] = v;
  }
}

}  // namespace smes

using namespace smes;

extern "C" {

static int fold_tm(int T) { return T <= 8 ? 8 : T <= 16 ? 16 : 32; }
static long a64(long x) { return (x + 63) / 64 * 64; }

// tensor-core path for large banks (c3/c5); the split-K CUDA-core tiles otherwise
static bool gemm_path(int E, int T, int d_out, int d_in) {
  return (long)E * d_out * d_in >= (1L << 24) && d_out % 64 == 0 && d_in % 64 == 0 && T <= 32;
}

struct FoldWork {            // offsets in floats
  long pw, seg, gf, wp, seg128, qbf, y, total;
};
static FoldWork fold_layout(int E, int T, int d_out, int d_in) {
  const int ldg = (T + 7) / 8 * 8;
  FoldWork w{};
  long o = 0;
  w.pw = o; o += a64((long)d_out * ldg / 2 + 1);
  w.seg = o; o += a64(E + 1);
  w.gf = o; o += a64((long)E * ldg * d_in);
  const long fold_end = o;
  o = 0;
  w.wp = o; o += a64((long)128 * d_out / 2);
  w.seg128 = o; o += a64(E + 1);
  w.qbf = o; o += a64((long)E * 128 * d_in / 2);
  w.y = o; o += a64((long)E * 128 * d_out);
  w.total = o > fold_end ? o : fold_end;
  return w;
}

int smes_fold_gemm_path(int E, int T, int d_out, int d_in) { return gemm_path(E, T, d_out, d_in) ? 1 : 0; }

int smes_fold_full_supported(int E, int T, int ldg, int d_out, int d_in) {
  return !gemm_path(E, T, d_out, d_in) && d_out <= FOLD_FULL_MAX_DOUT && T >= 1 && T <= 8 && ldg <= 8 && ldg >= T &&
         d_in % 8 == 0 && E >= 1;
}

int smes_fold_work_floats(int E, int T, int d_out, int d_in) {
  const int tm = fold_tm(T);
  const long a = (long)((d_out + 63) / 64) * E * tm * d_in;       // fold partials (CUDA-core path)
  const long b = (long)((d_in + 63) / 64) * E * tm * d_out;       // unfold partials
  long m = a > b ? a : b;
  if (gemm_path(E, T, d_out, d_in)) {
    const long g = fold_layout(E, T, d_out, d_in).total;
    m = g > m ? g : m;
  }
  return (int)m;
}

int smes_fold_heads(int E, int T, int ldg, int d_out, int d_in, const float* head_w, const void* W, const float* b,
                    void* G, float* c, float* work, void* stream) {
  if (T < 1 || T > 32 || ldg < T || ldg > 128) return set_error(SMES_ERR_SHAPE, "fold_heads: T=%d ldg=%d", T, ldg);
  if (E < 1 || d_out < 1 || d_in < 1 || d_in % 8) return set_error(SMES_ERR_SHAPE, "fold_heads: bad shape");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  auto Wb = reinterpret_cast<const __nv_bfloat16*>(W);
  auto Gb = reinterpret_cast<__nv_bfloat16*>(G);
  if (gemm_path(E, T, d_out, d_in) && ldg == (T + 7) / 8 * 8) {
    const FoldWork w = fold_layout(E, T, d_out, d_in);
    auto* Pw = reinterpret_cast<__nv_bfloat16*>(work + w.pw);
    auto* seg = reinterpret_cast<int32_t*>(work + w.seg);
    float* Gf = work + w.gf;
    smes_launch(fold_prep_kernel, (d_out * ldg + 255) / 256, 256, 0, st, T, ldg, d_out, head_w, Pw, nullptr);
    smes_launch(seg_arith_kernel, (E + 256) / 256, 256, 0, st, E, d_out, seg);
    int rc = smes_gemm_ragged_k_periodic(Pw, ldg, d_out, W, d_in, (long)E * d_out, E, ldg, d_in, seg, Gf, nullptr,
                                         d_out, stream);
    if (rc) return rc;
    const long n = (long)E * ldg * d_in;
    const long blocks = (n + 255) / 256 < 4096 ? (n + 255) / 256 : 4096;
    const long need = ((long)E * ldg * 32 + 255) / 256;
    smes_launch(fold_convert_kernel, (int)(blocks > need ? blocks : need), 256, 0, st, E, T, ldg, d_out, d_in, Gf, head_w, b,
                                                                               Gb, c);
  } else if (d_out <= FOLD_FULL_MAX_DOUT && T <= 8 && ldg <= 8) {
    smes_launch(fold_full_kernel<8>, dim3((d_in + 63) / 64, E), 256, fold_full_smem_bytes<8>(), st, T, ldg, d_out, d_in,
                head_w, Wb, b, Gb, c);
  } else {
    const int splits = (d_out + 63) / 64;
    dim3 grid((d_in + 63) / 64, E, splits);
    const int nfin = (int)(((long)E * ldg * d_in + 255) / 256);
    const int nfin_c = (E * ldg * 32 + 255) / 256;
    const int gfin = nfin > nfin_c ? nfin : nfin_c;
    switch (fold_tm(T)) {
      case 8:
        smes_launch(fold_tile_kernel<8, TILE_FOLD>, grid, 128, 0, st, T, ldg, d_out, d_in, head_w, nullptr, 0, 0, 0, Wb, work);
        smes_launch(fold_finish_kernel<8>, gfin, 256, 0, st, E, T, ldg, d_out, d_in, splits, work, head_w, b, Gb, c);
        break;
      case 16:
        smes_launch(fold_tile_kernel<16, TILE_FOLD>, grid, 128, 0, st, T, ldg, d_out, d_in, head_w, nullptr, 0, 0, 0, Wb, work);
        smes_launch(fold_finish_kernel<16>, gfin, 256, 0, st, E, T, ldg, d_out, d_in, splits, work, head_w, b, Gb, c);
        break;
      default:
        smes_launch(fold_tile_kernel<32, TILE_FOLD>, grid, 128, 0, st, T, ldg, d_out, d_in, head_w, nullptr, 0, 0, 0, Wb, work);
        smes_launch(fold_finish_kernel<32>, gfin, 256, 0, st, E, T, ldg, d_out, d_in, splits, work, head_w, b, Gb, c);
    }
  }
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? SMES_OK : set_error(SMES_ERR_CUDA, "fold_heads: %s", cudaGetErrorString(e));
}

int smes_unfold_grads(int E, int T, int ldg, int d_out, int d_in, const float* Q, long q_es, long q_ts, long q_ks,
                      const float* csum,
                      long cs_es, const float* head_w, const void* W, const float* b, float* dW, float* db,
                      float* work, float* d_head_w, void* stream) {
  if (T < 1 || T > 32 || ldg < T) return set_error(SMES_ERR_SHAPE, "unfold_grads: T=%d ldg=%d", T, ldg);
  if (d_in % 8) return set_error(SMES_ERR_SHAPE, "unfold_grads: d_in=%d must be a multiple of 8", d_in);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  auto Wb = reinterpret_cast<const __nv_bfloat16*>(W);
  if (gemm_path(E, T, d_out, d_in)) {
    const FoldWork w = fold_layout(E, T, d_out, d_in);
    auto* Wp = reinterpret_cast<__nv_bfloat16*>(work + w.wp);
    auto* seg = reinterpret_cast<int32_t*>(work + w.seg128);
    auto* Qbf = reinterpret_cast<__nv_bfloat16*>(work + w.qbf);
    float* Y = work + w.y;
    smes_launch(fold_prep_kernel, (128 * d_out + 255) / 256, 256, 0, st, T, ldg, d_out, head_w, nullptr, Wp);
    smes_launch(seg_arith_kernel, (E + 256) / 256, 256, 0, st, E, 128, seg);
    smes_launch(unfold_split_kernel, 4096, 256, 0, st, E, T, d_in, Q, q_es, q_ts, q_ks, Qbf);
    int rc = smes_gemm_ragged_k_periodic(Wp, d_out, 128, Qbf, d_in, (long)E * 128, E, d_out, d_in, seg, dW, nullptr,
                                         128, stream);
    if (rc) return rc;
    smes_launch(unfold_db_kernel, (E * d_out + 255) / 256, 256, 0, st, E, T, d_out, csum, cs_es, head_w, db);
    rc = smes_gemm_ragged_m(Qbf, d_in, (long)E * 128, W, E, d_out, d_in, 0, seg, nullptr, 0, nullptr, nullptr, 0, Y,
                            d_out, 1, (long)E * 128, stream);
    if (rc) return rc;
    dim3 g((d_out + 31) / 32, T);
    smes_launch(unfold_head_reduce_kernel, g, 256, 0, st, E, T, d_out, Y, csum, cs_es, b, d_head_w);
  } else {
    dim3 g1((d_in + 127) / 128, (d_out + 31) / 32, E);
    const int splits = (d_in + 63) / 64;
    dim3 g2((d_out + 63) / 64, E, splits);
    dim3 gfin((d_out + 31) / 32, T);
    const int npair = (int)(g1.x * g1.y * g1.z + g2.x * g2.y * g2.z);
    switch (fold_tm(T)) {
      case 8:
        smes_launch(unfold_pair_kernel<8>, npair, 128, 0, st, E, T, ldg, d_out, d_in, Q, q_es, q_ts, q_ks, csum, cs_es,
                                                         head_w, Wb, dW, db, work);
        smes_launch(unfold_finish_kernel<8>, gfin, 256, 0, st, E, T, d_out, splits, work, csum, cs_es, b, d_head_w);
        break;
      case 16:
        smes_launch(unfold_pair_kernel<16>, npair, 128, 0, st, E, T, ldg, d_out, d_in, Q, q_es, q_ts, q_ks, csum, cs_es,
                                                         head_w, Wb, dW, db, work);
        smes_launch(unfold_finish_kernel<16>, gfin, 256, 0, st, E, T, d_out, splits, work, csum, cs_es, b, d_head_w);
        break;
      default:
        smes_launch(unfold_pair_kernel<32>, npair, 128, 0, st, E, T, ldg, d_out, d_in, Q, q_es, q_ts, q_ks, csum, cs_es,
                                                         head_w, Wb, dW, db, work);
        smes_launch(unfold_finish_kernel<32>, gfin, 256, 0, st, E, T, d_out, splits, work, csum, cs_es, b, d_head_w);
    }
  }
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? SMES_OK : set_error(SMES_ERR_CUDA, "unfold_grads: %s", cudaGetErrorString(e));
}

}  // extern "C"
