// K5 / K9 / bias grads -- deterministic reductions (fixed order, no float atomics).
//
//   stats_finalize : LoadStats from the (possibly all-reduced) per-expert sums
//                    (taskmoe/balance.py:62-70): f = counts/(B T), p = mass/(B T),
//                    L_lb = (E/K) <f, p>
//   loss_finalize  : task loss (training.py:57) and total (training.py:90-94)
//   seg_colsum     : per-expert bias gradients db_e = sum_{rows in e} d_pre (training.py:190)
//   unpermute      : d_hidden[b] = d_router[b] + sum_u dX[row(b,u)] (training.py:192, :212)
//   part_reduce    : per-CTA partials -> one vector (head grads, training.py:151-152)
#include <algorithm>
#include <cstdint>
#include "ptx.cuh"
#include "smes_capi.h"

namespace smes {

__global__ void stats_finalize_kernel(int E, int K, int e_lb, double bt, int dense, const double* __restrict__ raw,
                                      double* __restrict__ out, float* __restrict__ freq_f32) {
  pdl_wait();
  // out: [freq E][mass E][counts E][value]
  __shared__ double red[32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double part = 0.0;
  for (int e = tid; e < E; e += blockDim.x) {
    const double f = raw[e] / bt;
    const double m = (dense ? raw[2 * E + e] : raw[E + e]) / bt;
    out[e] = f;
    out[E + e] = m;
    out[2 * E + e] = raw[e];
    freq_f32[e] = (float)f;
    part += f * m;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
  if (lane == 0) red[warp] = part;
  __syncthreads();
  if (tid == 0) {
    double s = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += red[w];
    out[3 * E] = ((double)e_lb / (double)K) * s;
  }
}

__global__ void loss_finalize_kernel(int n, const double* __restrict__ part, double inv_b, double beta,
                                     const double* __restrict__ stats_value, double* __restrict__ out) {
  pdl_wait();
  __shared__ double red[32];
  double v = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) v += part[i];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) s += red[i];
    const double task = s * inv_b;
    const double lb = stats_value ? *stats_value : 0.0;
    out[0] = task;
    out[1] = lb;
    out[2] = task + beta * lb;
  }
}

// stage 1: one block per 128-row tile (tiles never straddle groups).  Thread = 8 columns x
// a strided subset of the tile's rows; the row groups are combined in a fixed order.
__global__ void __launch_bounds__(256) seg_colsum_tiles_kernel(const __nv_bfloat16* __restrict__ M, long ld, int N,
                                                               const int32_t* __restrict__ seg, int G,
                                                               float* __restrict__ part) {
  pdl_wait();
  __shared__ float red[2048 + 64];
  const int tile = blockIdx.x;
  if (tile * 128 >= seg[G]) return;
  const int ct = N / 8;                       // column threads (<= 256)
  const int rg = 256 / ct;                    // row groups
  const int c = (threadIdx.x % ct) * 8, g = threadIdx.x / ct;
  for (int n0 = 0; n0 < N; n0 += 2048) {
    float s[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    if (g < rg && n0 + c < N) {
      const __nv_bfloat16* p = M + (long)tile * 128 * ld + n0 + c;
#pragma unroll 4
      for (int r = g; r < 128; r += rg) {
        uint4 v = __ldg(reinterpret_cast<const uint4*>(p + (long)r * ld));
        const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&v);
#pragma unroll
        for (int i = 0; i < 4; ++i) { float2 f = __bfloat1622float2(h[i]); s[2 * i] += f.x; s[2 * i + 1] += f.y; }
      }
    }
    // fixed-order combine of the row groups: group 0 first, then 1, ...
    for (int k = 0; k < rg; ++k) {
      if (g == k && n0 + c < N) {
#pragma unroll
        for (int i = 0; i < 8; ++i) red[c + i] = (k == 0 ? 0.f : red[c + i]) + s[i];
      }
      __syncthreads();
    }
    for (int i = threadIdx.x; i < min(2048, N - n0); i += blockDim.x) part[(long)tile * N + n0 + i] = red[i];
    __syncthreads();
  }
}

// stage 2: out[g][n] = sum of the group's tile partials in tile order
__global__ void seg_colsum_groups_kernel(const float* __restrict__ part, int N, const int32_t* __restrict__ seg,
                                         float* __restrict__ out) {
  pdl_wait();
  const int g = blockIdx.y;
  const int n = blockIdx.x * blockDim.x + threadIdx.x;
  if (n >= N) return;
  const int t0 = seg[g] / 128, t1 = seg[g + 1] / 128;
  float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
  int t = t0;
  for (; t + 4 <= t1; t += 4) {
    s0 += part[(long)t * N + n];
    s1 += part[(long)(t + 1) * N + n];
    s2 += part[(long)(t + 2) * N + n];
    s3 += part[(long)(t + 3) * N + n];
  }
  for (; t < t1; ++t) s0 += part[(long)t * N + n];
  out[(long)g * N + n] = (s0 + s1) + (s2 + s3);
}

template <int VEC>
__global__ void unpermute_kernel(int B, int d, const int32_t* __restrict__ usize, const int32_t* __restrict__ row_of,
                                 int umax, const __nv_bfloat16* __restrict__ dX, long ldx,
                                 const float* __restrict__ dh_router, float* __restrict__ dh) {
  pdl_wait();
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= B) return;
  const int b = warp;
  float acc[VEC][8];
#pragma unroll
  for (int v = 0; v < VEC; ++v) {
    const int c = (v * 32 + lane) * 8;
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[v][i] = 0.f;
    if (dh_router && c < d) {
      float4 x0 = __ldg(reinterpret_cast<const float4*>(dh_router + (long)b * d + c));
      float4 x1 = __ldg(reinterpret_cast<const float4*>(dh_router + (long)b * d + c + 4));
      acc[v][0] = x0.x; acc[v][1] = x0.y; acc[v][2] = x0.z; acc[v][3] = x0.w;
      acc[v][4] = x1.x; acc[v][5] = x1.y; acc[v][6] = x1.z; acc[v][7] = x1.w;
    }
  }
  // the instance's row indices come in one coalesced load (lane u holds row_of[u], read over the
  // full umax width alongside usize), then are broadcast: the row gathers no longer wait on a
  // dependent index load each
  const int U = usize[b];
  for (int base = 0; base < umax; base += 32) {
    const int myrow = base + lane < umax ? row_of[(long)b * umax + base + lane] : 0;
    const int n = min(32, U - base);
    if (n <= 0) break;
#pragma unroll 8
    for (int j = 0; j < n; ++j) {
      const long r = __shfl_sync(0xffffffffu, myrow, j);
#pragma unroll
      for (int v = 0; v < VEC; ++v) {
        const int c = (v * 32 + lane) * 8;
        if (c < d) {
          uint4 q = __ldg(reinterpret_cast<const uint4*>(dX + r * ldx + c));
          const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&q);
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            float2 f = __bfloat1622float2(h[i]);
            acc[v][2 * i] += f.x;
            acc[v][2 * i + 1] += f.y;
          }
        }
      }
    }
  }
#pragma unroll
  for (int v = 0; v < VEC; ++v) {
    const int c = (v * 32 + lane) * 8;
    if (c < d) {
      *reinterpret_cast<float4*>(dh + (long)b * d + c) = make_float4(acc[v][0], acc[v][1], acc[v][2], acc[v][3]);
      *reinterpret_cast<float4*>(dh + (long)b * d + c + 4) = make_float4(acc[v][4], acc[v][5], acc[v][6], acc[v][7]);
    }
  }
}

__global__ void __launch_bounds__(1024) part_reduce_kernel(const float* __restrict__ part, int nparts, int n,
                                                            float* __restrict__ out) {
  pdl_wait();
  __shared__ float red[32][33];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int i = blockIdx.x * 32 + lane;
  const int per = (nparts + nw - 1) / nw;
  const int p0 = warp * per, p1 = min(nparts, p0 + per);
  float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
  if (i < n) {
    int p = p0;
    for (; p + 4 <= p1; p += 4) {
      s0 += part[(long)p * n + i];
      s1 += part[(long)(p + 1) * n + i];
      s2 += part[(long)(p + 2) * n + i];
      s3 += part[(long)(p + 3) * n + i];
    }
    for (; p < p1; ++p) s0 += part[(long)p * n + i];
  }
  red[warp][lane] = (s0 + s1) + (s2 + s3);
  __syncthreads();
  if (warp == 0 && i < n) {
    float t = 0.f;
    for (int w = 0; w < nw; ++w) t += red[w][lane];
    out[i] = t;
  }
}

// out = sum_p part[p] for a handful of partials, in partial order (deterministic)
__global__ void __launch_bounds__(256) part_sum_few_kernel(const float4* __restrict__ part, int nparts, int n4,
                                                           float4* __restrict__ out) {
  pdl_wait();
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += gridDim.x * blockDim.x) {
    float4 acc = part[i];
    for (int p = 1; p < nparts; ++p) {
      const float4 v = part[(long)p * n4 + i];
      acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    }
    out[i] = acc;
  }
}

// dL_lb/dz (balance.py:83-99): one warp per (t, b) row; sparse reading uses the
// renormalised weights on the active set, dense reading the full softmax of z.
__global__ void lb_grad_kernel(int T, int B, int E, int K, const int32_t* __restrict__ active,
                               const float* __restrict__ wsel, const float* __restrict__ z, long zst, long zsb,
                               const float* __restrict__ freq, float coef, int dense, float* __restrict__ out) {
  pdl_wait();
  const int row = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (row >= T * B) return;
  const int t = row / B, b = row - t * B;
  float* o = out + (long)row * E;
  if (!dense) {
    for (int e = lane; e < E; e += 32) o[e] = 0.f;
    __syncwarp();
    float wf = 0.f, w = 0.f;
    int e = 0;
    if (lane < K) {
      e = active[(long)row * K + lane];
      w = wsel[(long)row * K + lane];
      wf = w * freq[e];
    }
    float F = wf;
#pragma unroll
    for (int s = 16; s > 0; s >>= 1) F += __shfl_xor_sync(0xffffffffu, F, s);
    if (lane < K) o[e] = coef * w * (freq[e] - F);
  } else {
    const float* zr = z + (long)t * zst + (long)b * zsb;
    float mx = -INFINITY;
    for (int e = lane; e < E; e += 32) mx = fmaxf(mx, zr[e]);
#pragma unroll
    for (int s = 16; s > 0; s >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, s));
    float sum = 0.f, F = 0.f;
    for (int e = lane; e < E; e += 32) { const float q = expf(zr[e] - mx); sum += q; F += q * freq[e]; }
#pragma unroll
    for (int s = 16; s > 0; s >>= 1) {
      sum += __shfl_xor_sync(0xffffffffu, sum, s);
      F += __shfl_xor_sync(0xffffffffu, F, s);
    }
    F /= sum;
    for (int e = lane; e < E; e += 32) o[e] = coef * (expf(zr[e] - mx) / sum) * (freq[e] - F);
  }
}

// weighted clamped BCE (training.py:54-57) -> per-block fp64 partials
__global__ void bce_kernel(int T, int B, const float* __restrict__ pred, const float* __restrict__ y,
                           const float* __restrict__ lam, double* __restrict__ part, int32_t* __restrict__ bad) {
  pdl_wait();
  __shared__ double red[32];
  double v = 0.0;
  int badv = 0;
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < (long)T * B; i += (long)gridDim.x * blockDim.x) {
    const int t = (int)(i / B);
    const double p = pred[i], yy = y[i];
    if (!(p >= 0.0 && p <= 1.0)) badv |= 1;
    if (!(yy == 0.0 || yy == 1.0)) badv |= 2;
    const double c = p < 1e-7 ? 1e-7 : (p > 1.0 - 1e-7 ? 1.0 - 1e-7 : p);
    v += (double)lam[t] * -(yy * log(c) + (1.0 - yy) * log1p(-c));
  }
  if (badv) atomicOr(bad, badv);
#pragma unroll
  for (int s = 16; s > 0; s >>= 1) v += __shfl_xor_sync(0xffffffffu, v, s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += red[w];
    part[blockIdx.x] = s;
  }
}


// Every reduction that depends only on the training combine's per-CTA partials, in one launch:
// task loss (+ L_lb) -> loss_out, per-(expert, task) sums of C, router bias grads, head bias grads.
// Blocks [0, n_cs) column tiles of csum, then router-bias tiles, then head-bias tiles, last block the
// loss; each tile: 32 warps split the partials, fixed-order combine (deterministic).
struct PostArgs {
  int nparts;
  const float* part_csum; int n_cs; float* csum;
  const float* part_rb; int n_rb; float* rb;
  const float* part_db; int n_db; float* db;
  const double* loss_part; double inv_b, beta; const double* stats_value; double* loss_out;
};

__device__ __forceinline__ void tile_sum(const float* __restrict__ part, int nparts, int n, int tile,
                                         float* __restrict__ out, float (*red)[33]) {
  // 32 warps x 4 independent loads in flight per lane: ~nparts/128 dependent rounds
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int i = tile * 32 + lane;
  float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
  if (i < n) {
    int p = warp;
    for (; p + 96 < nparts; p += 128) {
      s0 += part[(long)p * n + i]; s1 += part[(long)(p + 32) * n + i];
      s2 += part[(long)(p + 64) * n + i]; s3 += part[(long)(p + 96) * n + i];
    }
    for (; p < nparts; p += 32) s0 += part[(long)p * n + i];
  }
  red[warp][lane] = (s0 + s1) + (s2 + s3);
  __syncthreads();
  if (warp == 0 && i < n) {
    float t = 0.f;
#pragma unroll
    for (int w = 0; w < 32; ++w) t += red[w][lane];
    out[i] = t;
  }
}

__global__ void __launch_bounds__(1024) post_combine_kernel(const PostArgs a) {
  pdl_wait();
  __shared__ float red[32][33];
  __shared__ double dred[32];
  const int t_cs = a.part_csum ? (a.n_cs + 31) / 32 : 0;
  const int t_rb = a.part_rb ? (a.n_rb + 31) / 32 : 0;
  const int t_db = (a.n_db + 31) / 32;
  int bid = blockIdx.x;
  if (bid < t_cs) { tile_sum(a.part_csum, a.nparts, a.n_cs, bid, a.csum, red); return; }
  bid -= t_cs;
  if (bid < t_rb) { tile_sum(a.part_rb, a.nparts, a.n_rb, bid, a.rb, red); return; }
  bid -= t_rb;
  if (bid < t_db) { tile_sum(a.part_db, a.nparts, a.n_db, bid, a.db, red); return; }
  // loss
  double v = 0.0;
  for (int i = threadIdx.x; i < a.nparts; i += blockDim.x) v += a.loss_part[i];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) dred[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int i = 0; i < 32; ++i) s += dred[i];
    const double task = s * a.inv_b;
    const double lb = a.stats_value ? *a.stats_value : 0.0;
    a.loss_out[0] = task;
    a.loss_out[1] = lb;
    a.loss_out[2] = task + a.beta * lb;
  }
}

}  // namespace smes

using namespace smes;

static int launch_check(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_error(SMES_ERR_CUDA, "%s launch: %s", what, cudaGetErrorString(e));
  return SMES_OK;
}

extern "C" {

int smes_stats_finalize(int E, int K, int lb_experts, double batch_times_tasks, int dense, const double* raw,
                        double* out, float* freq_f32, void* stream) {
  const int e_lb = lb_experts > 0 ? lb_experts : E;
  smes_launch(stats_finalize_kernel, 1, 256, 0, reinterpret_cast<cudaStream_t>(stream), E, K, e_lb, batch_times_tasks, dense, raw,
                                                                               out, freq_f32);
  return launch_check("stats_finalize");
}

int smes_loss_finalize(int nparts, const double* part, double inv_b, double beta, const double* stats_value,
                       double* out, void* stream) {
  smes_launch(loss_finalize_kernel, 1, 256, 0, reinterpret_cast<cudaStream_t>(stream), nparts, part, inv_b, beta, stats_value,
                                                                            out);
  return launch_check("loss_finalize");
}

int smes_seg_colsum(const void* M, long ld, long rows_cap, int N, const int32_t* seg, int G, float* part, float* out,
                    void* stream) {
  if (N % 8 || ld % 8) return set_error(SMES_ERR_SHAPE, "seg_colsum: N=%d and ld must be multiples of 8", N);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (N / 8 > 256 || N % 8) return set_error(SMES_ERR_SHAPE, "seg_colsum: N=%d must be <= 2048", N);
  const int tiles = (int)(rows_cap / 128);
  smes_launch(seg_colsum_tiles_kernel, tiles, 256, 0, st, reinterpret_cast<const __nv_bfloat16*>(M), ld, N, seg, G, part);
  int rc = launch_check("seg_colsum_tiles");
  if (rc) return rc;
  dim3 g2((N + 63) / 64, G);
  smes_launch(seg_colsum_groups_kernel, g2, 64, 0, st, part, N, seg, out);
  return launch_check("seg_colsum_groups");
}

int smes_unpermute(int B, int d, const int32_t* usize, const int32_t* row_of, int umax, const void* dX, long ldx,
                   const float* dh_router, float* dh, void* stream) {
  if (d % 8 || d > 2048) return set_error(SMES_ERR_SHAPE, "unpermute: d=%d", d);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const int vec = (d + 255) / 256;
  const int blocks = (B * 32 + 255) / 256;
  auto* x = reinterpret_cast<const __nv_bfloat16*>(dX);
  if (vec <= 1) smes_launch(unpermute_kernel<1>, blocks, 256, 0, st, B, d, usize, row_of, umax, x, ldx, dh_router, dh);
  else if (vec <= 2) smes_launch(unpermute_kernel<2>, blocks, 256, 0, st, B, d, usize, row_of, umax, x, ldx, dh_router, dh);
  else if (vec <= 4) smes_launch(unpermute_kernel<4>, blocks, 256, 0, st, B, d, usize, row_of, umax, x, ldx, dh_router, dh);
  else smes_launch(unpermute_kernel<8>, blocks, 256, 0, st, B, d, usize, row_of, umax, x, ldx, dh_router, dh);
  return launch_check("unpermute");
}

int smes_lb_grad(int T, int B, int E, int K, const int32_t* active, const float* wsel, const float* z, long zst,
                 long zsb, const float* freq, float coef, int dense, float* out, void* stream) {
  if (K > 32) return set_error(SMES_ERR_CONFIG, "lb_grad: K=%d exceeds 32", K);
  const long rows = (long)T * B;
  smes_launch(lb_grad_kernel, (unsigned)((rows * 32 + 255) / 256), 256, 0, reinterpret_cast<cudaStream_t>(stream), 
      T, B, E, K, active, wsel, z, zst, zsb, freq, coef, dense, out);
  return launch_check("lb_grad");
}

int smes_bce_loss(int T, int B, const float* pred, const float* labels, const float* lam, double* part, int nparts,
                  int32_t* bad, void* stream) {
  smes_launch(bce_kernel, nparts, 256, 0, reinterpret_cast<cudaStream_t>(stream), T, B, pred, labels, lam, part, bad);
  return launch_check("bce_loss");
}

int smes_part_reduce(const float* part, int nparts, int n, float* out, void* stream) {
  if (nparts <= 8 && n % 4 == 0 && (reinterpret_cast<uintptr_t>(part) % 16) == 0 &&
      (reinterpret_cast<uintptr_t>(out) % 16) == 0) {
    // few partials over a long vector (the router wgrad at large T*E*d): one float4 per thread; the
    // column-block kernel below would launch n / 32 CTAs with most warps idle
    const int n4 = n / 4;
    const int blocks = (int)std::min<long>((n4 + 255) / 256, 148L * 16);
    smes_launch(part_sum_few_kernel, blocks, 256, 0, reinterpret_cast<cudaStream_t>(stream),
                reinterpret_cast<const float4*>(part), nparts, n4, reinterpret_cast<float4*>(out));
    return launch_check("part_reduce");
  }
  smes_launch(part_reduce_kernel, (n + 31) / 32, nparts >= 256 ? 1024 : 256, 0, reinterpret_cast<cudaStream_t>(stream), part, nparts, n, out);
  return launch_check("part_reduce");
}


int smes_post_combine(int nparts, const float* part_csum, int n_csum, float* csum, const float* part_rb, int n_rb,
                      float* rb, const float* part_db, int n_db, float* db, const double* loss_part, double inv_b,
                      double beta, const double* stats_value, double* loss_out, void* stream) {
  PostArgs a{nparts, part_csum, n_csum, csum, part_rb, n_rb, rb, part_db, n_db, db, loss_part, inv_b, beta,
             stats_value, loss_out};
  const int blocks = (part_csum ? (n_csum + 31) / 32 : 0) + (part_rb ? (n_rb + 31) / 32 : 0) + (n_db + 31) / 32 + 1;
  smes_launch(post_combine_kernel, blocks, 1024, 0, reinterpret_cast<cudaStream_t>(stream), a);
  return launch_check("post_combine");
}
}  // extern "C"
