// K2 -- execution plan: per-expert loads + stable counting sort + gather.
//
// Restates `build_execution_plan` (taskmoe/execution.py:85-123) and the gather
// `hidden[plan.gather_instances]` (taskmoe/model.py:301) on the device:
//   loads[e]  = #instances whose union holds e           (execution.py:109, bincount)
//   order     = expert-major, instance-ascending          (execution.py:110, lexsort((b, e)))
//   offsets   = exclusive prefix of loads                 (execution.py:113)
// The router already produced per-chunk union histograms, so the sort is a
// two-level counting sort: chunk_reduce scans each expert's column of chunk
// counts (chunk base), scatter then ranks rows inside a chunk with per-warp
// counts + in-order walks.  The result is bit-identical to lexsort.
// Physical layout: each expert segment is padded to a multiple of 128 rows
// (zero rows) so GEMM tiles never straddle experts; logical offsets are kept
// alongside for the reference-facing ExecutionPlan view.
#include "ptx.cuh"
#include "fold_full.cuh"
#include "smes_capi.h"

namespace smes {

constexpr int PL_WARPS = 4;       // must match the router's RT_WARPS
constexpr int SEG_ALIGN = 128;

// grid = E blocks: column scans of the (C, E) chunk tables.  (A chunk-range-parallel variant with
// coalesced row loads and a cross-block prefix measured 19 us against this kernel's 15 us at c2:
// its cross-block flag / aggregate round trips cost more than the column loads save.)  The last block to
// finish derives the padded / logical segment offsets (ticket counter, reset
// in-kernel so the kernel is CUDA-graph replayable).
__device__ __forceinline__ void chunk_reduce_body(int nblocks, int e, int C, int E, const int32_t* __restrict__ chunk_union,
                                    const int32_t* __restrict__ chunk_active, const double* __restrict__ chunk_mass,
                                    const double* __restrict__ chunk_dmass, int32_t* __restrict__ chunk_base,
                                    int32_t* __restrict__ loads, double* __restrict__ stats_raw,
                                    int32_t* __restrict__ seg_pad, int32_t* __restrict__ seg_log,
                                    int32_t* __restrict__ totals, unsigned int* __restrict__ ticket,
                                    int32_t* __restrict__ seg_half, double lb_scale, double bt, int dense,
                                    double* __restrict__ st_out, float* __restrict__ freq_f32) {
  __shared__ int32_t warp_tot[32];
  __shared__ double red[3][32];
  __shared__ bool is_last;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  int32_t carry = 0;
  double s_act = 0.0, s_m = 0.0, s_dm = 0.0;
  // stats sums in fixed per-thread strided order, then fixed tree
  for (int c = tid; c < C; c += blockDim.x) {
    s_act += (double)chunk_active[(long)c * E + e];
    s_m += chunk_mass[(long)c * E + e];
    s_dm += chunk_dmass[(long)c * E + e];
  }
  // exclusive scan of chunk_union[:, e]: each thread owns a contiguous run of up to 16 chunks,
  // loaded in one round trip; thread sums are scanned across the block, then written back
  constexpr int PT = 16;
  const int per = (C + blockDim.x - 1) / blockDim.x;
  if (per <= PT) {
    int v[PT];
    int tsum = 0;
    const int cb = tid * per;
#pragma unroll
    for (int k = 0; k < PT; ++k) {
      v[k] = (k < per && cb + k < C) ? chunk_union[(long)(cb + k) * E + e] : 0;
      tsum += v[k];
    }
    int x = tsum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) warp_tot[warp] = x;
    __syncthreads();
    if (warp == 0) {
      int w = lane < nw ? warp_tot[lane] : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, w, o);
        if (lane >= o) w += y;
      }
      warp_tot[lane] = w;
    }
    __syncthreads();
    int run = x - tsum + (warp > 0 ? warp_tot[warp - 1] : 0);
#pragma unroll
    for (int k = 0; k < PT; ++k) {
      if (k < per && cb + k < C) chunk_base[(long)(cb + k) * E + e] = run;
      run += v[k];
    }
    carry = warp_tot[nw - 1];
  } else {
    for (int c0 = 0; c0 < C; c0 += blockDim.x) {
      int c = c0 + tid;
      int v = c < C ? chunk_union[(long)c * E + e] : 0;
      int x = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      if (lane == 31) warp_tot[warp] = x;
      __syncthreads();
      if (warp == 0) {
        int w = lane < nw ? warp_tot[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          int y = __shfl_up_sync(0xffffffffu, w, o);
          if (lane >= o) w += y;
        }
        warp_tot[lane] = w;  // inclusive over warps
      }
      __syncthreads();
      int excl = x - v + (warp > 0 ? warp_tot[warp - 1] : 0) + carry;
      if (c < C) chunk_base[(long)c * E + e] = excl;
      carry += warp_tot[nw - 1];
      __syncthreads();
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    s_act += __shfl_xor_sync(0xffffffffu, s_act, o);
    s_m += __shfl_xor_sync(0xffffffffu, s_m, o);
    s_dm += __shfl_xor_sync(0xffffffffu, s_dm, o);
  }
  if (lane == 0) { red[0][warp] = s_act; red[1][warp] = s_m; red[2][warp] = s_dm; }
  __syncthreads();
  if (tid == 0) {
    double a = 0, m = 0, dm = 0;
    for (int w = 0; w < nw; ++w) { a += red[0][w]; m += red[1][w]; dm += red[2][w]; }
    loads[e] = carry;
    stats_raw[e] = a;            // active counts (as fp64, all-reduce friendly)
    stats_raw[E + e] = m;        // sparse mass sum
    stats_raw[2 * E + e] = dm;   // dense mass sum
    __threadfence();
    unsigned int t = atomicAdd(ticket, 1u);
    is_last = (t == (unsigned)(nblocks - 1));
  }
  __syncthreads();
  if (!is_last) return;
  // last block: every expert's load in one parallel round trip (a serial chain of E volatile
  // L2 loads here cost ~10 us), then the prefix by one thread from shared memory
  __shared__ int32_t s_ld[1024];
  __threadfence();
  for (int i = tid; i < E; i += blockDim.x) s_ld[i] = ((volatile int32_t*)loads)[i];
  __syncthreads();
  if (tid == 0) {
    int p = 0, l = 0;
    for (int i = 0; i < E; ++i) {
      const int ld = s_ld[i];
      const int len = (ld + SEG_ALIGN - 1) / SEG_ALIGN * SEG_ALIGN;
      seg_pad[i] = p;
      seg_log[i] = l;
      if (seg_half) { seg_half[2 * i] = p; seg_half[2 * i + 1] = p + len / 2; }   // 64-row aligned halves
      p += len;
      l += ld;
    }
    if (seg_half) seg_half[2 * E] = p;
    seg_pad[E] = p;
    seg_log[E] = l;
    totals[0] = 0;   // totals[0:2] doubles as the one-group segment table [0, padded rows]
    totals[1] = p;   // physical rows incl. padding
    totals[2] = l;   // N_act (logical rows)
    *ticket = 0u;
  }
  if (st_out != nullptr) {
    // LoadStats finalize (balance.py:54-80) when no cross-device exchange sits between the sums
    // and their use: the stats_finalize launch folded into the last block (same arithmetic)
    double part = 0.0;
    for (int i = tid; i < E; i += blockDim.x) {
      const double cnt = ((volatile double*)stats_raw)[i];
      const double f = cnt / bt;
      const double m = (dense ? ((volatile double*)stats_raw)[2 * E + i] : ((volatile double*)stats_raw)[E + i]) / bt;
      st_out[i] = f;
      st_out[E + i] = m;
      st_out[2 * E + i] = cnt;
      freq_f32[i] = (float)f;
      part += f * m;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
    if (lane == 0) red[0][warp] = part;
    __syncthreads();
    if (tid == 0) {
      double v = 0.0;
      for (int w = 0; w < nw; ++w) v += red[0][w];
      st_out[3 * E] = lb_scale * v;     // (E / K) <f, p>
    }
  }
}

__global__ void chunk_reduce_kernel(int C, int E, const int32_t* __restrict__ chunk_union,
                                    const int32_t* __restrict__ chunk_active, const double* __restrict__ chunk_mass,
                                    const double* __restrict__ chunk_dmass, int32_t* __restrict__ chunk_base,
                                    int32_t* __restrict__ loads, double* __restrict__ stats_raw,
                                    int32_t* __restrict__ seg_pad, int32_t* __restrict__ seg_log,
                                    int32_t* __restrict__ totals, unsigned int* __restrict__ ticket,
                                    int32_t* __restrict__ seg_half, double lb_scale, double bt, int dense,
                                    double* __restrict__ st_out, float* __restrict__ freq_f32) {
  pdl_wait();
  chunk_reduce_body(gridDim.x, blockIdx.x, C, E, chunk_union, chunk_active, chunk_mass, chunk_dmass, chunk_base, loads,
                    stats_raw, seg_pad, seg_log, totals, ticket, seg_half, lb_scale, bt, dense, st_out, freq_f32);
}

// The plan reduce (blocks [0, E)) and the head fold of a training step (blocks [E, E + nx E),
// fold_full.cuh) in one launch: the reduce's E column-scan blocks leave most SMs idle, so the
// fold (which depends on the weights only) runs in that slack instead of as its own kernel on
// the forward's critical path.
struct FoldArgsPR {
  int T, ldg, d_out, d_in;
  const float* head_w;
  const __nv_bfloat16* W;
  const float* b;
  __nv_bfloat16* G;
  float* c;
};
__global__ void __launch_bounds__(256)
    plan_reduce_fold_kernel(int C, int E, const int32_t* __restrict__ chunk_union, const int32_t* __restrict__ chunk_active,
                            const double* __restrict__ chunk_mass, const double* __restrict__ chunk_dmass,
                            int32_t* __restrict__ chunk_base, int32_t* __restrict__ loads, double* __restrict__ stats_raw,
                            int32_t* __restrict__ seg_pad, int32_t* __restrict__ seg_log, int32_t* __restrict__ totals,
                            unsigned int* __restrict__ ticket, int32_t* __restrict__ seg_half, double lb_scale,
                            double bt, int dense, double* __restrict__ st_out, float* __restrict__ freq_f32,
                            const FoldArgsPR f) {
  pdl_wait();
  extern __shared__ __align__(16) uint8_t fsm[];
  if ((int)blockIdx.x >= E) {
    const int nx = (f.d_in + 63) / 64;
    const int k = blockIdx.x - E;
    fold_full_body<8>(k % nx, k / nx, f.T, f.ldg, f.d_out, f.d_in, f.head_w, f.W, f.b, f.G, f.c, fsm);
    return;
  }
  chunk_reduce_body(E, blockIdx.x, C, E, chunk_union, chunk_active, chunk_mass, chunk_dmass, chunk_base, loads,
                    stats_raw, seg_pad, seg_log, totals, ticket, seg_half, lb_scale, bt, dense, st_out, freq_f32);
}

// grid = C + E blocks.  Blocks < C: stable scatter of chunk c's (instance, expert)
// pairs + vectorised gather of hidden rows.  Blocks >= C: zero the pad rows of
// expert (blockIdx - C) in X (and optionally in the d_packed buffer).
template <int EPL, int VEC>
__global__ void __launch_bounds__(PL_WARPS * 32)
    scatter_kernel(int B, int E, int d, int rows_per_warp, const uint32_t* __restrict__ umask,
                   const int32_t* __restrict__ chunk_base, const int32_t* __restrict__ seg_pad,
                   const int32_t* __restrict__ loads, const __nv_bfloat16* __restrict__ h, long ldh,
                   __nv_bfloat16* __restrict__ X, long ldx, int32_t* __restrict__ row_of, int umax,
                   int32_t* __restrict__ gather_inst, int32_t* __restrict__ gather_exp,
                   __nv_bfloat16* __restrict__ zero_rows2, long ldz2, int d2) {
  pdl_wait();
  const int C = (B + PL_WARPS * rows_per_warp - 1) / (PL_WARPS * rows_per_warp);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int EW = (E + 31) >> 5;
  if ((int)blockIdx.x >= C) {
    // ---- pad fill for expert e
    const int e = blockIdx.x - C;
    const int lo = seg_pad[e] + loads[e], hi = seg_pad[e + 1];
    const uint4 z4 = make_uint4(0, 0, 0, 0);
    for (int r = lo + warp; r < hi; r += PL_WARPS) {
      if (X != nullptr)
        for (int c = lane * 8; c < d; c += 256) *reinterpret_cast<uint4*>(X + (long)r * ldx + c) = z4;
      if (zero_rows2 != nullptr)
        for (int c = lane * 8; c < d2; c += 256) *reinterpret_cast<uint4*>(zero_rows2 + (long)r * ldz2 + c) = z4;
      if (lane == 0) { gather_inst[r] = -1; gather_exp[r] = e; }
    }
    return;
  }
  __shared__ int32_t s_cnt[PL_WARPS][1024];
  const int c = blockIdx.x;
  const int row0 = c * PL_WARPS * rows_per_warp + warp * rows_per_warp;
  const int rend = min(row0 + rows_per_warp, B);
  // phase 1: per-warp counts of union membership (lane owns experts lane + 32 j)
  int cnt[EPL];
#pragma unroll
  for (int j = 0; j < EPL; ++j) cnt[j] = 0;
  for (int b = row0; b < rend; ++b) {
#pragma unroll
    for (int j = 0; j < EPL; ++j)
      if (j < EW) cnt[j] += (__ldg(&umask[(long)b * EW + j]) >> lane) & 1u;
  }
#pragma unroll
  for (int j = 0; j < EPL; ++j) {
    int e = lane + 32 * j;
    if (e < E) s_cnt[warp][e] = cnt[j];
  }
  __syncthreads();
  // phase 2: running row index per owned expert = seg_pad + chunk_base + earlier warps
  int run[EPL];
#pragma unroll
  for (int j = 0; j < EPL; ++j) {
    int e = lane + 32 * j;
    if (e < E) {
      int base = __ldg(&seg_pad[e]) + __ldg(&chunk_base[(long)c * E + e]);
      for (int w = 0; w < warp; ++w) base += s_cnt[w][e];
      run[j] = base;
    } else {
      run[j] = 0;
    }
  }
  // phase 3: in-order walk; each row's copies land at consecutive positions per expert.  The next
  // instance's hidden row and mask words are fetched while this one's copies are stored, and the
  // per-copy metadata (row_of / gather tables) is written by the owning lanes in parallel.
  uint4 hv[VEC];
  uint32_t wv[EPL];
  auto fetch = [&](int b, uint4 (&hh)[VEC], uint32_t (&ww)[EPL]) {
#pragma unroll
    for (int v = 0; v < VEC; ++v) {
      int col = (v * 32 + lane) * 8;
      hh[v] = (h != nullptr && col < d && b < rend) ? __ldg(reinterpret_cast<const uint4*>(h + (long)b * ldh + col))
                                                    : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int j = 0; j < EPL; ++j) ww[j] = (j < EW && b < rend) ? __ldg(&umask[(long)b * EW + j]) : 0u;
  };
  fetch(row0, hv, wv);
  const uint32_t lt = (1u << lane) - 1u;
  for (int b = row0; b < rend; ++b) {
    uint4 hn[VEC];
    uint32_t wn[EPL];
    fetch(b + 1, hn, wn);
    int u = 0;
#pragma unroll
    for (int j = 0; j < EPL; ++j) {
      if (j >= EW) break;
      uint32_t word = wv[j];
      const int my_r = run[j];
      if ((word >> lane) & 1u) {
        run[j]++;
        const int rank = u + __popc(word & lt);
        row_of[(long)b * umax + rank] = my_r;
        gather_inst[my_r] = b;
        gather_exp[my_r] = j * 32 + lane;
      }
      u += __popc(word);
      while (word) {
        int bit = __ffs(word) - 1;
        word &= word - 1;
        int r = __shfl_sync(0xffffffffu, my_r, bit);
#pragma unroll
        for (int v = 0; v < VEC; ++v) {
          int col = (v * 32 + lane) * 8;
          if (h != nullptr && col < d) *reinterpret_cast<uint4*>(X + (long)r * ldx + col) = hv[v];
        }
      }
    }
#pragma unroll
    for (int v = 0; v < VEC; ++v) hv[v] = hn[v];
#pragma unroll
    for (int j = 0; j < EPL; ++j) wv[j] = wn[j];
  }
}

// chunk histograms of union membership for an arbitrary union bitmask (the
// build_execution_plan(unions, E) entry point, when no router ran before it)
__global__ void __launch_bounds__(PL_WARPS * 32)
    plan_counts_kernel(int B, int E, int rows_per_warp, const uint32_t* __restrict__ umask,
                       int32_t* __restrict__ chunk_union, int32_t* __restrict__ usize) {
  pdl_wait();
  __shared__ int32_t s_cnt[PL_WARPS][1024];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int EW = (E + 31) >> 5;
  const int row0 = blockIdx.x * PL_WARPS * rows_per_warp + warp * rows_per_warp;
  const int rend = min(row0 + rows_per_warp, B);
  for (int e = lane; e < E; e += 32) s_cnt[warp][e] = 0;
  __syncwarp();
  for (int b = row0; b < rend; ++b) {
    int sz = 0;
    for (int j = 0; j < EW; ++j) {
      const uint32_t w = umask[(long)b * EW + j];
      sz += __popc(w);
      const int e = j * 32 + lane;
      if (e < E && ((w >> lane) & 1u)) s_cnt[warp][e] += 1;
    }
    if (lane == 0) usize[b] = sz;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < E; e += blockDim.x) {
    int c = 0;
    for (int w = 0; w < PL_WARPS; ++w) c += s_cnt[w][e];
    chunk_union[(long)blockIdx.x * E + e] = c;
  }
}

}  // namespace smes

using namespace smes;

extern "C" {

int smes_plan_reduce(int C, int E, const int32_t* chunk_union, const int32_t* chunk_active, const double* chunk_mass,
                     const double* chunk_dmass, int32_t* chunk_base, int32_t* loads, double* stats_raw,
                     int32_t* seg_pad, int32_t* seg_log, int32_t* totals, unsigned int* ticket, int32_t* seg_half,
                     void* stream) {
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  smes_launch(chunk_reduce_kernel, E, 256, 0, st, C, E, chunk_union, chunk_active, chunk_mass, chunk_dmass,
              chunk_base, loads, stats_raw, seg_pad, seg_log, totals, ticket, seg_half, 1.0, 1.0, 0, nullptr, nullptr);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_error(SMES_ERR_CUDA, "plan_reduce launch: %s", cudaGetErrorString(e));
  return SMES_OK;
}

int smes_plan_reduce_work_ints(int C, int E) { (void)C; (void)E; return 1; }   // the ticket

int smes_plan_reduce_stats(int C, int E, const int32_t* chunk_union, const int32_t* chunk_active,
                           const double* chunk_mass, const double* chunk_dmass, int32_t* chunk_base, int32_t* loads,
                           double* stats_raw, int32_t* seg_pad, int32_t* seg_log, int32_t* totals,
                           unsigned int* ticket, int32_t* seg_half, int K, int lb_experts, double batch_times_tasks,
                           int dense, double* stats_out, float* freq_f32, void* stream) {
  if (E > 1024) return set_error(SMES_ERR_SHAPE, "plan: E=%d exceeds 1024", E);
  if (K < 1 || batch_times_tasks <= 0.0) return set_error(SMES_ERR_CONFIG, "plan_reduce_stats: K=%d B*T=%g", K,
                                                          batch_times_tasks);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  smes_launch(chunk_reduce_kernel, E, 256, 0, st, C, E, chunk_union, chunk_active, chunk_mass, chunk_dmass,
              chunk_base, loads, stats_raw, seg_pad, seg_log, totals, ticket, seg_half,
              (double)(lb_experts > 0 ? lb_experts : E) / (double)K, batch_times_tasks, dense, stats_out, freq_f32);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_error(SMES_ERR_CUDA, "plan_reduce launch: %s", cudaGetErrorString(e));
  return SMES_OK;
}

int smes_plan_reduce_stats_fold(int C, int E, const int32_t* chunk_union, const int32_t* chunk_active,
                                const double* chunk_mass, const double* chunk_dmass, int32_t* chunk_base,
                                int32_t* loads, double* stats_raw, int32_t* seg_pad, int32_t* seg_log, int32_t* totals,
                                unsigned int* ticket, int32_t* seg_half, int K, int lb_experts,
                                double batch_times_tasks, int dense, double* stats_out, float* freq_f32, int T,
                                int ldg, int d_out, int d_in, const float* head_w, const void* W, const float* b,
                                void* G, float* c, void* stream) {
  if (E > 1024) return set_error(SMES_ERR_SHAPE, "plan: E=%d exceeds 1024", E);
  if (K < 1 || batch_times_tasks <= 0.0) return set_error(SMES_ERR_CONFIG, "plan_reduce_stats: K=%d B*T=%g", K,
                                                          batch_times_tasks);
  if (!smes_fold_full_supported(E, T, ldg, d_out, d_in))
    return set_error(SMES_ERR_SHAPE, "plan_reduce_stats_fold: fold shape T=%d ldg=%d d_out=%d d_in=%d", T, ldg, d_out,
                     d_in);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const FoldArgsPR f{T, ldg, d_out, d_in, head_w, reinterpret_cast<const __nv_bfloat16*>(W), b,
                     reinterpret_cast<__nv_bfloat16*>(G), c};
  const int nfold = ((d_in + 63) / 64) * E;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(plan_reduce_fold_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, fold_full_smem_bytes<8>());
    attr = true;
  }
  smes_launch(plan_reduce_fold_kernel, E + nfold, 256, fold_full_smem_bytes<8>(), st, C, E, chunk_union, chunk_active,
              chunk_mass, chunk_dmass, chunk_base, loads, stats_raw, seg_pad, seg_log, totals, ticket, seg_half,
              (double)(lb_experts > 0 ? lb_experts : E) / (double)K, batch_times_tasks, dense, stats_out, freq_f32, f);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_error(SMES_ERR_CUDA, "plan_reduce_fold launch: %s", cudaGetErrorString(e));
  return SMES_OK;
}

int smes_plan_counts(int B, int E, int rows_per_warp, const uint32_t* umask, int32_t* chunk_union, int32_t* usize,
                     void* stream) {
  if (E > 1024) return set_error(SMES_ERR_SHAPE, "plan: E=%d exceeds 1024", E);
  const int C = (B + PL_WARPS * rows_per_warp - 1) / (PL_WARPS * rows_per_warp);
  smes_launch(plan_counts_kernel, C, PL_WARPS * 32, 0, reinterpret_cast<cudaStream_t>(stream), B, E, rows_per_warp, umask,
                                                                                     chunk_union, usize);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_error(SMES_ERR_CUDA, "plan_counts launch: %s", cudaGetErrorString(e));
  return SMES_OK;
}

int smes_plan_scatter(int B, int E, int d, int rows_per_warp, const uint32_t* umask, const int32_t* chunk_base,
                      const int32_t* seg_pad, const int32_t* loads, const void* h, long ldh, void* X, long ldx,
                      int32_t* row_of, int umax, int32_t* gather_inst, int32_t* gather_exp, void* zero_rows2,
                      long ldz2, int d2, void* stream) {
  if (E > 1024) return set_error(SMES_ERR_SHAPE, "plan: E=%d exceeds 1024", E);
  if (d % 8 || d > 2048 || (zero_rows2 && d2 % 8))
    return set_error(SMES_ERR_SHAPE, "plan: d=%d must be a multiple of 8 and <= 2048", d);
  const int C = (B + PL_WARPS * rows_per_warp - 1) / (PL_WARPS * rows_per_warp);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const int epl = (E + 31) / 32;
  const int vec = (d + 255) / 256;
  dim3 grid(C + E);
  auto* hh = reinterpret_cast<const __nv_bfloat16*>(h);
  auto* xx = reinterpret_cast<__nv_bfloat16*>(X);
  auto* zz = reinterpret_cast<__nv_bfloat16*>(zero_rows2);
#define PL_CASE(EP, VV)                                                                                       \
  if (epl <= EP && vec <= VV) {                                                                               \
    smes_launch(scatter_kernel<EP, VV>, grid, PL_WARPS * 32, 0, st, B, E, d, rows_per_warp, umask, chunk_base, seg_pad, \
                                                           loads, hh, ldh, xx, ldx, row_of, umax, gather_inst, \
                                                           gather_exp, zz, ldz2, d2);                          \
  } else
  PL_CASE(1, 1) PL_CASE(1, 2) PL_CASE(1, 4) PL_CASE(1, 8) PL_CASE(2, 1) PL_CASE(2, 2) PL_CASE(2, 4) PL_CASE(2, 8)
  PL_CASE(8, 1) PL_CASE(8, 2) PL_CASE(8, 4) PL_CASE(8, 8) PL_CASE(32, 2) PL_CASE(32, 4) PL_CASE(32, 8) {}
#undef PL_CASE
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_error(SMES_ERR_CUDA, "plan_scatter launch: %s", cudaGetErrorString(e));
  return SMES_OK;
}

}  // extern "C"
