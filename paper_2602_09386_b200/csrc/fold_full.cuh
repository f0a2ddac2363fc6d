// fold_full: the single-launch head fold for d_out <= 256 (csrc/fold.cu), shared with plan.cu.
#pragma once
#include "ptx.cuh"

namespace smes {

// Single-launch fold for d_out <= 256 (the c1/c2 shapes): a block owns (64 columns k, expert e),
// loads all of W_e[:, k-tile] (d_out x 64 bf16, one memory latency) and head_w, and reduces over
// the full d_out -- no split partials, no finish pass.  Blocks with k-tile 0 also write c_e.
// Runs as its own kernel (fold_full_kernel) or as the extra blocks of the plan reduce
// (plan_reduce_fold_kernel, plan.cu), whose column scans leave most SMs idle.  256 threads,
// fold_full_smem_bytes<TM>() of dynamic shared memory.
constexpr int FOLD_FULL_MAX_DOUT = 256;
template <int TM>
__host__ __device__ constexpr int fold_full_smem_bytes() {
  return FOLD_FULL_MAX_DOUT * 72 * 2 + TM * (FOLD_FULL_MAX_DOUT + 4) * 4;
}
template <int TM>
__device__ __forceinline__ void fold_full_body(int bx, int e, int T, int ldg, int d_out, int d_in,
                                               const float* __restrict__ head_w, const __nv_bfloat16* __restrict__ W,
                                               const float* __restrict__ b, __nv_bfloat16* __restrict__ G,
                                               float* __restrict__ c, uint8_t* smem) {
  // W tile (d_out x 64 bf16, padded rows); reused as the [8][TM][64] fp32 group-sum buffer
  auto sW = reinterpret_cast<__nv_bfloat16 (*)[72]>(smem);
  static_assert(FOLD_FULL_MAX_DOUT * 72 * 2 >= 8 * TM * 64 * 4, "fold_full reduction buffer");
  auto sX = reinterpret_cast<float (*)[FOLD_FULL_MAX_DOUT + 4]>(smem + FOLD_FULL_MAX_DOUT * 72 * 2);
  const int k0 = bx * 64, tid = threadIdx.x;
  const __nv_bfloat16* We = W + (size_t)e * d_out * d_in;
  for (int idx = tid; idx < d_out * 8; idx += 256) {
    const int row = idx >> 3, cg = (idx & 7) * 8;
    uint4 v = make_uint4(0, 0, 0, 0);
    if (k0 + cg < d_in) v = __ldg(reinterpret_cast<const uint4*>(We + (size_t)row * d_in + k0 + cg));
    *reinterpret_cast<uint4*>(&sW[row][cg]) = v;
  }
  for (int i = tid; i < TM * d_out; i += 256) {
    const int t = i / d_out, j = i - t * d_out;
    sX[t][j] = t < T ? head_w[(size_t)t * d_out + j] : 0.f;
  }
  __syncthreads();
  // thread = (column pair cp, j-group g): all TM tasks for 2 columns over d_out/8 rows j, then a
  // fixed-order sum of the 8 j-groups through shared memory
  const int cp = tid & 31, g = tid >> 5;
  const int jn = (d_out + 7) / 8, ja = g * jn, jb = min(d_out, ja + jn);
  float acc[TM][2];
#pragma unroll
  for (int t = 0; t < TM; ++t) { acc[t][0] = 0.f; acc[t][1] = 0.f; }
  for (int j = ja; j < jb; ++j) {
    const float2 w = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&sW[j][2 * cp]));
#pragma unroll
    for (int t = 0; t < TM; ++t) {
      const float x = sX[t][j];
      acc[t][0] = fmaf(x, w.x, acc[t][0]);
      acc[t][1] = fmaf(x, w.y, acc[t][1]);
    }
  }
  __syncthreads();                                           // sW is reused as the reduction buffer
  float* red = reinterpret_cast<float*>(&sW[0][0]);          // [8 groups][TM][64]
#pragma unroll
  for (int t = 0; t < TM; ++t) {
    red[(g * TM + t) * 64 + 2 * cp] = acc[t][0];
    red[(g * TM + t) * 64 + 2 * cp + 1] = acc[t][1];
  }
  __syncthreads();
  for (int i = tid; i < TM * 64; i += 256) {
    const int t = i >> 6, col = i & 63;
    float v = 0.f;
#pragma unroll
    for (int gg = 0; gg < 8; ++gg) v += red[(gg * TM + t) * 64 + col];
    if (t < ldg && k0 + col < d_in) G[((size_t)e * ldg + t) * d_in + k0 + col] = __float2bfloat16_rn(v);
  }
  if (bx == 0) {
    const int warp = tid >> 5, lane = tid & 31;
    for (int t = warp; t < ldg; t += 8) {
      float s = 0.f;
      if (t < T)
        for (int j = lane; j < d_out; j += 32) s = fmaf(sX[t][j], b[(size_t)e * d_out + j], s);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (lane == 0) c[(size_t)e * ldg + t] = s;
    }
  }
}

}  // namespace smes
