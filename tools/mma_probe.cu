// Microbenchmark (profiling aid, not part of the library): tcgen05.mma throughput and
// issue->commit latency on one SM, alone and with concurrent TMEM loads / smem stores from
// 8 epilogue-like warps.   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17
//   -I paper_2602_09386_b200/csrc tools/mma_probe.cu -o /tmp/mma_probe -lcuda
#include <cstdio>
#include <vector>

#include "ptx.cuh"

using namespace smes;

struct Res {
  long long cyc;
};

// mode bit 0: epilogue warps spin on tcgen05.ld of cols [256, 384); bit 1: they spin on st.shared
// of a 32 KB region; bit 2: MMAs are dependent chains of `chain` on one accumulator, else they
// rotate over 2 accumulators
__global__ void __launch_bounds__(384, 1) probe(int n_mma, int N, int mode, long long* out) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = sm_raw + ((1024u - (smem_u32(sm_raw) & 1023u)) & 1023u);
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + 3 * 32768);
  uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 2);
  volatile int* stop = reinterpret_cast<volatile int*>(slot + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 3 * 32768 / 16; i += blockDim.x) reinterpret_cast<uint4*>(sm)[i] = make_uint4(0, 0, 0, 0);
  if (threadIdx.x == 0) { mbar_init(bar, 1); *stop = 0; fence_mbar_init(); }
  if (warp == 2) tmem_alloc(slot, 512);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *slot;
  if (warp == 1 && lane == 0) {
    const uint32_t idesc = umma_idesc_bf16(128, N, 0, 0);
    const uint32_t a = smem_u32(sm), b = smem_u32(sm + 32768);
    // warm
    tc_mma_f16(tmem, umma_desc_sw128(a, 16, 1024), umma_desc_sw128(b, 16, 1024), idesc, 0);
    tc_commit(bar);
    mbar_wait(bar, 0);
    long long t0 = clock64();
    for (int i = 0; i < n_mma; ++i) {
      const uint32_t d = (mode & 4) ? tmem : tmem + ((i & 1) ? 0 : 0);
      tc_mma_f16(d, umma_desc_sw128(a + (i & 3) * 32, 16, 1024), umma_desc_sw128(b + (i & 3) * 32, 16, 1024), idesc,
                 1);
    }
    long long t_issue = clock64();
    tc_commit(bar);
    mbar_wait(bar, 1);
    long long t1 = clock64();
    // single-MMA latency
    tc_mma_f16(tmem, umma_desc_sw128(a, 16, 1024), umma_desc_sw128(b, 16, 1024), idesc, 1);
    tc_commit(bar);
    mbar_wait(bar, 0);
    long long t2 = clock64();
    *stop = 1;
    if (blockIdx.x == 0) { out[0] = t_issue - t0; out[1] = t1 - t0; out[2] = t2 - t1; }
  } else if (warp >= 4) {
    long long n = 0;
    const int q = warp & 3;
    uint8_t* dst = sm + 65536 + (warp - 4) * 4096 + lane * 128;
    while (!*stop) {
      if (mode & 1) {
        uint32_t r[32];
        tmem_ld32(tmem + ((uint32_t)(32 * q) << 16) + 256 + ((warp - 4) >> 2) * 32, r);
        tmem_ld_wait();
        n += r[0] & 1;
      }
      if (mode & 2) {
#pragma unroll
        for (int c = 0; c < 8; ++c) reinterpret_cast<uint4*>(dst)[c] = make_uint4(n, c, 1, 2);
        ++n;
      }
      if (!(mode & 3)) break;
    }
    if (n == 12345678) out[3] = n;
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_dealloc(tmem, 512);
}

// Pipeline probe: S-MMA issuer (k MMAs of N=128 per chunk into a double-buffered accumulator)
// + 8 epilogue warps (wait sfull, tcgen05.ld 2 x 32 cols, arrive sempty) [+ P-MMA warp chained
// through hfull/hempty when pm > 0].  Returns cycles per chunk.
__global__ void __launch_bounds__(384, 1) pipe_probe(int chunks, int kmma, int pm, long long* out, int epi = 0) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = sm_raw + ((1024u - (smem_u32(sm_raw) & 1023u)) & 1023u);
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + 3 * 32768);
  uint64_t* sfull = bar; uint64_t* sempty = bar + 2; uint64_t* hfull = bar + 4; uint64_t* hempty = bar + 5;
  uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 8);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 3 * 32768 / 16; i += blockDim.x) reinterpret_cast<uint4*>(sm)[i] = make_uint4(0, 0, 0, 0);
  if (threadIdx.x == 0) {
    for (int i = 0; i < 2; ++i) { mbar_init(&sfull[i], 1); mbar_init(&sempty[i], 8); }
    mbar_init(hfull, 8); mbar_init(hempty, 1);
    mbar_init(&bar[7], 1);
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc(slot, 512);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *slot;
  long long t0 = clock64();
  if (warp == 1 && lane == 0) {
    const uint32_t idesc = umma_idesc_bf16(128, 128, 0, 0);
    const uint32_t a = smem_u32(sm), b = smem_u32(sm + 32768);
    for (int si = 0; si < chunks; ++si) {
      const int sb = si & 1;
      mbar_wait(&sempty[sb], ((si >> 1) & 1) ^ 1);
      tc_fence_after();
      for (int k = 0; k < kmma; ++k) {
        tc_mma_f16(tmem + sb * 128, umma_desc_sw128(a + (k & 3) * 32, 16, 1024),
                   umma_desc_sw128(b + (k & 3) * 32, 16, 1024), idesc, k != 0);
        if ((epi & 16) && (k & 3) == 3) tc_commit(&bar[7]);     // per-k-block commit (stage release)
      }
      tc_commit(&sfull[sb]);
    }
  } else if (warp == 3 && lane == 0 && pm > 0) {
    const uint32_t idesc = umma_idesc_bf16(128, 16, 0, 0);
    const uint32_t a = smem_u32(sm + 65536), b = smem_u32(sm + 32768);
    for (int hi = 0; hi < chunks; ++hi) {
      mbar_wait(hfull, hi & 1);
      tc_fence_after();
      for (int k = 0; k < pm; ++k)
        tc_mma_f16(tmem + 256, umma_desc_sw128(a + (k & 3) * 32, 16, 1024), umma_desc_sw128(b + (k & 3) * 32, 16, 1024),
                   idesc, k != 0);
      tc_commit(hempty);
    }
  } else if (warp >= 4) {
    const int q = warp & 3, par = (warp - 4) >> 2;
    uint32_t acc = 0;
    for (int si = 0; si < chunks; ++si) {
      const int sb = si & 1;
      mbar_wait(&sfull[sb], (si >> 1) & 1);
      tc_fence_after();
      uint32_t t0r[32], t1r[32];
      const uint32_t ta = tmem + ((uint32_t)(32 * q) << 16) + sb * 128 + par * 64;
      tmem_ld32(ta, t0r);
      tmem_ld32(ta + 32, t1r);
      tmem_ld_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&sempty[sb]);
      float f[64];
#pragma unroll
      for (int j = 0; j < 32; ++j) { f[j] = __uint_as_float(t0r[j]); f[32 + j] = __uint_as_float(t1r[j]); }
      if (epi & 1) {          // bias + relu through a warp-private smem broadcast
        float* sbias = reinterpret_cast<float*>(sm + 98304 + 2048) + (warp - 4) * 64;
        sbias[lane] = (float)si;
        sbias[32 + lane] = (float)lane;
        __syncwarp();
#pragma unroll
        for (int j = 0; j < 64; j += 4) {
          const float4 bb = *reinterpret_cast<const float4*>(sbias + j);
          f[j] = fmaxf(f[j] + bb.x, 0.f); f[j + 1] = fmaxf(f[j + 1] + bb.y, 0.f);
          f[j + 2] = fmaxf(f[j + 2] + bb.z, 0.f); f[j + 3] = fmaxf(f[j + 3] + bb.w, 0.f);
        }
      }
      if (epi & 2) {          // relu bit-masks to global
        for (int h = 0; h < 2; ++h) out[8 + (h * 8 + (warp - 4)) * 32 + lane] = pos_mask32(f + h * 32);
      }
      if (pm > 0) {
        mbar_wait(hempty, (si & 1) ^ 1);
        if (epi & 4) {        // H tile (bf16, SW128) into smem
          uint8_t* hrow = sm + 65536 + ((warp - 4) >> 2) * 16384 + (32 * q + lane) * 128;
#pragma unroll
          for (int cc = 0; cc < 8; ++cc) {
            const uint4 pk = make_uint4(pack_bf16(f[8 * cc], f[8 * cc + 1]), pack_bf16(f[8 * cc + 2], f[8 * cc + 3]),
                                        pack_bf16(f[8 * cc + 4], f[8 * cc + 5]), pack_bf16(f[8 * cc + 6], f[8 * cc + 7]));
            *reinterpret_cast<uint4*>(hrow + ((cc ^ (lane & 7)) << 4)) = pk;
          }
        } else {
#pragma unroll
          for (int j = 0; j < 64; ++j) acc += __float_as_uint(f[j]);
        }
        if (!(epi & 8)) fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(hfull);
      }
    }
    if (acc == 0x12345) out[5] = acc;
    if (pm > 0 && warp == 4 && lane == 0) mbar_wait(hempty, (chunks & 1) ^ 1);
    if (warp == 4 && lane == 0 && blockIdx.x == 0) out[0] = clock64() - t0;
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_dealloc(tmem, 512);
}

// MMA throughput (N=128, independent of the epilogue) while one warp streams 1D bulk copies
// (global -> smem, `inflight` x 16 KB in flight) from an L2-resident buffer.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__global__ void __launch_bounds__(384, 1) tma_probe(int n_mma, int inflight, const uint8_t* src, long long* out) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = sm_raw + ((1024u - (smem_u32(sm_raw) & 1023u)) & 1023u);
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + 6 * 32768);
  uint64_t* cb = bar + 2;              // [8] copy barriers
  uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 12);
  volatile int* stop = reinterpret_cast<volatile int*>(slot + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    for (int i = 0; i < 8; ++i) mbar_init(&cb[i], 1);
    *stop = 0;
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc(slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *slot;
  if (warp == 1 && lane == 0) {
    const uint32_t idesc = umma_idesc_bf16(128, 128, 0, 0);
    const uint32_t a = smem_u32(sm), b = smem_u32(sm + 32768);
    for (int w = 0; w < 64; ++w)      // let the copy stream ramp
      tc_mma_f16(tmem, umma_desc_sw128(a, 16, 1024), umma_desc_sw128(b, 16, 1024), idesc, 1);
    tc_commit(bar);
    mbar_wait(bar, 0);
    long long t0 = clock64();
    for (int i = 0; i < n_mma; ++i)
      tc_mma_f16(tmem + (i & 1) * 128, umma_desc_sw128(a + (i & 3) * 32, 16, 1024),
                 umma_desc_sw128(b + (i & 3) * 32, 16, 1024), idesc, 1);
    tc_commit(bar);
    mbar_wait(bar, 1);
    long long t1 = clock64();
    *stop = 1;
    if (blockIdx.x == 0) out[0] = t1 - t0;
  } else if (warp == 0 && lane == 0 && inflight > 0) {
    long long n = 0, bytes = 0;
    long long t0 = clock64();
    const uint8_t* base = src + (size_t)blockIdx.x * (1 << 20);
    for (int i = 0; i < inflight; ++i) {
      mbar_expect_tx(&cb[i], 16384);
      bulk_g2s(sm + 65536 + i * 16384, base + (i * 16384) % (1 << 20), 16384, &cb[i]);
    }
    for (long long i = 0; !*stop; ++i) {
      const int s = (int)(i % inflight);
      mbar_wait(&cb[s], (uint32_t)((i / inflight) & 1));
      bytes += 16384;
      mbar_expect_tx(&cb[s], 16384);
      bulk_g2s(sm + 65536 + s * 16384, base + ((i + inflight) * 16384) % (1 << 20), 16384, &cb[s]);
      ++n;
    }
    for (int i = 0; i < inflight; ++i) mbar_wait(&cb[(n + i) % inflight], (uint32_t)(((n + i) / inflight) & 1));
    if (blockIdx.x == 0) { out[1] = bytes; out[2] = clock64() - t0; }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_dealloc(tmem, 512);
}

int main() {
  long long* d_out;
  cudaMalloc(&d_out, 1 << 16);
  const int smem = 3 * 32768 + 2048;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int grid : {1, 148}) {
    for (int N : {16, 128, 256}) {
      for (int mode : {0, 4, 1, 2, 3}) {
        const int n_mma = 512;
        probe<<<grid, 384, smem>>>(n_mma, N, mode, d_out);
        cudaError_t e = cudaDeviceSynchronize();
        long long h[4];
        cudaMemcpy(h, d_out, 32, cudaMemcpyDeviceToHost);
        const double floor = 128.0 * N / 256.0;
        printf("grid %3d N %3d mode %d (%s%s%s): issue %.1f cyc/mma, complete %.1f cyc/mma (floor %.0f), "
               "single latency %lld  %s\n",
               grid, N, mode, mode & 1 ? "tmem-ld " : "", mode & 2 ? "sts " : "", mode & 4 ? "dep" : "",
               (double)h[0] / n_mma, (double)h[1] / n_mma, floor, h[2], e == cudaSuccess ? "" : cudaGetErrorString(e));
      }
    }
  }
  {
    uint8_t* src;
    cudaMalloc(&src, (size_t)148 << 20);
    cudaMemset(src, 0, (size_t)148 << 20);
    const int smem2 = 6 * 32768 + 2048;
    cudaFuncSetAttribute(tma_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem2);
    for (int inflight : {0, 2, 4, 8}) {
      const int n_mma = 2048;
      tma_probe<<<148, 384, smem2>>>(n_mma, inflight, src, d_out);
      cudaError_t e = cudaDeviceSynchronize();
      long long h[3];
      cudaMemcpy(h, d_out, 24, cudaMemcpyDeviceToHost);
      printf("tma: %d x 16KB in flight: MMA %.1f cyc/mma (floor 64); copy %.1f B/cyc  %s\n", inflight,
             (double)h[0] / n_mma, inflight ? (double)h[1] / h[2] : 0.0, e == cudaSuccess ? "" : cudaGetErrorString(e));
    }
  }
  const int smem3 = 3 * 32768 + 8192;
  cudaFuncSetAttribute(pipe_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem3);
  for (int epi : {0, 16, 7, 23}) {
    const int pm = 8, kmma = 16;
    {
      const int chunks = 256;
      pipe_probe<<<148, 384, smem3>>>(chunks, kmma, pm, d_out, epi);
      cudaError_t e = cudaDeviceSynchronize();
      long long h[1];
      cudaMemcpy(h, d_out, 8, cudaMemcpyDeviceToHost);
      printf("pipe: epi %2d (bias-relu %d bits %d H-sts %d no-fence %d) S-MMAs/chunk %2d P-MMAs/chunk %d: %.0f cycles/chunk %s\n",
             epi, epi & 1, (epi >> 1) & 1, (epi >> 2) & 1, (epi >> 3) & 1, kmma, pm, (double)h[0] / chunks,
             e == cudaSuccess ? "" : cudaGetErrorString(e));
    }
  }
  return 0;
}
