// One-shot all-reduce over CUDA-IPC-mapped peer memory (NVLink / NVSwitch) for the small,
// latency-critical exchange of a data-parallel step: the 3E raw LoadStats sums (counts, sparse
// and dense mass), which the regularizer needs as global-batch means (balance.py:62-70).
//
// Every rank stores its vector straight into slot [me] of every peer's receive buffer, raises
// its flag in every peer's flag array, waits for all n flags, then sums the n slots in rank
// order: the result is bitwise identical on every rank and deterministic.  The epoch lives on the
// device (incremented by the kernel), so the exchange can be captured in a CUDA graph and
// replayed.  Receive buffers are double-buffered by epoch parity: a rank can only reach epoch
// e + 2 (writing parity e again) after every peer raised its epoch e + 1 flag, which each peer
// does only after it finished reading epoch e.
#include "ptx.cuh"
#include "smes_capi.h"

namespace smes {

__device__ __forceinline__ void st_release_sys(int32_t* p, int32_t v) {
  asm volatile("st.release.sys.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ int32_t ld_acquire_sys(const int32_t* p) {
  int32_t v;
  asm volatile("ld.acquire.sys.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// recv layout (every rank): [2 parities][n ranks][count] fp64; flags: [n] int32; epoch: 1 int32
__global__ void __launch_bounds__(512) peer_allreduce_f64_kernel(int n, int me, int count, const double* __restrict__ in,
                                                                 double* const* __restrict__ peer_recv,
                                                                 int32_t* const* __restrict__ peer_flags,
                                                                 const double* __restrict__ my_recv,
                                                                 int32_t* __restrict__ my_flags,
                                                                 int32_t* __restrict__ epoch_ctr,
                                                                 double* __restrict__ out) {
  pdl_wait();
  __shared__ int32_t s_epoch;
  if (threadIdx.x == 0) s_epoch = *epoch_ctr + 1;
  __syncthreads();
  const int32_t epoch = s_epoch;
  const size_t par = (size_t)(epoch & 1) * n * count;
  for (int p = 0; p < n; ++p) {
    double* dst = peer_recv[p] + par + (size_t)me * count;
    for (int i = threadIdx.x; i < count; i += blockDim.x) dst[i] = in[i];
  }
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x < n) st_release_sys(peer_flags[threadIdx.x] + me, epoch);
  if (threadIdx.x < n)
    while (ld_acquire_sys(my_flags + threadIdx.x) < epoch) {
    }
  __syncthreads();
  __threadfence_system();
  for (int i = threadIdx.x; i < count; i += blockDim.x) {
    double s = 0.0;     // rank order: the same bits on every rank
    for (int p = 0; p < n; ++p) s += __ldcv(my_recv + par + (size_t)p * count + i);   // peers' stores, no stale L1
    out[i] = s;
  }
  if (threadIdx.x == 0) *epoch_ctr = epoch;
}

}  // namespace smes

using namespace smes;

extern "C" {

int smes_peer_allreduce_f64(int n, int me, int count, const double* in, void* const* peer_recv_dev,
                            int32_t* const* peer_flags_dev, const double* my_recv, int32_t* my_flags,
                            int32_t* epoch_ctr, double* out, void* stream) {
  if (n < 1 || n > 512 || me < 0 || me >= n) return set_error(SMES_ERR_SHAPE, "peer_allreduce: rank %d of %d", me, n);
  if (count < 0) return set_error(SMES_ERR_SHAPE, "peer_allreduce: count %d", count);
  smes_launch(peer_allreduce_f64_kernel, 1, 512, 0, reinterpret_cast<cudaStream_t>(stream), 
      n, me, count, in, reinterpret_cast<double* const*>(peer_recv_dev), peer_flags_dev, my_recv, my_flags,
      epoch_ctr, out);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_error(SMES_ERR_CUDA, "peer_allreduce launch: %s", cudaGetErrorString(e));
  return SMES_OK;
}

}  // extern "C"
